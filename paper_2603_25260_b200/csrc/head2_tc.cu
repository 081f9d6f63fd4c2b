// head2_tc.cu — occupancy predictor (Eq.7) + integer softmax to a Q16 pmf
// (Eq.15; readings Q20-Q22), TWO threads per node.
//
// TMEM holds two 128 x 256 int32 logit tiles per SM (512 columns), which caps the
// one-thread-per-node kernel (head1_tc.cu) at 8 warps per SM, latency-bound.  Here each
// node's 256 logit columns are split between two threads in two warps (column halves
// [0,128) and [128,256) of the same TMEM lane), so one CTA per SM runs 16 warps: 2 tile
// groups x (4 lane quarters x 2 column halves).  The two halves exchange one pair of
// values twice per tile (partial max, partial mass) through shared memory with a named
// barrier of the tile group.  Per tile:
//   1. hidden layer a = prq(W1 F + b1): each half computes H/2 of the node's hidden
//      units into the tcgen05 A operand; b2 of its 128 columns into its TMEM lane;
//   2. one tcgen05.mma.kind::i8 (M = 128, N = 256, K = 32): z = b2 + a W2^T;
//   3. pass 1: partial max z (min z if the model can saturate) of the half; exchange;
//      mu = l(max z) (the Q8 logit requant is monotone);
//   4. pass 2: delta = mu - l(z), e = LUT[delta >> 2] (0 beyond 16 nats) from a 32-copy
//      interleaved table (conflict-free), 16-symbol block sums and the half's mass;
//      exchange; encoder: the half holding the true symbol writes (C_sym, freq) (two exact
//      divisions, reading Q21); decoder: both halves stage their parts of the 112-byte
//      row (S, 65281 * 2^32 / S, mu, E_{16k}, a) and the group copies the rows out.
// Bit-exact with the oracle's head_logits / cdf_quantize.
#include "pcc_internal.cuh"
#include "rq.cuh"
#include "tc.cuh"

namespace pcc {

namespace {

constexpr int TILE = 128, NT2 = 512, GT = 256;  // threads per CTA / per tile group
constexpr uint32_t IDESC = tc::idesc_i8(128, 256);

__device__ __forceinline__ int32_t lq8(int32_t z, const RQ& q) {  // Q8 logit, clamp +-2^24
  int64_t v = int64_t(z) * int64_t(q.mp);
  if (q.r > 0) v = (v + (int64_t(1) << (q.r - 1))) >> q.r;
  v = v < -(int64_t(1) << 24) ? -(int64_t(1) << 24) : (v > (int64_t(1) << 24) ? (int64_t(1) << 24) : v);
  return int32_t(v);
}

__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}

struct Smem2 {
  static constexpr int B = 0;                      // W2 operand 256 x 32 (8 KB)
  static constexpr int A = 8192;                   // a operands, one 128 x 32 tile per group (2 x 4 KB)
  static constexpr int B2 = A + 8192;              // b2 [256] (1 KB)
  static constexpr int W1 = B2 + 1024;             // W1 words [H][C/4] (<= 1 KB)
  static constexpr int B1 = W1 + 1024;             // b1 [H] (<= 256 B)
  static constexpr int XCH = B1 + 256;             // [group][half][128] x 2 u32: pass-1 exchange (4 KB)
  static constexpr int XS = XCH + 4096;            // [group][half][128] u32: pass-2 exchange (2 KB)
  static constexpr int MBAR = XS + 2048;           // 2 mbarriers
  static constexpr int THOLD = MBAR + 16;
  static constexpr int STAGE = MBAR + 128;         // decoder: [group][128][DROW_BYTES] (28 KB)
  static constexpr int LUT = STAGE + 2 * TILE * DROW_BYTES;  // [1025][32] u32 (131 KB)
  static constexpr int END = LUT + 1025 * 32 * 4;
};

template <int C, int H, int MODE, bool SAT>
__global__ void __launch_bounds__(NT2, 1) k_head2_tc(const int8_t* __restrict__ F, uint32_t n,
                                                     const int8_t* __restrict__ W1, const int32_t* __restrict__ b1, RQ rq1,
                                                     const int8_t* __restrict__ W2, const int32_t* __restrict__ b2, RQ rql,
                                                     const uint32_t* __restrict__ lut, const uint8_t* __restrict__ X,
                                                     uint32_t* __restrict__ cf, uint8_t* __restrict__ rows,
                                                     int8_t* __restrict__ a_dbg, int32_t zsat_lo, int32_t zsat_hi) {
  extern __shared__ __align__(1024) uint8_t sm[];
  using S = Smem2;
  constexpr int CW = C / 4, HW = H / 4, HH = H / 2;  // HH hidden units per half
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tg = warp >> 3;              // tile group
  const int hf = (warp >> 2) & 1;        // column half
  const int r = 32 * (warp & 3) + lane;  // node of the group's tile = TMEM lane
  const int gt = tid & (GT - 1);         // thread within the group
  uint8_t* sB = sm + S::B;
  uint8_t* sA = sm + S::A + 4096 * tg;
  int32_t* sb2 = reinterpret_cast<int32_t*>(sm + S::B2);
  int32_t* sW1 = reinterpret_cast<int32_t*>(sm + S::W1);
  int32_t* sb1 = reinterpret_cast<int32_t*>(sm + S::B1);
  uint32_t* xch = reinterpret_cast<uint32_t*>(sm + S::XCH) + tg * 2 * 2 * TILE;  // [half][128][2]
  uint32_t* xs = reinterpret_cast<uint32_t*>(sm + S::XS) + tg * 2 * TILE;        // [half][128]
  uint8_t* stage = sm + S::STAGE + tg * TILE * DROW_BYTES;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + S::MBAR) + tg;
  uint32_t* thold = reinterpret_cast<uint32_t*>(sm + S::THOLD);

  for (int k = tid; k < 256 * 8; k += NT2) {
    const int rr = k >> 3, w = k & 7;
    const uint32_t v = (w < HW) ? reinterpret_cast<const uint32_t*>(W2)[rr * HW + w] : 0u;
    *reinterpret_cast<uint32_t*>(sB + tc::kmaj_off(rr, 4 * w)) = v;
  }
  for (int k = tid; k < 2048; k += NT2) reinterpret_cast<uint32_t*>(sm + S::A)[k] = 0u;  // K padding stays 0
  for (int k = tid; k < 2 * TILE * DROW_BYTES / 4; k += NT2) reinterpret_cast<uint32_t*>(sm + S::STAGE)[k] = 0u;
  for (int k = tid; k < 1025 * 32; k += NT2) {
    const int idx = k >> 5;  // delta >= 4096 (16 nats): index 1024, e = 0 (reading Q20)
    reinterpret_cast<uint32_t*>(sm + S::LUT)[k] = idx < 1024 ? lut[idx] : 0u;
  }
  for (int k = tid; k < 256; k += NT2) sb2[k] = b2[k];
  for (int k = tid; k < H * CW; k += NT2) sW1[k] = reinterpret_cast<const int32_t*>(W1)[k];
  for (int k = tid; k < H; k += NT2) sb1[k] = b1[k];
  if (warp == 0) tc::tmem_alloc<512>(thold);
  if (tid < 2) tc::mbar_init(reinterpret_cast<uint64_t*>(sm + S::MBAR) + tid, 1);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *thold + 256u * uint32_t(tg);  // the group's 256 columns
  const uint32_t taddr = tbase + (uint32_t(32 * (warp & 3)) << 16) + 128u * uint32_t(hf);
  const uint64_t adesc = tc::sdesc(tc::smem_u32(sA));
  const uint64_t bdesc = tc::sdesc(tc::smem_u32(sB));
  // word 32 idx + lane of the 32-copy table: byte offset ((min(delta, 4096) << 5) & ~127) | 4 lane
  const uint8_t* lutb = sm + S::LUT;
  const uint32_t lane4 = 4u * uint32_t(lane);
  auto lut_e = [&](uint32_t dl) -> uint32_t {
    const uint32_t off = (min(dl << 5, 4096u << 5) & ~127u) | lane4;  // dl < 2^26: no overflow
    return *reinterpret_cast<const uint32_t*>(lutb + off);
  };
  // fast form: X = z * (-M) + mu 2^32 + 2^31 - 1 >= 0 and delta = X >> 32; y = X >> 27 =
  // 32 delta + (0..31), and (min(y, 4096 * 32) & ~127) is exactly ((min(delta, 4096) >> 2) << 7)
  const uint32_t lutu = tc::smem_u32(lutb);
  auto lut_e_fast = [&](int32_t z, int32_t nM, int64_t C2) -> uint32_t {
    const uint32_t y = uint32_t(uint64_t(int64_t(z) * nM + C2) >> 27);
    const uint32_t off = (min(y, 4096u << 5) & ~127u) | lane4;
    uint32_t e;
    asm("ld.shared.u32 %0, [%1];" : "=r"(e) : "r"(lutu + off));
    return e;
  };
  const uint32_t ntiles = (n + TILE - 1) / TILE;
  const uint32_t tstride = 2u * gridDim.x;
  const int64_t lhalf = rql.r > 0 ? (int64_t(1) << (rql.r - 1)) : 0;
  auto bar_group = [&]() { asm volatile("bar.sync %0, 256;" ::"r"(1 + tg) : "memory"); };
  uint32_t phase = 0;

  auto load_f = [&](uint32_t tl, uint32_t (&fw)[CW]) {
    const uint32_t rw = tl * TILE + uint32_t(r);
    if (tl < ntiles && rw < n) {
      const uint32_t* src = reinterpret_cast<const uint32_t*>(F + size_t(rw) * C);
      if constexpr (CW % 4 == 0) {
#pragma unroll
        for (int w = 0; w < CW; w += 4) {
          const uint4 v = *reinterpret_cast<const uint4*>(src + w);
          fw[w] = v.x, fw[w + 1] = v.y, fw[w + 2] = v.z, fw[w + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int w = 0; w < CW; ++w) fw[w] = src[w];
      }
    } else {
#pragma unroll
      for (int w = 0; w < CW; ++w) fw[w] = 0u;
    }
  };
  // this half's H/2 hidden units of the node into the A operand (and the decoder's staged
  // row), then b2 of its 128 columns into its TMEM lane
  auto hidden_and_bias = [&](uint32_t tl, const uint32_t (&fw)[CW]) {
    const uint32_t rw = tl * TILE + uint32_t(r);
    uint32_t aw[HH / 4 > 0 ? HH / 4 : 1];
#pragma unroll
    for (int g4 = 0; g4 < HH / 4; ++g4) {
      int32_t hacc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int h = hf * HH + 4 * g4 + u;
        int32_t acc = sb1[h];
#pragma unroll
        for (int w = 0; w < CW; ++w) acc = __dp4a(int32_t(fw[w]), sW1[h * CW + w], acc);
        hacc[u] = acc;
      }
      if (rq1.fast_s)
        aw[g4] = pack_sat4(rq_s(hacc[0], rq1), rq_s(hacc[1], rq1), rq_s(hacc[2], rq1), rq_s(hacc[3], rq1));
      else
        aw[g4] = (uint32_t(rq8(hacc[0], rq1)) & 0xffu) | (uint32_t(rq8(hacc[1], rq1)) & 0xffu) << 8 |
                 (uint32_t(rq8(hacc[2], rq1)) & 0xffu) << 16 | (uint32_t(rq8(hacc[3], rq1)) & 0xffu) << 24;
      *reinterpret_cast<uint32_t*>(sA + tc::kmaj_off(uint32_t(r), hf * HH + 4 * g4)) = aw[g4];
      if (MODE == 1) reinterpret_cast<uint32_t*>(stage + r * DROW_BYTES + DROW_A + hf * HH)[g4] = aw[g4];
      if (a_dbg && rw < n) reinterpret_cast<uint32_t*>(a_dbg + size_t(rw) * H + hf * HH)[g4] = aw[g4];
    }
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) {
      uint32_t bv[16];
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        const uint4 b4 = *reinterpret_cast<const uint4*>(sb2 + 128 * hf + 16 * ch + 4 * k4);
        bv[4 * k4] = b4.x, bv[4 * k4 + 1] = b4.y, bv[4 * k4 + 2] = b4.z, bv[4 * k4 + 3] = b4.w;
      }
      st16(taddr + ch * 16, bv);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  };

  uint32_t fw[CW];
  const uint32_t t0 = 2u * blockIdx.x + uint32_t(tg);
  load_f(t0, fw);
  if (t0 < ntiles) hidden_and_bias(t0, fw);
  load_f(t0 + tstride, fw);
  for (uint32_t tile = t0; tile < ntiles; tile += tstride) {
    const uint32_t row = tile * TILE + uint32_t(r);
    const bool valid = row < n;
    // the group's A operand and bias-initialised accumulator are complete
    tc::fence_async_smem();
    tc::fence_before();
    bar_group();
    tc::fence_after();
    if (gt == 0) {
      tc::mma_i8(tbase, adesc, bdesc, IDESC, 1u);
      tc::commit(mbar);
    }
    tc::mbar_wait(mbar, phase);
    phase ^= 1u;
    tc::fence_after();

    // ---- pass 1: partial max z (and min z) of this half (column 255 is padding) ----
    int32_t zmx = INT32_MIN, zmn = INT32_MAX;
#pragma unroll 1
    for (int ch = 0; ch < 8; ++ch) {
      uint32_t v[16];
      ld16(taddr + ch * 16, v);
      tc::tmem_wait_ld();
      if (hf == 1 && ch == 7) v[15] = v[14];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        zmx = max(zmx, int32_t(v[k]));
        if (SAT) zmn = min(zmn, int32_t(v[k]));
      }
    }
    xch[(hf * TILE + r) * 2] = uint32_t(zmx);
    xch[(hf * TILE + r) * 2 + 1] = uint32_t(zmn);
    bar_group();
    zmx = max(zmx, int32_t(xch[((1 - hf) * TILE + r) * 2]));
    zmn = min(zmn, int32_t(xch[((1 - hf) * TILE + r) * 2 + 1]));
    const int32_t mu = lq8(zmx, rql);
    const bool nosat = !SAT || (zmx <= zsat_hi && zmn >= zsat_lo);
    const bool fastl = rql.fast_s && nosat;
    const int32_t nM = -rql.Sp;
    const int64_t C2 = (int64_t(mu) << 32) + 0x7fffffff;
    const int sym = (MODE == 0 && valid) ? int(X[row]) - 1 : -1;
    const int sl = sym - 128 * hf;  // the true symbol's column within this half (encoder)

    // ---- pass 2: e_i = LUT[(mu - l_i) >> 2], 16-symbol block sums, the half's mass ----
    uint32_t Sh = 0, pre = 0, es = 0;
    uint32_t Eb[8];  // decoder: mass before each of the half's blocks, within the half
#pragma unroll 1
    for (int ch = 0; ch < 8; ++ch) {
      uint32_t v[16];
      ld16(taddr + ch * 16, v);
      tc::tmem_wait_ld();
      if (fastl) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          v[k] = lut_e_fast(int32_t(v[k]), nM, C2);
        }
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int32_t zz = int32_t(v[k]);
          int32_t lv = int32_t((int64_t(zz) * int64_t(rql.mp) + lhalf) >> rql.r);
          if (SAT && !nosat) {
            lv = zz > zsat_hi ? (1 << 24) : lv;
            lv = zz < zsat_lo ? -(1 << 24) : lv;
          }
          v[k] = lut_e(uint32_t(mu - lv));
        }
      }
      if (hf == 1 && ch == 7) v[15] = 0u;  // column 255 is padding, not a symbol
      uint32_t cs = 0;
#pragma unroll
      for (int k = 0; k < 16; ++k) cs += v[k];
      if constexpr (MODE == 0) {
        const int i0 = 16 * ch;
        if (sl >= i0 + 16) {
          pre += cs;
        } else if (sl >= i0) {
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            pre += (i0 + k < sl) ? v[k] : 0u;
            es = (i0 + k == sl) ? v[k] : es;
          }
        }
      } else {
        Eb[ch] = Sh;
      }
      Sh += cs;
    }
    xs[hf * TILE + r] = Sh;
    bar_group();
    const uint32_t So = xs[(1 - hf) * TILE + r];  // the other half's mass
    const uint32_t Stot = Sh + So;                        // <= 255 * 2^24 < 2^32
    const uint32_t base = hf ? So : 0u;                   // mass before this half
    if constexpr (MODE == 0) {
      if (valid && sl >= 0 && sl < 128) {  // (cum, freq) = (C_sym, C_{sym+1} - C_sym), reading Q21
        const uint32_t E = base + pre;
        const uint32_t c0 = uint32_t(sym) + uint32_t((uint64_t(E) * 65281ull) / Stot);
        const uint32_t c1 = uint32_t(sym) + 1u + uint32_t((uint64_t(E + es) * 65281ull) / Stot);
        cf[row] = c0 | ((c1 - c0) << 16);
      }
    } else {
      // staged row (pcc_internal.cuh DROW_*): S, inv32, mu, E_{16k} at word 2 + k, 0, 0, a
      uint32_t* hd = reinterpret_cast<uint32_t*>(stage + r * DROW_BYTES);
      if (hf == 0) {
        hd[0] = Stot;
        hd[1] = uint32_t((65281ull << 32) / uint64_t(Stot));
        hd[2] = uint32_t(mu);
      }
#pragma unroll
      for (int ch = 0; ch < 8; ++ch)
        if (hf == 1 || ch > 0) hd[2 + 8 * hf + ch] = base + Eb[ch];  // block 8 hf + ch
      bar_group();
      // coalesced copy-out of the group's 128 rows: 128 x 7 16-byte chunks over 256 threads
      const uint32_t rows_here = (n - tile * TILE) < uint32_t(TILE) ? (n - tile * TILE) : uint32_t(TILE);
      constexpr uint32_t RCH16 = DROW_BYTES / 16;
      const uint4* sp = reinterpret_cast<const uint4*>(stage);
      uint4* gp = reinterpret_cast<uint4*>(rows + size_t(tile) * TILE * DROW_BYTES);
      for (uint32_t t = uint32_t(gt); t < rows_here * RCH16; t += GT) gp[t] = sp[t];
    }
    // next tile: hidden layer into A (this tile's MMA has completed) and b2 into TMEM;
    // the staged rows are rewritten only after the next tile's first two group barriers
    if (tile + tstride < ntiles) {
      if (MODE == 1) bar_group();  // the copy-out has read the staged a of this tile
      hidden_and_bias(tile + tstride, fw);
      load_f(tile + 2 * tstride, fw);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(*thold);
}

template <int C, int H, int MODE, bool SAT>
void launch_head2(pcc_ctx c, const int8_t* F, uint32_t n, const DHead& L, const uint32_t* lut, const uint8_t* X,
                  uint32_t* cf, uint16_t* rows, int8_t* a_dbg) {
  auto kern = k_head2_tc<C, H, MODE, SAT>;
  PCC_SMEM_ATTR(kern, Smem2::END);
  const uint32_t ntiles = (n + TILE - 1) / TILE;
  const unsigned grid = std::max(1u, std::min((ntiles + 1) / 2, unsigned(c->sm_count)));
  kern<<<grid, NT2, Smem2::END, c->stream>>>(F, n, L.W1, L.b1, L.rq1, L.W2, L.b2, L.rql, lut, X, cf,
                                            reinterpret_cast<uint8_t*>(rows), a_dbg, L.zsat_lo, L.zsat_hi);
  launched(c);
}

}  // namespace

void head_cdf_tc2(pcc_ctx c, const int8_t* F, uint32_t n, int C, int H, const DHead& L, const uint32_t* lut, int mode,
                  const uint8_t* X, uint32_t* cf, uint16_t* cdf, int8_t* a_dbg) {
  if (n == 0) return;
  Prof p(c, mode == 0 ? "head_enc" : "head_dec", size_t(n) * (C + (mode == 0 ? 1 + 4 : DROW_BYTES)));
#define PCC_HEAD2(CC)                                                                                    \
  if (C == CC && H == CC) {                                                                              \
    if (mode == 0 && L.can_saturate) launch_head2<CC, CC, 0, true>(c, F, n, L, lut, X, cf, cdf, a_dbg);  \
    else if (mode == 0) launch_head2<CC, CC, 0, false>(c, F, n, L, lut, X, cf, cdf, a_dbg);              \
    else if (L.can_saturate) launch_head2<CC, CC, 1, true>(c, F, n, L, lut, X, cf, cdf, a_dbg);          \
    else launch_head2<CC, CC, 1, false>(c, F, n, L, lut, X, cf, cdf, a_dbg);                             \
    return;                                                                                              \
  }
  PCC_HEAD2(8)
  PCC_HEAD2(16)
  PCC_HEAD2(32)
#undef PCC_HEAD2
  throw Error{PCC_ERR_INVALID_ARG};
}

}  // namespace pcc
