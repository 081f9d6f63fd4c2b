// head3_tc.cu — occupancy predictor (Eq.7) + integer softmax to a Q16 pmf
// (Eq.15; readings Q20-Q22), one thread per node, half-width accumulators.
//
// head1_tc.cu keeps a tile's 256 logit columns in TMEM, which caps an SM at 2 tiles
// (512 columns) = 8 warps.  Here a tile group owns only 128 TMEM columns and computes
// the logits in two N = 128 halves, each twice (once for the maximum, once for the
// exponentials): 4 small tcgen05.mma (M = 128, N = 128, K = 32) per tile instead of one,
// with the bias half stored into the columns before each.  NG = 3 or 4 tile groups per
// SM (12 or 16 warps) share the W2 operand and the 32-copy conflict-free exp table.
// Per tile, per half h: bias -> TMEM, group barrier, MMA, wait; pass 1 (max) over both
// halves, then pass 2 (exponentials, block sums, the encoder's prefix mass / the decoder
// row) over both halves again.  Bit-exact with the oracle's head_logits / cdf_quantize.
#include "pcc_internal.cuh"
#include "rq.cuh"
#include "tc.cuh"

namespace pcc {

namespace {

constexpr int TILE = 128;
constexpr uint32_t IDESC = tc::idesc_i8(128, 128);

__device__ __forceinline__ int32_t lq8(int32_t z, const RQ& q) {  // Q8 logit, clamp +-2^24
  int64_t v = int64_t(z) * int64_t(q.mp);
  if (q.r > 0) v = (v + (int64_t(1) << (q.r - 1))) >> q.r;
  v = v < -(int64_t(1) << 24) ? -(int64_t(1) << 24) : (v > (int64_t(1) << 24) ? (int64_t(1) << 24) : v);
  return int32_t(v);
}

__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}

// One CTA per SM: 8 warps = 2 tile groups of 4 warps, each group an independent 128-node
// tile pipeline with its own A operand, 256 TMEM columns (512 per SM), mbarrier and named
// barrier; they share the W2 operand, b2 / W1 / b1 and the exp table.  The table is held
// as 32 interleaved copies of the compact LUT (1025 entries, LUT[1024] = 0): lane l reads
// copy l, word 32 idx + l, so a warp's 32 random lookups hit 32 distinct banks (one
// shared-memory wavefront each).
template <int NG>
struct Smem3 {
  static constexpr int B = 0;                      // W2 operand 256 x 32 (8 KB)
  static constexpr int A = 8192;                   // a operands, one 128 x 32 tile per group
  static constexpr int B2 = A + 4096 * NG;         // b2 [256] (1 KB)
  static constexpr int W1 = B2 + 1024;             // W1 words [H][C/4] (<= 1 KB)
  static constexpr int B1 = W1 + 1024;             // b1 [H] (<= 256 B)
  static constexpr int MBAR = B1 + 256;            // NG mbarriers
  static constexpr int THOLD = MBAR + 8 * NG;
  static constexpr int LUT = MBAR + 128;           // [1025][32] u32
  static constexpr int END = LUT + 1025 * 32 * 4;
};

template <int C, int H, int MODE, bool SAT, int NG>
__global__ void __launch_bounds__(NG * 128, 1) k_head3_tc(const int8_t* __restrict__ F, uint32_t n,
                                                     const int8_t* __restrict__ W1, const int32_t* __restrict__ b1, RQ rq1,
                                                     const int8_t* __restrict__ W2, const int32_t* __restrict__ b2, RQ rql,
                                                     const uint32_t* __restrict__ lut, const uint8_t* __restrict__ X,
                                                     uint32_t* __restrict__ cf, uint8_t* __restrict__ rows,
                                                     int8_t* __restrict__ a_dbg, int32_t zsat_lo, int32_t zsat_hi) {
  extern __shared__ __align__(1024) uint8_t sm[];
  using S = Smem3<NG>;
  constexpr int NT1 = NG * 128;
  constexpr int CW = C / 4, HW = H / 4;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tg = warp >> 2;          // tile group
  const int r = tid & (TILE - 1);    // node of the group's tile = TMEM lane
  uint8_t* sB = sm + S::B;
  uint8_t* sA = sm + S::A + 4096 * tg;
  int32_t* sb2 = reinterpret_cast<int32_t*>(sm + S::B2);
  int32_t* sW1 = reinterpret_cast<int32_t*>(sm + S::W1);
  int32_t* sb1 = reinterpret_cast<int32_t*>(sm + S::B1);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + S::MBAR) + tg;
  uint32_t* thold = reinterpret_cast<uint32_t*>(sm + S::THOLD);

  for (int k = tid; k < 256 * 8; k += NT1) {
    const int rr = k >> 3, w = k & 7;
    const uint32_t v = (w < HW) ? reinterpret_cast<const uint32_t*>(W2)[rr * HW + w] : 0u;
    *reinterpret_cast<uint32_t*>(sB + tc::kmaj_off(rr, 4 * w)) = v;
  }
  for (int k = tid; k < 1024 * NG; k += NT1) reinterpret_cast<uint32_t*>(sm + S::A)[k] = 0u;  // K padding stays 0
  for (int k = tid; k < 1025 * 32; k += NT1) {
    const int idx = k >> 5;  // delta >= 4096 (16 nats): index 1024, e = 0 (reading Q20)
    reinterpret_cast<uint32_t*>(sm + S::LUT)[k] = idx < 1024 ? lut[idx] : 0u;
  }
  for (int k = tid; k < 256; k += NT1) sb2[k] = b2[k];
  for (int k = tid; k < H * CW; k += NT1) sW1[k] = reinterpret_cast<const int32_t*>(W1)[k];
  for (int k = tid; k < H; k += NT1) sb1[k] = b1[k];
  if (warp == 0) tc::tmem_alloc<512>(thold);
  if (tid < NG) tc::mbar_init(reinterpret_cast<uint64_t*>(sm + S::MBAR) + tid, 1);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *thold + 128u * uint32_t(tg);                 // the group's 128 columns
  const uint32_t taddr = tbase + (uint32_t(32 * (warp & 3)) << 16);   // this thread's TMEM lane
  const uint64_t adesc = tc::sdesc(tc::smem_u32(sA));
  // W2 rows 128h .. 128h + 127 of the canonical K-major operand start at byte 4096 h
  const uint64_t bdesc0 = tc::sdesc(tc::smem_u32(sB)), bdesc1 = tc::sdesc(tc::smem_u32(sB + 4096));
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
  // index form (r <= 30, so 4 | Sp): idx = delta >> 2 = floor(X / 2^34) = hi32(z * (-Sp / 4) +
  // mu 2^30 + 2^29 - 1) (z * Sp / 4 is an integer, so the floor of C2 / 4 may replace C2 / 4):
  // the LUT index is the high word of one IMAD.WIDE; the word address is min(idx, 1024) * 128
  // + 4 lane: one min (alu pipe) and one multiply-add (fma pipe) instead of shift, min, and
  auto lut_e_idx = [&](int32_t z, int32_t nM4, int64_t C4) -> uint32_t {
    const uint32_t idx = uint32_t(uint64_t(int64_t(z) * nM4 + C4) >> 32);  // delta >= 0
    uint32_t off, e;
    asm("mad.lo.u32 %0, %1, 128, %2;" : "=r"(off) : "r"(min(idx, 1024u)), "r"(lutu + lane4));
    asm("ld.shared.u32 %0, [%1];" : "=r"(e) : "r"(off));
    return e;
  };
  const uint32_t ntiles = (n + TILE - 1) / TILE;
  const uint32_t tstride = uint32_t(NG) * gridDim.x;
  const int64_t lhalf = rql.r > 0 ? (int64_t(1) << (rql.r - 1)) : 0;
  auto bar_group = [&]() { asm volatile("bar.sync %0, 128;" ::"r"(1 + tg) : "memory"); };
  uint32_t phase = 0;

  // the thread's node row F (C bytes) of tile tl, as C/4 words
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
  // hidden layer of the thread's node into the A operand (and aw), then b2 into its TMEM lane
  auto hidden_and_bias = [&](uint32_t tl, const uint32_t (&fw)[CW], uint32_t (&aw)[HW]) {
    const uint32_t rw = tl * TILE + uint32_t(r);
#pragma unroll
    for (int g4 = 0; g4 < HW; ++g4) {
      int32_t hacc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int h = 4 * g4 + u;
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
      *reinterpret_cast<uint32_t*>(sA + tc::kmaj_off(uint32_t(r), 4 * g4)) = aw[g4];
    }
    if (a_dbg && rw < n) {
#pragma unroll
      for (int g4 = 0; g4 < HW; ++g4) reinterpret_cast<uint32_t*>(a_dbg + size_t(rw) * H)[g4] = aw[g4];
    }
  };
  // b2 of half h into the thread's 128 TMEM columns (the MMA accumulates onto it)
  auto bias_half = [&](int h) {
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) {
      uint32_t bv[16];
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        const uint4 b4 = *reinterpret_cast<const uint4*>(sb2 + 128 * h + 16 * ch + 4 * k4);
        bv[4 * k4] = b4.x, bv[4 * k4 + 1] = b4.y, bv[4 * k4 + 2] = b4.z, bv[4 * k4 + 3] = b4.w;
      }
      st16(taddr + ch * 16, bv);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  };
  // half h of z = b2 + a W2^T into the group's columns: all of the group's TMEM reads of
  // the previous half and its A operand / bias stores precede the MMA (fence + barrier)
  auto mma_half = [&](int h) {
    bias_half(h);
    tc::fence_async_smem();
    tc::fence_before();
    bar_group();
    tc::fence_after();
    if (r == 0) {
      tc::mma_i8(tbase, adesc, h ? bdesc1 : bdesc0, IDESC, 1u);
      tc::commit(mbar);
    }
    tc::mbar_wait(mbar, phase);
    phase ^= 1u;
    tc::fence_after();
  };

  uint32_t fw[CW], aw[HW];
  const uint32_t t0 = uint32_t(NG) * blockIdx.x + uint32_t(tg);
  load_f(t0, fw);
  if (t0 < ntiles) hidden_and_bias(t0, fw, aw);
  load_f(t0 + tstride, fw);
  for (uint32_t tile = t0; tile < ntiles; tile += tstride) {
    const uint32_t row = tile * TILE + uint32_t(r);
    const bool valid = row < n;
    // ---- pass 1: max z (and min z) over the 255 symbols (column 255 is padding) ----
    int32_t zmx = INT32_MIN, zmn = INT32_MAX;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      mma_half(h);
#pragma unroll 1
      for (int ch = 0; ch < 4; ++ch) {
        uint32_t v[32];
        tc::tmem_ld32(taddr + ch * 32, v);
        tc::tmem_wait_ld();
        if (h == 1 && ch == 3) v[31] = v[30];  // column 255 is padding, not a symbol
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          zmx = max(zmx, int32_t(v[k]));
          if (SAT) zmn = min(zmn, int32_t(v[k]));
        }
      }
    }
    const int32_t mu = lq8(zmx, rql);
    const bool nosat = !SAT || (zmx <= zsat_hi && zmn >= zsat_lo);
    const bool fastl = rql.fast_s && nosat;
    const bool fasti = fastl && rql.r <= 30;
    const int32_t nM = -rql.Sp;
    const int64_t C2 = (int64_t(mu) << 32) + 0x7fffffff;
    const int32_t nM4 = -(rql.Sp >> 2);
    const int64_t C4 = (int64_t(mu) << 30) + ((int64_t(1) << 29) - 1);
    const int sym = (MODE == 0 && valid) ? int(X[row]) - 1 : 0;

    // ---- pass 2: e_i = LUT[(mu - l_i) >> 2], 16-symbol block sums, the encoder's prefix mass ----
    uint32_t Sacc = 0, pre = 0, es = 0;
    uint32_t Eb[16];  // decoder: prefix mass before each 16-symbol block
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      mma_half(h);
#pragma unroll 1
      for (int ch4 = 0; ch4 < 4; ++ch4) {
        const int ch = 4 * h + ch4;
        uint32_t v[32];
        tc::tmem_ld32(taddr + ch4 * 32, v);
        tc::tmem_wait_ld();
        if (fasti) {
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] = lut_e_idx(int32_t(v[k]), nM4, C4);
        } else if (fastl) {
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] = lut_e_fast(int32_t(v[k]), nM, C2);
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const int32_t zz = int32_t(v[k]);
            int32_t lv = int32_t((int64_t(zz) * int64_t(rql.mp) + lhalf) >> rql.r);
            if (SAT && !nosat) {
              lv = zz > zsat_hi ? (1 << 24) : lv;
              lv = zz < zsat_lo ? -(1 << 24) : lv;
            }
            v[k] = lut_e(uint32_t(mu - lv));
          }
        }
        if (ch == 7) v[31] = 0u;  // column 255 is padding, not a symbol
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          uint32_t cs = 0;
#pragma unroll
          for (int k = 0; k < 16; ++k) cs += v[16 * hf + k];
          if constexpr (MODE == 0) {
            const int i0 = 32 * ch + 16 * hf;
            if (sym >= i0 + 16) {
              pre += cs;
            } else if (sym >= i0) {
#pragma unroll
              for (int k = 0; k < 16; ++k) {
                pre += (i0 + k < sym) ? v[16 * hf + k] : 0u;
                es = (i0 + k == sym) ? v[16 * hf + k] : es;
              }
            }
          } else {
            Eb[2 * ch + hf] = Sacc;
          }
          Sacc += cs;  // <= 255 * 2^24 < 2^32
        }
      }
    }
    const uint32_t Ssum = Sacc;
    // all of this thread's TMEM reads are done: the next tile may be set up
    if constexpr (MODE == 0) {
      if (valid) {  // (cum, freq) = (C_sym, C_{sym+1} - C_sym), reading Q21
        const uint32_t c0 = uint32_t(sym) + uint32_t((uint64_t(pre) * 65281ull) / Ssum);
        const uint32_t c1 = uint32_t(sym) + 1u + uint32_t((uint64_t(pre + es) * 65281ull) / Ssum);
        cf[row] = c0 | ((c1 - c0) << 16);
      }
    } else if (valid) {
      // decoder row (pcc_internal.cuh DROW_*): S, inv32, mu, E_{16k} k = 1..15, 0, 0, a
      uint4* dst = reinterpret_cast<uint4*>(rows + size_t(row) * DROW_BYTES);
      const uint32_t inv32 = uint32_t((65281ull << 32) / uint64_t(Ssum));
      dst[0] = make_uint4(Ssum, inv32, uint32_t(mu), Eb[1]);
      dst[1] = make_uint4(Eb[2], Eb[3], Eb[4], Eb[5]);
      dst[2] = make_uint4(Eb[6], Eb[7], Eb[8], Eb[9]);
      dst[3] = make_uint4(Eb[10], Eb[11], Eb[12], Eb[13]);
      dst[4] = make_uint4(Eb[14], Eb[15], 0u, 0u);
      uint32_t ap[8];
#pragma unroll
      for (int w = 0; w < 8; ++w) ap[w] = w < HW ? aw[w < HW ? w : 0] : 0u;
      dst[5] = make_uint4(ap[0], ap[1], ap[2], ap[3]);
      dst[6] = make_uint4(ap[4], ap[5], ap[6], ap[7]);
    }
    // next tile: hidden layer into A (this tile's last MMA has completed)
    if (tile + tstride < ntiles) {
      hidden_and_bias(tile + tstride, fw, aw);
      load_f(tile + 2 * tstride, fw);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(*thold);
}

template <int C, int H, int MODE, bool SAT, int NG>
void launch_head3(pcc_ctx c, const int8_t* F, uint32_t n, const DHead& L, const uint32_t* lut, const uint8_t* X,
                  uint32_t* cf, uint16_t* rows, int8_t* a_dbg) {
  auto kern = k_head3_tc<C, H, MODE, SAT, NG>;
  PCC_SMEM_ATTR(kern, Smem3<NG>::END);
  const uint32_t ntiles = (n + TILE - 1) / TILE;
  const unsigned grid = std::max(1u, std::min((ntiles + NG - 1) / NG, unsigned(c->sm_count)));
  kern<<<grid, NG * 128, Smem3<NG>::END, c->stream>>>(F, n, L.W1, L.b1, L.rq1, L.W2, L.b2, L.rql, lut, X, cf,
                                                    reinterpret_cast<uint8_t*>(rows), a_dbg, L.zsat_lo, L.zsat_hi);
  launched(c);
}

}  // namespace

void head_cdf_tc3(pcc_ctx c, const int8_t* F, uint32_t n, int C, int H, const DHead& L, const uint32_t* lut, int mode,
                  const uint8_t* X, uint32_t* cf, uint16_t* cdf, int8_t* a_dbg, int ng) {
  if (n == 0) return;
  Prof p(c, mode == 0 ? "head_enc" : "head_dec", size_t(n) * (C + (mode == 0 ? 1 + 4 : DROW_BYTES)));
#define PCC_HEAD3(CC, NGG)                                                                                  \
  if (C == CC && H == CC && ng == NGG) {                                                                     \
    if (mode == 0 && L.can_saturate) launch_head3<CC, CC, 0, true, NGG>(c, F, n, L, lut, X, cf, cdf, a_dbg);  \
    else if (mode == 0) launch_head3<CC, CC, 0, false, NGG>(c, F, n, L, lut, X, cf, cdf, a_dbg);              \
    else if (L.can_saturate) launch_head3<CC, CC, 1, true, NGG>(c, F, n, L, lut, X, cf, cdf, a_dbg);          \
    else launch_head3<CC, CC, 1, false, NGG>(c, F, n, L, lut, X, cf, cdf, a_dbg);                             \
    return;                                                                                                  \
  }
  PCC_HEAD3(8, 3)
  PCC_HEAD3(16, 3)
  PCC_HEAD3(32, 3)
  PCC_HEAD3(8, 4)
  PCC_HEAD3(16, 4)
  PCC_HEAD3(32, 4)
#undef PCC_HEAD3
  throw Error{PCC_ERR_INVALID_ARG};
}

}  // namespace pcc
