// head4_tc.cu — occupancy predictor (Eq.7) + integer softmax to a Q16 pmf
// (Eq.15; readings Q20-Q22), one thread per node, both layers on tcgen05.
//
// head3_tc.cu computes the hidden layer a = prq(W1 F + b1) with 256 dp4a per node and
// seeds each logit half with b2 by TMEM stores before every MMA.  Here:
//  * the hidden layer is one more tcgen05.mma (M = 128, N = 32, K = 32) from the tile's
//    feature rows staged in shared memory, read back with one tcgen05.ld;
//  * both biases ride inside the MMAs as a second K = 32 slab: A = a constant row
//    [127 x 31, 1], B = the bias written as 31 base-127 digits plus a remainder
//    (b = 127 sum_j d_j + r, |d_j| <= 127, 0 <= r < 127), so acc = a.W^T + b exactly in
//    int32 (Eq.13's integer accumulation; any split of the sum gives the same integer,
//    reading O6).  Exact whenever |b| <= 500000 (checked at model load, DHead::bias_fold;
//    otherwise head3 runs);
//  * the logits are computed in N = 128 halves: h0 then h1 for the maximum, then h1 (still
//    in TMEM) and h0 again for the exponentials: 3 logit MMAs per tile instead of 4;
//  * the encoder's two normalisation divisions use a float estimate plus one exact fix.
// Bit-exact with the oracle's head_logits / cdf_quantize.
#include "pcc_internal.cuh"
#include "rq.cuh"
#include "tc.cuh"

namespace pcc {

namespace {

constexpr int TILE = 128;
constexpr uint32_t IDESC_Z = tc::idesc_i8(128, 128);
constexpr uint32_t IDESC_H = tc::idesc_i8(128, 32);

__device__ __forceinline__ int32_t lq8(int32_t z, const RQ& q) {  // Q8 logit, clamp +-2^24
  int64_t v = int64_t(z) * int64_t(q.mp);
  if (q.r > 0) v = (v + (int64_t(1) << (q.r - 1))) >> q.r;
  v = v < -(int64_t(1) << 24) ? -(int64_t(1) << 24) : (v > (int64_t(1) << 24) ? (int64_t(1) << 24) : v);
  return int32_t(v);
}

// floor(E * 65281 / S) for E <= S (E, S < 2^32): a float estimate (relative error < 2^-21,
// so it is q - 1, q or q + 1) and one exact 64-bit remainder test each way
__device__ __forceinline__ uint32_t qdiv(uint32_t E, uint32_t S, float rS) {
  uint32_t q = uint32_t(__fmul_rz(float(E), rS));
  const int64_t rem = int64_t(uint64_t(E) * 65281ull) - int64_t(uint64_t(q) * uint64_t(S));
  q = rem < 0 ? q - 1u : (rem >= int64_t(S) ? q + 1u : q);
  return q;
}

template <int NG>
struct Smem4 {
  static constexpr int W2 = 0;                 // B operand, logits: W2 256 x 32 (8 KB)
  static constexpr int B2D = 8192;             // B operand, logit bias digits 256 x 32 (8 KB)
  static constexpr int W1 = 16384;             // B operand, hidden: W1 32 x 32 (1 KB)
  static constexpr int B1D = 17408;            // B operand, hidden bias digits 32 x 32 (1 KB)
  static constexpr int KC = 18432;             // A operand, the constant rows [127 x 31, 1] (4 KB)
  static constexpr int A = 22528;              // per group: hidden activations 128 x 32 (4 KB)
  static constexpr int F = A + 4096 * NG;      // per group: feature rows 128 x 32 (4 KB)
  static constexpr int MBAR = F + 4096 * NG;   // NG mbarriers
  static constexpr int THOLD = MBAR + 8 * NG;
  static constexpr int LUT = MBAR + 128;       // [1025][32] u32, 32 interleaved copies
  static constexpr int CS = LUT + 1025 * 32 * 4;  // [16][NG * 128] u32: decoder block sums / encoder's symbol block
  static constexpr int END = CS + 16 * NG * 128 * 4;
};

template <int C, int H, int MODE, bool SAT, int NG>
__global__ void __launch_bounds__(NG * 128, 1) k_head4_tc(const int8_t* __restrict__ F, uint32_t n,
                                                     const int8_t* __restrict__ W1, RQ rq1,
                                                     const int8_t* __restrict__ W2, RQ rql,
                                                     const int8_t* __restrict__ B1d, const int8_t* __restrict__ B2d,
                                                     const uint32_t* __restrict__ lut, const uint8_t* __restrict__ X,
                                                     uint32_t* __restrict__ cf, uint8_t* __restrict__ rows,
                                                     int8_t* __restrict__ a_dbg, int32_t zsat_lo, int32_t zsat_hi) {
  extern __shared__ __align__(1024) uint8_t sm[];
  using S = Smem4<NG>;
  constexpr int NT1 = NG * 128;
  constexpr int CW = C / 4, HW = H / 4;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tg = warp >> 2;          // tile group
  const int r = tid & (TILE - 1);    // node of the group's tile = TMEM lane
  uint8_t* sA = sm + S::A + 4096 * tg;
  uint8_t* sF = sm + S::F + 4096 * tg;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + S::MBAR) + tg;
  uint32_t* thold = reinterpret_cast<uint32_t*>(sm + S::THOLD);

  // operands: row rr of a B matrix is 32 K-bytes; words beyond the layer's width are 0
  for (int k = tid; k < 256 * 8; k += NT1) {
    const int rr = k >> 3, w = k & 7;
    const uint32_t v = (w < HW) ? reinterpret_cast<const uint32_t*>(W2)[rr * HW + w] : 0u;
    *reinterpret_cast<uint32_t*>(sm + S::W2 + tc::kmaj_off(rr, 4 * w)) = v;
    *reinterpret_cast<uint32_t*>(sm + S::B2D + tc::kmaj_off(rr, 4 * w)) = reinterpret_cast<const uint32_t*>(B2d)[k];
  }
  for (int k = tid; k < 32 * 8; k += NT1) {
    const int rr = k >> 3, w = k & 7;
    const uint32_t v = (rr < H && w < CW) ? reinterpret_cast<const uint32_t*>(W1)[rr * CW + w] : 0u;
    *reinterpret_cast<uint32_t*>(sm + S::W1 + tc::kmaj_off(rr, 4 * w)) = v;
    *reinterpret_cast<uint32_t*>(sm + S::B1D + tc::kmaj_off(rr, 4 * w)) = reinterpret_cast<const uint32_t*>(B1d)[k];
  }
  for (int k = tid; k < 128 * 8; k += NT1) {  // [127 x 31, 1]
    const int rr = k >> 3, w = k & 7;
    *reinterpret_cast<uint32_t*>(sm + S::KC + tc::kmaj_off(rr, 4 * w)) = w < 7 ? 0x7f7f7f7fu : 0x017f7f7fu;
  }
  for (int k = tid; k < 2048 * NG; k += NT1) reinterpret_cast<uint32_t*>(sm + S::A)[k] = 0u;  // A and F, K padding 0
  for (int k = tid; k < 1025 * 32; k += NT1) {
    const int idx = k >> 5;  // delta >= 4096 (16 nats): index 1024, e = 0 (reading Q20)
    reinterpret_cast<uint32_t*>(sm + S::LUT)[k] = idx < 1024 ? lut[idx] : 0u;
  }
  if (warp == 0) tc::tmem_alloc<512>(thold);
  if (tid < NG) tc::mbar_init(reinterpret_cast<uint64_t*>(sm + S::MBAR) + tid, 1);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *thold + 128u * uint32_t(tg);                 // the group's 128 columns
  const uint32_t taddr = tbase + (uint32_t(32 * (warp & 3)) << 16);   // this thread's TMEM lane
  const uint64_t adesc = tc::sdesc(tc::smem_u32(sA)), fdesc = tc::sdesc(tc::smem_u32(sF));
  const uint64_t kdesc = tc::sdesc(tc::smem_u32(sm + S::KC));
  const uint64_t w1desc = tc::sdesc(tc::smem_u32(sm + S::W1)), b1desc = tc::sdesc(tc::smem_u32(sm + S::B1D));
  // rows 128h .. 128h + 127 of a canonical K-major 256-row operand start at byte 4096 h
  const uint64_t w2d0 = tc::sdesc(tc::smem_u32(sm + S::W2)), w2d1 = tc::sdesc(tc::smem_u32(sm + S::W2 + 4096));
  const uint64_t b2d0 = tc::sdesc(tc::smem_u32(sm + S::B2D)), b2d1 = tc::sdesc(tc::smem_u32(sm + S::B2D + 4096));
  const uint8_t* lutb = sm + S::LUT;
  const uint32_t lane4 = 4u * uint32_t(lane);
  const uint32_t lutu = tc::smem_u32(lutb);
  // generic form: word 32 idx + lane of the 32-copy table
  auto lut_e = [&](uint32_t dl) -> uint32_t {
    const uint32_t off = (min(dl << 5, 4096u << 5) & ~127u) | lane4;  // dl < 2^26: no overflow
    return *reinterpret_cast<const uint32_t*>(lutb + off);
  };
  // signed one-multiply form (RQ::fast_s): X = z (-Sp) + mu 2^32 + 2^31 - 1, delta = X >> 32
  auto lut_e_fast = [&](int32_t z, int32_t nM, int64_t C2) -> uint32_t {
    const uint32_t y = uint32_t(uint64_t(int64_t(z) * nM + C2) >> 27);
    const uint32_t off = (min(y, 4096u << 5) & ~127u) | lane4;
    uint32_t e;
    asm("ld.shared.u32 %0, [%1];" : "=r"(e) : "r"(lutu + off));
    return e;
  };
  // index form (fast_s and r <= 30, so 4 | Sp): delta >> 2 = hi32(z (-Sp / 4) + mu 2^30 + 2^29 - 1)
  // (head3_tc.cu): one IMAD.HI, one min, one IMAD per symbol
  auto lut_e_idx = [&](int32_t z, int32_t nM4, int64_t C4) -> uint32_t {
    const uint32_t idx = uint32_t(uint64_t(int64_t(z) * nM4 + C4) >> 32);
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
  // all of the group's smem operand stores and TMEM reads precede the MMA (fence + barrier);
  // one thread issues acc = A0 W0^T + A1 W1^T into the group's columns and waits
  auto mma2 = [&](uint64_t a0, uint64_t b0, uint64_t a1, uint64_t b1, uint32_t idesc) {
    tc::fence_async_smem();
    tc::fence_before();
    bar_group();
    tc::fence_after();
    if (r == 0) {
      tc::mma_i8(tbase, a0, b0, idesc, 0u);
      tc::mma_i8(tbase, a1, b1, idesc, 1u);
      tc::commit(mbar);
    }
    tc::mbar_wait(mbar, phase);
    phase ^= 1u;
    tc::fence_after();
  };

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
  // a row of W words into the canonical K-major operand (16-byte stores where possible)
  auto store_row = [&](uint8_t* op, const uint32_t* wv, int W) {
    if (W >= 4) {
#pragma unroll
      for (int w = 0; w < W; w += 4)
        *reinterpret_cast<uint4*>(op + tc::kmaj_off(uint32_t(r), 4 * w)) = make_uint4(wv[w], wv[w + 1], wv[w + 2], wv[w + 3]);
    } else {
#pragma unroll
      for (int w = 0; w < W; ++w) *reinterpret_cast<uint32_t*>(op + tc::kmaj_off(uint32_t(r), 4 * w)) = wv[w];
    }
  };

  uint32_t fw[CW], aw[HW];
  const uint32_t t0 = uint32_t(NG) * blockIdx.x + uint32_t(tg);
  load_f(t0, fw);
  store_row(sF, fw, CW);
  for (uint32_t tile = t0; tile < ntiles; tile += tstride) {
    const uint32_t row = tile * TILE + uint32_t(r);
    const bool valid = row < n;
    // ---- hidden layer: a = prq(F W1^T + b1) (Eq.7), TMEM -> registers -> A operand ----
    mma2(fdesc, w1desc, kdesc, b1desc, IDESC_H);
    {
      uint32_t hv[32];
      tc::tmem_ld32(taddr, hv);
      tc::tmem_wait_ld();
#pragma unroll
      for (int g4 = 0; g4 < HW; ++g4) {
        const int32_t h0 = int32_t(hv[4 * g4]), h1 = int32_t(hv[4 * g4 + 1]), h2 = int32_t(hv[4 * g4 + 2]),
                      h3 = int32_t(hv[4 * g4 + 3]);
        if (rq1.fast_s)
          aw[g4] = pack_sat4(rq_s(h0, rq1), rq_s(h1, rq1), rq_s(h2, rq1), rq_s(h3, rq1));
        else
          aw[g4] = (uint32_t(rq8(h0, rq1)) & 0xffu) | (uint32_t(rq8(h1, rq1)) & 0xffu) << 8 |
                   (uint32_t(rq8(h2, rq1)) & 0xffu) << 16 | (uint32_t(rq8(h3, rq1)) & 0xffu) << 24;
      }
    }
    store_row(sA, aw, HW);
    if (a_dbg && valid) {
#pragma unroll
      for (int g4 = 0; g4 < HW; ++g4) reinterpret_cast<uint32_t*>(a_dbg + size_t(row) * H)[g4] = aw[g4];
    }
    load_f(tile + tstride, fw);  // next tile's rows, stored into sF after this tile's passes

    // ---- pass 1: max z (and min z) over the 255 symbols (column 255 is padding) ----
    int32_t zmx = INT32_MIN, zmn = INT32_MAX;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      mma2(adesc, h ? w2d1 : w2d0, kdesc, h ? b2d1 : b2d0, IDESC_Z);
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

    // ---- pass 2: e_i = LUT[(mu - l_i) >> 2], 16-symbol block sums, the encoder's prefix mass.
    // Half 1 first (its logits are still in TMEM), then half 0 again.
    uint32_t Sacc = 0, pre = 0, es = 0;
    uint32_t* scs = reinterpret_cast<uint32_t*>(sm + S::CS) + tid;  // word k of this thread at scs[k * NT1]
#pragma unroll 1
    for (int hh = 0; hh < 2; ++hh) {
      const int h = 1 - hh;
      if (hh == 1) mma2(adesc, w2d0, kdesc, b2d0, IDESC_Z);
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
          uint32_t s16 = 0;
#pragma unroll
          for (int k = 0; k < 16; ++k) s16 += v[16 * hf + k];
          if constexpr (MODE == 0) {
            // whole blocks below the symbol add to its prefix mass; the symbol's own block
            // is parked in shared memory and finished after the pass (16 stores instead of
            // a 16-step compare-select chain under a divergent branch)
            const int i0 = 32 * ch + 16 * hf;
            pre += sym >= i0 + 16 ? s16 : 0u;
            if (sym >= i0 && sym < i0 + 16) {
#pragma unroll
              for (int k = 0; k < 16; ++k) scs[k * NT1] = v[16 * hf + k];
            }
          } else {
            scs[(2 * ch + hf) * NT1] = s16;
          }
          Sacc += s16;  // <= 255 * 2^24 < 2^32
        }
      }
    }
    const uint32_t Ssum = Sacc;
    if constexpr (MODE == 0) {
      {  // the symbol's block: prefix within it and the symbol's own e
        const int m = sym & 15;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const uint32_t e = scs[k * NT1];
          pre += k < m ? e : 0u;
          es = k == m ? e : es;
        }
      }
      if (valid) {  // (cum, freq) = (C_sym, C_{sym+1} - C_sym), reading Q21
        const float rS = 65281.0f / float(Ssum);
        const uint32_t c0 = uint32_t(sym) + qdiv(pre, Ssum, rS);
        const uint32_t c1 = uint32_t(sym) + 1u + qdiv(pre + es, Ssum, rS);
        cf[row] = c0 | ((c1 - c0) << 16);
      }
    } else if (valid) {
      // decoder row (pcc_internal.cuh DROW_*): S, inv32, mu, E_{16k} k = 1..15, 0, 0, a
      uint32_t Eb[16];
      Eb[0] = 0u;
#pragma unroll
      for (int k = 1; k < 16; ++k) Eb[k] = Eb[k - 1] + scs[(k - 1) * NT1];
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
    // next tile's feature rows (this tile's hidden MMA, the last reader of sF, completed)
    if (tile + tstride < ntiles) store_row(sF, fw, CW);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(*thold);
}

template <int C, int H, int MODE, bool SAT, int NG>
void launch_head4(pcc_ctx c, const int8_t* F, uint32_t n, const DHead& L, const uint32_t* lut, const uint8_t* X,
                  uint32_t* cf, uint16_t* rows, int8_t* a_dbg) {
  auto kern = k_head4_tc<C, H, MODE, SAT, NG>;
  PCC_SMEM_ATTR(kern, Smem4<NG>::END);
  const uint32_t ntiles = (n + TILE - 1) / TILE;
  const unsigned grid = std::max(1u, std::min((ntiles + NG - 1) / NG, unsigned(c->sm_count)));
  kern<<<grid, NG * 128, Smem4<NG>::END, c->stream>>>(F, n, L.W1, L.rq1, L.W2, L.rql, L.B1d, L.B2d, lut, X, cf,
                                                    reinterpret_cast<uint8_t*>(rows), a_dbg, L.zsat_lo, L.zsat_hi);
  launched(c);
}

}  // namespace

void head_cdf_tc4(pcc_ctx c, const int8_t* F, uint32_t n, int C, int H, const DHead& L, const uint32_t* lut, int mode,
                  const uint8_t* X, uint32_t* cf, uint16_t* cdf, int8_t* a_dbg) {
  if (n == 0) return;
  if (!L.bias_fold) throw Error{PCC_ERR_INVALID_ARG};
  Prof p(c, mode == 0 ? "head_enc" : "head_dec", size_t(n) * (C + (mode == 0 ? 1 + 4 : DROW_BYTES)));
#define PCC_HEAD4(CC)                                                                                   \
  if (C == CC && H == CC) {                                                                              \
    if (mode == 0 && L.can_saturate) launch_head4<CC, CC, 0, true, 4>(c, F, n, L, lut, X, cf, cdf, a_dbg);  \
    else if (mode == 0) launch_head4<CC, CC, 0, false, 4>(c, F, n, L, lut, X, cf, cdf, a_dbg);              \
    else if (L.can_saturate) launch_head4<CC, CC, 1, true, 4>(c, F, n, L, lut, X, cf, cdf, a_dbg);          \
    else launch_head4<CC, CC, 1, false, 4>(c, F, n, L, lut, X, cf, cdf, a_dbg);                             \
    return;                                                                                              \
  }
  PCC_HEAD4(8)
  PCC_HEAD4(16)
  PCC_HEAD4(32)
#undef PCC_HEAD4
  throw Error{PCC_ERR_INVALID_ARG};
}

}  // namespace pcc
