// head_tc.cu — occupancy predictor (Eq.7) + integer softmax to a Q16 pmf
// (Eq.15; readings Q20-Q22) on the 5th-generation tensor cores.
//
// One CTA = 512 threads = one 128-node tile per iteration (persistent over tiles).
//   1. hidden layer a = prq(W1 F + b1) (C -> H, int8 dp4a) written straight into the
//      tcgen05 A operand (canonical K-major smem tile, K padded to 32 with zeros);
//   2. z = a W2^T: ONE tcgen05.mma.kind::i8 (M = 128, N = 256, K = 32) into TMEM
//      (int32; column 255 is padding);
//   3. four threads own TMEM lane r = node r of the tile (one 64-column quarter each)
//      and run the softmax over the row with 16-column tcgen05.ld loads: pass 1 finds
//      max z (the logit requant is monotone), pass 2 turns the logits into LUT
//      exponentials and the quarter sums of e; the normalisation is reading Q21's
//      cumulative floors C_i = i + floor(E_i * 65281 / S) (E_i = prefix sum of e):
//      the encoder needs only C_sym and C_{sym+1} (prefix mass before the true symbol
//      from pass 2, two exact divisions per node); the decoder writes a 112-byte row per
//      node (pcc_internal.cuh DROW_*: S, 65281 * 2^32 / S, the maximum logit mu, the 15
//      block prefix masses E_{16k} and the hidden activations a), staged in smem and
//      copied out whole: the rANS decoder recomputes the 16 logits of the block it needs.
// Bit-exact with the oracle's cdf_quantize / head_logits (integer arithmetic only).
#include "pcc_internal.cuh"
#include "rq.cuh"
#include "tc.cuh"

namespace pcc {

namespace {

#ifdef PCC_TRACE
// development-only phase timer (tools/micro/trace_head.py): cycles per phase, summed over
// the CTAs' thread 0 (row 0, quarter 0) and thread 480 (row 96, quarter 3)
__device__ unsigned long long g_head_trace[2][8];
#define HEAD_TRACE(slot, t0)                                                          \
  do {                                                                                \
    if ((threadIdx.x & 0x1df) == 0) {                                                 \
      const long long t1_ = clock64();                                                \
      atomicAdd(&g_head_trace[MODE][slot], (unsigned long long)(t1_ - (t0)));         \
      (t0) = t1_;                                                                     \
    }                                                                                 \
  } while (0)
#else
#define HEAD_TRACE(slot, t0) \
  do {                       \
  } while (0)
#endif

constexpr int TILE = 128;
constexpr uint32_t IDESC = tc::idesc_i8(128, 256);

__device__ __forceinline__ int32_t lq8(int32_t z, RQ q) {  // Q8 logit, clamp +-2^24
  int64_t v = int64_t(z) * int64_t(q.mp);
  if (q.r > 0) v = (v + (int64_t(1) << (q.r - 1))) >> q.r;
  v = v < -(int64_t(1) << 24) ? -(int64_t(1) << 24) : (v > (int64_t(1) << 24) ? (int64_t(1) << 24) : v);
  return int32_t(v);
}

__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}

// 512 threads per CTA: 16 warps.  Warp w may only touch TMEM lanes 32*(w%4)..+31, so
// thread t owns row r = 32*(w%4) + t%32 of the tile and column quarter q = w/4
// (columns 64q..64q+63); the 4 threads of a row combine max / sum / totals in smem.
constexpr int NT = 512;
template <int MODE>
struct SmemLayout {
  static constexpr int B = 0;           // W2 operand 256 x 32 (8 KB)
  static constexpr int A = 8192;        // a operand 128 x 32 (4 KB)
  // exp table indexed by delta itself, LUT4[j] = LUT[j >> 2] for j < 4096, LUT4[4096] = 0
  static constexpr int LUT = 12288;
  static constexpr int LUT_N = 4097;
  static constexpr int B2 = LUT + ((LUT_N * 4 + 15) & ~15);  // 1 KB
  static constexpr int W1 = B2 + 1024;           // <= 1 KB
  static constexpr int B1 = W1 + 1024;           // <= 256 B
  static constexpr int MBAR = B1 + 256;
  static constexpr int THOLD = MBAR + 8;
  static constexpr int RED = MBAR + 16;          // [4][128] x (a, b) int32 = 4 KB
  static constexpr int ROWI = RED + 4096;        // [128] x 8 int32 = 4 KB
  static constexpr int STAGE = ROWI + 4096;      // decoder: 128 rows x DROW_BYTES (14 KB)
  static constexpr int FST = STAGE + (MODE == 1 ? TILE * DROW_BYTES : 0);  // the tile's F rows (cp.async, <= 8 KB)
  static constexpr int END = FST + TILE * 64;
};

// SAT = false when the model proves |z| can never reach the logit saturation thresholds
// (checked at load from |b2| + 128 * sum|W2|): no min tracking, no saturation selects.
template <int C, int H, int MODE, bool SAT>
__global__ void __launch_bounds__(NT, 2) k_head_tc(const int8_t* __restrict__ F, uint32_t n,
                                                   const int8_t* __restrict__ W1, const int32_t* __restrict__ b1, RQ rq1,
                                                   const int8_t* __restrict__ W2, const int32_t* __restrict__ b2, RQ rql,
                                                   const uint32_t* __restrict__ lut, const uint8_t* __restrict__ X,
                                                   uint32_t* __restrict__ cf, uint16_t* __restrict__ cdf,
                                                   int8_t* __restrict__ a_dbg, int32_t zsat_lo, int32_t zsat_hi) {
  extern __shared__ __align__(1024) uint8_t sm[];
  using S = SmemLayout<MODE>;
  const int64_t lhalf = rql.r > 0 ? (int64_t(1) << (rql.r - 1)) : 0;
  uint8_t* sB = sm + S::B;
  uint8_t* sA = sm + S::A;
  uint32_t* sLut = reinterpret_cast<uint32_t*>(sm + S::LUT);
  int32_t* sb2 = reinterpret_cast<int32_t*>(sm + S::B2);
  int32_t* sW1 = reinterpret_cast<int32_t*>(sm + S::W1);
  int32_t* sb1 = reinterpret_cast<int32_t*>(sm + S::B1);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + S::MBAR);
  uint32_t* thold = reinterpret_cast<uint32_t*>(sm + S::THOLD);
  int32_t* red = reinterpret_cast<int32_t*>(sm + S::RED);    // red[(q*128 + r)*2 + {0,1}]
  int32_t* rowi = reinterpret_cast<int32_t*>(sm + S::ROWI);  // rowi[r*8 + k]
  const int tid = threadIdx.x, warp = tid >> 5;
  const int r = 32 * (warp & 3) + (tid & 31);  // row of the tile (= TMEM lane)
  const int q = warp >> 2;                     // column quarter
  // the 4 threads of a row are the 4 warps with the same warp % 4: row exchanges (red,
  // rowi, the staged cdf rows) synchronise only those 128 threads (named barrier 1 + w%4)
  auto bar_rows = [&]() { asm volatile("bar.sync %0, 128;" ::"r"(1 + (warp & 3)) : "memory"); };
  constexpr int CW = C / 4, HW = H / 4, HQ = H / 4;  // HQ hidden units per thread

  for (int k = tid; k < 256 * 8; k += NT) {
    const int rr = k >> 3, w = k & 7;
    const uint32_t v = (w < HW) ? reinterpret_cast<const uint32_t*>(W2)[rr * HW + w] : 0u;
    *reinterpret_cast<uint32_t*>(sB + tc::kmaj_off(rr, 4 * w)) = v;
  }
  for (int k = tid; k < 1024; k += NT) reinterpret_cast<uint32_t*>(sA)[k] = 0u;  // K padding stays 0
  for (int k = tid; k < 4096; k += NT) sLut[k] = lut[k >> 2];
  if (tid == 0) sLut[4096] = 0u;  // delta >= 4096 (16 nats): e = 0 (reading Q20)
  if constexpr (MODE == 1)  // row padding stays 0
    for (int k = tid; k < TILE * DROW_BYTES / 4; k += NT) reinterpret_cast<uint32_t*>(sm + S::STAGE)[k] = 0u;
  for (int k = tid; k < 256; k += NT) sb2[k] = b2[k];
  for (int k = tid; k < H * CW; k += NT) sW1[k] = reinterpret_cast<const int32_t*>(W1)[k];
  for (int k = tid; k < H; k += NT) sb1[k] = b1[k];
  if (warp == 0) tc::tmem_alloc<256>(thold);
  if (tid == 0) tc::mbar_init(mbar, 1);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *thold;
  const uint32_t taddr = tbase + (uint32_t(32 * (warp & 3)) << 16) + uint32_t(64 * q);
  const uint64_t adesc = tc::sdesc(tc::smem_u32(sA));
  const uint64_t bdesc = tc::sdesc(tc::smem_u32(sB));
  const uint32_t ntiles = (n + TILE - 1) / TILE;
  uint32_t phase = 0;

  // The next tile's feature rows are copied (cp.async) into smem while this tile runs;
  // row r's chunks are copied by the row's own quarter threads q < RCH, so a row barrier
  // makes them visible to the row's 4 threads.
  constexpr int CB = C < 16 ? C : 16, RCH = C / CB;  // copy chunk, chunks per row
  auto prefetch_f = [&](uint32_t tl) {
    const uint32_t rw = tl * TILE + r;
    if (tl < ntiles && q < RCH && rw < n) {
      if constexpr (CB == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(tc::smem_u32(sm + S::FST + r * C + 16 * q)),
                     "l"(F + size_t(rw) * C + 16 * q));
      else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(tc::smem_u32(sm + S::FST + r * C + CB * q)),
                     "l"(F + size_t(rw) * C + CB * q), "n"(CB));
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  // hidden layer of tile tl: this thread's H/4 units of row r, into the A operand; then the
  // logit bias b2 initialises the accumulator (columns 64q.. of row r): the MMA adds a W2^T
  // onto it, so the passes read z = b2 + a W2^T directly
  auto hidden_and_bias = [&](uint32_t tl) {
    const uint32_t rw = tl * TILE + r;
    const bool vr = rw < n;
    uint32_t ab[2] = {0u, 0u};
    int32_t hacc[HQ];
    int32_t fw[CW];
#pragma unroll
    for (int w = 0; w < CW; ++w) fw[w] = vr ? reinterpret_cast<const int32_t*>(sm + S::FST + r * C)[w] : 0;
#pragma unroll
    for (int hh = 0; hh < HQ; ++hh) {
      const int h = q * HQ + hh;
      int32_t acc = sb1[h];
#pragma unroll
      for (int w = 0; w < CW; ++w) acc = __dp4a(fw[w], sW1[h * CW + w], acc);
      hacc[hh] = acc;
    }
    if (HQ % 4 == 0 && rq1.fast_s) {
#pragma unroll
      for (int g4 = 0; g4 < HQ / 4; ++g4)
        ab[g4] = pack_sat4(rq_s(hacc[4 * g4], rq1), rq_s(hacc[4 * g4 + 1], rq1), rq_s(hacc[4 * g4 + 2], rq1),
                           rq_s(hacc[4 * g4 + 3], rq1));
    } else {
#pragma unroll
      for (int hh = 0; hh < HQ; ++hh) ab[hh >> 2] |= (uint32_t(rq8(hacc[hh], rq1)) & 0xffu) << (8 * (hh & 3));
    }
    uint8_t* dst = sA + tc::kmaj_off(r, q * HQ);
    // decoder: the hidden activations also go into the node's staged row (DROW_A)
    uint8_t* dra = sm + S::STAGE + r * DROW_BYTES + DROW_A + q * HQ;
    if constexpr (HQ == 8) {
      *reinterpret_cast<uint2*>(dst) = make_uint2(ab[0], ab[1]);
      if (MODE == 1) *reinterpret_cast<uint2*>(dra) = make_uint2(ab[0], ab[1]);
    } else if constexpr (HQ == 4) {
      *reinterpret_cast<uint32_t*>(dst) = ab[0];
      if (MODE == 1) *reinterpret_cast<uint32_t*>(dra) = ab[0];
    } else {
      *reinterpret_cast<uint16_t*>(dst) = uint16_t(ab[0]);
      if (MODE == 1) *reinterpret_cast<uint16_t*>(dra) = uint16_t(ab[0]);
    }
    if (a_dbg && vr) {
      int8_t* ad = a_dbg + size_t(rw) * H + q * HQ;
#pragma unroll
      for (int hh = 0; hh < HQ; ++hh) ad[hh] = int8_t(ab[hh >> 2] >> (8 * (hh & 3)));
    }
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {
      uint32_t bv[16];
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        const uint4 b4 = *reinterpret_cast<const uint4*>(sb2 + 64 * q + 16 * ch + 4 * k4);
        bv[4 * k4] = b4.x, bv[4 * k4 + 1] = b4.y, bv[4 * k4 + 2] = b4.z, bv[4 * k4 + 3] = b4.w;
      }
      tmem_st16(taddr + ch * 16, bv);
    }
    tmem_wait_st();
  };
  if (blockIdx.x < ntiles) {
    prefetch_f(blockIdx.x);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    bar_rows();
    hidden_and_bias(blockIdx.x);
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  long long tr0 = clock64();
  (void)tr0;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t row = tile * TILE + r;
    const bool valid = row < n;
    // A operand and bias-initialised accumulator of this tile are complete (end of the
    // previous iteration / prologue)
    if (tid == 0) {
      tc::mma_i8(tbase, adesc, bdesc, IDESC, 1u);
      tc::commit(mbar);
    }
    prefetch_f(tile + gridDim.x);  // the previous F rows were consumed before the barrier
    tc::mbar_wait(mbar, phase);
    phase ^= 1u;
    tc::fence_after();
    HEAD_TRACE(1, tr0);

    // ---- pass 1: max of z (the requant is monotone non-decreasing, m >= 0, so
    //      max_i lq(z_i) = lq(max_i z_i)) ----
    int32_t zmax = INT32_MIN, zmin = INT32_MAX;
#pragma unroll 1
    for (int ch = 0; ch < 4; ++ch) {
      uint32_t v[16];
      tmem_ld16(taddr + ch * 16, v);
      tc::tmem_wait_ld();
      const bool pad = q == 3 && ch == 3;  // column 255 is padding, not a symbol
#pragma unroll
      for (int k = 0; k < 15; ++k) {
        zmax = max(zmax, int32_t(v[k]));
        if (SAT) zmin = min(zmin, int32_t(v[k]));
      }
      zmax = max(zmax, pad ? INT32_MIN : int32_t(v[15]));
      if (SAT) zmin = min(zmin, pad ? INT32_MAX : int32_t(v[15]));
    }
    red[(q * TILE + r) * 2] = zmax;
    red[(q * TILE + r) * 2 + 1] = zmin;
    bar_rows();
    const int32_t zmx = max(max(red[r * 2], red[(TILE + r) * 2]), max(red[(2 * TILE + r) * 2], red[(3 * TILE + r) * 2]));
    const int32_t zmn =
        min(min(red[r * 2 + 1], red[(TILE + r) * 2 + 1]), min(red[(2 * TILE + r) * 2 + 1], red[(3 * TILE + r) * 2 + 1]));
    const int32_t mu = lq8(zmx, rql);
    // the whole row avoids saturation: l = low word of the 64-bit shift, no selects
    const bool nosat = !SAT || (zmx <= zsat_hi && zmn >= zsat_lo);
    HEAD_TRACE(2, tr0);
    // ---- pass 2: Q8 logit, e = LUT[delta >> 2] (0 beyond 16 nats) and the quarter sum;
    //      decoder: e stored back into TMEM; encoder: the prefix mass before the true
    //      symbol and its own e (reading Q21: C_i = i + floor(E_i * 65281 / S)) ----
    const int sym = (MODE == 0 && valid) ? int(X[row]) - 1 : 0;
    uint32_t ssum = 0, pre = 0, es = 0;
    const int64_t lm = rql.mp;
    const int lr = rql.r;
    // one-multiply form (rq.cuh, signed): delta = mu - lq(z) = hi32(z * (-M) + mu 2^32 + 2^31 - 1)
    const bool fastl = rql.fast_s && nosat;
    const int32_t nM = -rql.Sp;
    const int64_t C2 = (int64_t(mu) << 32) + 0x7fffffff;
    uint32_t csum[4];  // decoder: the quarter's chunk sums (prefix mass at 16-symbol blocks)
#pragma unroll 1
    for (int ch = 0; ch < 4; ++ch) {
      uint32_t v[16];
      tmem_ld16(taddr + ch * 16, v);
      tc::tmem_wait_ld();
      if (fastl) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const uint32_t dl = uint32_t(int32_t((int64_t(int32_t(v[k])) * nM + C2) >> 32));
          v[k] = sLut[min(dl, 4096u)];  // LUT4[4096] = 0: delta >= 4096
        }
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int32_t zz = int32_t(v[k]);
          // lq8(zz) without the 64-bit clamp: saturation is decided in the z domain and
          // selected (branch-free) over the low word of the 64-bit shift
          int32_t lv = int32_t((int64_t(zz) * lm + lhalf) >> lr);
          if (SAT && !nosat) {
            lv = zz > zsat_hi ? (1 << 24) : lv;
            lv = zz < zsat_lo ? -(1 << 24) : lv;
          }
          v[k] = sLut[min(uint32_t(mu - lv), 4096u)];
        }
      }
      if (q == 3 && ch == 3) v[15] = 0u;  // column 255 is padding, not a symbol
      uint32_t cs16 = 0;
#pragma unroll
      for (int k = 0; k < 16; ++k) cs16 += v[k];
      ssum += cs16;
      if constexpr (MODE == 0) {
        const int i0 = 64 * q + ch * 16;
        if (sym >= i0 + 16) {
          pre += cs16;  // the whole chunk precedes the symbol
        } else if (sym >= i0) {  // the chunk holding the symbol (one per row)
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            pre += (i0 + k < sym) ? v[k] : 0u;
            es = (i0 + k == sym) ? v[k] : es;
          }
        }
      } else {
        csum[ch] = cs16;
      }
    }
    bar_rows();  // everyone has read red (pass-1 values) before it is overwritten
    red[(q * TILE + r) * 2] = int32_t(ssum);
    red[(q * TILE + r) * 2 + 1] = int32_t(pre);
    if (MODE == 0) rowi[r * 8 + q] = int32_t(es);
    bar_rows();
    const uint32_t s0 = uint32_t(red[r * 2]), s1 = uint32_t(red[(TILE + r) * 2]), s2 = uint32_t(red[(2 * TILE + r) * 2]),
                   s3 = uint32_t(red[(3 * TILE + r) * 2]);
    const uint32_t Ssum = s0 + s1 + s2 + s3;  // <= 255 * 2^24 < 2^32
    HEAD_TRACE(3, tr0);
    if constexpr (MODE == 0) {
      // encoder: (cum, freq) = (C_sym, C_{sym+1} - C_sym), two exact divisions per node
      if (q == 0 && valid) {
        const uint64_t E = uint64_t(uint32_t(red[r * 2 + 1])) + uint32_t(red[(TILE + r) * 2 + 1]) +
                           uint32_t(red[(2 * TILE + r) * 2 + 1]) + uint32_t(red[(3 * TILE + r) * 2 + 1]);
        const uint64_t e1 = uint64_t(uint32_t(rowi[r * 8])) + uint32_t(rowi[r * 8 + 1]) + uint32_t(rowi[r * 8 + 2]) +
                            uint32_t(rowi[r * 8 + 3]);
        const uint32_t c0 = uint32_t(sym) + uint32_t((E * 65281ull) / Ssum);
        const uint32_t c1 = uint32_t(sym) + 1u + uint32_t(((E + e1) * 65281ull) / Ssum);
        cf[row] = c0 | ((c1 - c0) << 16);
      }
      HEAD_TRACE(4, tr0);
    } else {
      // decoder row header: S, inv32 = floor(65281 * 2^32 / S), mu, and the prefix mass
      // E_{16k} before each 16-symbol block (word 2 + k; this quarter's blocks k = 4q + ch);
      // the rANS decoder rebuilds C_i = i + floor(E_i * 65281 / S) where its search needs it
      uint32_t* hdr = reinterpret_cast<uint32_t*>(sm + S::STAGE + r * DROW_BYTES);
      uint32_t E = (q > 0 ? s0 : 0u) + (q > 1 ? s1 : 0u) + (q > 2 ? s2 : 0u);  // mass before this quarter
      if (q == 0) {
        hdr[0] = Ssum;
        hdr[1] = uint32_t((65281ull << 32) / uint64_t(Ssum));
        hdr[2] = uint32_t(mu);
      } else {
        hdr[2 + 4 * q] = E;  // block 4q
      }
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        E += csum[ch];
        hdr[3 + 4 * q + ch] = E;  // block 4q + ch + 1
      }
      HEAD_TRACE(4, tr0);
      bar_rows();
      // coalesced copy-out of the lane group's 32 rows (contiguous in global and in smem):
      // 32 x 7 16-byte chunks over the group's 128 threads
      const uint32_t rows_here = (n - tile * TILE) < uint32_t(TILE) ? (n - tile * TILE) : uint32_t(TILE);
      const uint32_t g0 = 32u * uint32_t(warp & 3);
      const uint32_t grow = rows_here > g0 ? min(32u, rows_here - g0) : 0u;
      constexpr uint32_t RCH16 = DROW_BYTES / 16;
      const uint4* sp = reinterpret_cast<const uint4*>(sm + S::STAGE + g0 * DROW_BYTES);
      uint4* gp = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(cdf) + (size_t(tile) * TILE + g0) * DROW_BYTES);
      const uint32_t gt = uint32_t(warp >> 2) * 32u + (uint32_t(tid) & 31u);  // 0..127 within the group
#pragma unroll 2
      for (uint32_t t = gt; t < grow * RCH16; t += 128u) gp[t] = sp[t];
      (void)csum;
    }
    HEAD_TRACE(5, tr0);
    // next tile: its F rows landed (own copies + row barrier), hidden layer into A and the
    // bias into this thread's TMEM columns (all of this tile's TMEM reads are done)
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    bar_rows();
    if (tile + gridDim.x < ntiles) hidden_and_bias(tile + gridDim.x);
    HEAD_TRACE(0, tr0);
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();  // A operand + bias complete; stage / red / rowi reused by the next tile
    tc::fence_after();
    HEAD_TRACE(6, tr0);
    tc::fence_after();
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<256>(tbase);
}

// Self-test of the tcgen05 int8 primitive: D[128][N] = A[128][32] * B[N][32]^T.
__global__ void __launch_bounds__(128) k_gemm_i8_test(const int8_t* __restrict__ A, const int8_t* __restrict__ B, int N,
                                                      int32_t* __restrict__ D) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sB = sm;
  uint8_t* sA = sm + 8192;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + 12288);
  uint32_t* thold = reinterpret_cast<uint32_t*>(sm + 12296);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int k = tid; k < N * 8; k += 128) {
    const int r = k >> 3, w = k & 7;
    *reinterpret_cast<uint32_t*>(sB + tc::kmaj_off(r, 4 * w)) = reinterpret_cast<const uint32_t*>(B)[k];
  }
  for (int k = tid; k < 128 * 8; k += 128) {
    const int r = k >> 3, w = k & 7;
    *reinterpret_cast<uint32_t*>(sA + tc::kmaj_off(r, 4 * w)) = reinterpret_cast<const uint32_t*>(A)[k];
  }
  if (warp == 0) tc::tmem_alloc<256>(thold);
  if (tid == 0) tc::mbar_init(mbar, 1);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *thold;
  if (tid == 0) {
    tc::mma_i8(tbase, tc::sdesc(tc::smem_u32(sA)), tc::sdesc(tc::smem_u32(sB)), tc::idesc_i8(128, uint32_t(N)), 0u);
    tc::commit(mbar);
  }
  tc::mbar_wait(mbar, 0);
  tc::fence_after();
  for (int ch = 0; ch < N / 32; ++ch) {
    uint32_t v[32];
    tc::tmem_ld32(tbase + (uint32_t(warp * 32) << 16) + ch * 32, v);
    tc::tmem_wait_ld();
    for (int k = 0; k < 32; ++k) D[size_t(tid) * N + ch * 32 + k] = int32_t(v[k]);
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<256>(tbase);
}

template <int C, int H, int MODE, bool SAT>
void launch_head(pcc_ctx c, const int8_t* F, uint32_t n, const DHead& L, const uint32_t* lut, const uint8_t* X,
                 uint32_t* cf, uint16_t* cdf, int8_t* a_dbg) {
  auto kern = k_head_tc<C, H, MODE, SAT>;
  PCC_SMEM_ATTR(kern, SmemLayout<MODE>::END);
  const uint32_t ntiles = (n + TILE - 1) / TILE;
  const unsigned grid = std::max(1u, std::min(ntiles, unsigned(c->sm_count) * 2u));
  kern<<<grid, NT, SmemLayout<MODE>::END, c->stream>>>(F, n, L.W1, L.b1, L.rq1, L.W2, L.b2, L.rql, lut, X, cf, cdf, a_dbg,
                                                 L.zsat_lo, L.zsat_hi);
  launched(c);
}

}  // namespace

void head_cdf_tc(pcc_ctx c, const int8_t* F, uint32_t n, int C, int H, const DHead& L, const uint32_t* lut, int mode,
                 const uint8_t* X, uint32_t* cf, uint16_t* cdf, int8_t* a_dbg) {
  if (n == 0) return;
  Prof p(c, mode == 0 ? "head_enc" : "head_dec", size_t(n) * (C + (mode == 0 ? 1 + 4 : DROW_BYTES)));
#define PCC_HEAD(CC)                                                         \
  if (C == CC && H == CC) {                                                  \
    if (mode == 0 && L.can_saturate) launch_head<CC, CC, 0, true>(c, F, n, L, lut, X, cf, cdf, a_dbg);  \
    else if (mode == 0) launch_head<CC, CC, 0, false>(c, F, n, L, lut, X, cf, cdf, a_dbg);       \
    else if (L.can_saturate) launch_head<CC, CC, 1, true>(c, F, n, L, lut, X, cf, cdf, a_dbg);   \
    else launch_head<CC, CC, 1, false>(c, F, n, L, lut, X, cf, cdf, a_dbg);                      \
    return;                                                                  \
  }
  PCC_HEAD(8)
  PCC_HEAD(16)
  PCC_HEAD(32)
#undef PCC_HEAD
  throw Error{PCC_ERR_INVALID_ARG};
}

void gemm_i8_test(pcc_ctx c, const int8_t* dA, const int8_t* dB, int N, int32_t* dD) {
  if (N < 32 || N > 256 || N % 32) throw Error{PCC_ERR_INVALID_ARG};
  PCC_SMEM_ATTR(k_gemm_i8_test, 80 * 1024);
  k_gemm_i8_test<<<1, 128, 80 * 1024, c->stream>>>(dA, dB, N, dD);
  launched(c);
}

}  // namespace pcc

#ifdef PCC_TRACE
extern "C" int pcc_trace_head(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, pcc::g_head_trace, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(pcc::g_head_trace, z, sizeof(z));
  }
  return 0;
}
#endif
