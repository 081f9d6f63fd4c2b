// head_tc.cu — occupancy predictor (Eq.7) + integer softmax to a Q16 pmf
// (Eq.15; readings Q20-Q22) on the 5th-generation tensor cores.
//
// One CTA = 128 threads = one 128-node tile per iteration (persistent over tiles).
//   1. hidden layer a = prq(W1 F + b1) (C -> H, int8 dp4a) written straight into the
//      tcgen05 A operand (canonical K-major smem tile, K padded to 32 with zeros);
//   2. z = a W2^T: ONE tcgen05.mma.kind::i8 (M = 128, N = 256, K = 32) into TMEM
//      (int32; column 255 is padding);
//   3. thread t owns TMEM lane t = node t of the tile and runs the softmax over its
//      row with 32-column tcgen05.ld loads: pass 1 requantises z to Q8 logits (written
//      back with tcgen05.st) and finds max / first argmax, pass 2 turns them into LUT
//      exponentials (written back) and their sum S, pass 3 forms p = 1 + floor(e*65281/S)
//      (exact: 64-bit reciprocal + one integer correction) and either the (cum, freq)
//      of the true symbol (encoder) or the cumulative row (decoder, staged in smem and
//      written with coalesced stores).
// Bit-exact with the oracle's cdf_quantize / head_logits (integer arithmetic only).
#include "pcc_internal.cuh"
#include "tc.cuh"

namespace pcc {

namespace {

constexpr int TILE = 128;
constexpr uint32_t IDESC = tc::idesc_i8(128, 256);
constexpr int STG = 258;  // staged cdf row stride in u16 (516 B: conflict-free)

__device__ __forceinline__ int32_t rq8(int32_t acc, RQ q) {
  int64_t v = int64_t(acc) * int64_t(acc >= 0 ? q.mp : q.mn);
  if (q.r > 0) v = (v + (int64_t(1) << (q.r - 1))) >> q.r;
  return int32_t(v < -128 ? -128 : (v > 127 ? 127 : v));
}

__device__ __forceinline__ int32_t lq8(int32_t z, RQ q) {  // Q8 logit, clamp +-2^24
  int64_t v = int64_t(z) * int64_t(q.mp);
  if (q.r > 0) v = (v + (int64_t(1) << (q.r - 1))) >> q.r;
  v = v < -(int64_t(1) << 24) ? -(int64_t(1) << 24) : (v > (int64_t(1) << 24) ? (int64_t(1) << 24) : v);
  return int32_t(v);
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

struct SmemLayout {
  static constexpr int B = 0;           // W2 operand 256 x 32 (8 KB)
  static constexpr int A = 8192;        // a operand 128 x 32 (4 KB)
  static constexpr int LUT = 12288;     // 4 KB
  static constexpr int B2 = 16384;      // 1 KB
  static constexpr int W1 = 17408;      // <= 1 KB
  static constexpr int B1 = 18432;      // <= 256 B
  static constexpr int MBAR = 18688;
  static constexpr int THOLD = 18696;
  static constexpr int ROWI = 18704;    // 128 x (left, istar)
  static constexpr int STAGE = 19776;   // decoder: 128 x STG u16
  static constexpr int END_DEC = STAGE + TILE * STG * 2;
  static constexpr int END = 88 * 1024; // >= END_DEC; caps residency at 2 CTAs/SM (TMEM: 2 x 256 cols)
};
static_assert(SmemLayout::END_DEC <= SmemLayout::END, "decoder staging exceeds the smem budget");

template <int C, int H, int MODE>
__global__ void __launch_bounds__(TILE, 2) k_head_tc(const int8_t* __restrict__ F, uint32_t n,
                                                     const int8_t* __restrict__ W1, const int32_t* __restrict__ b1, RQ rq1,
                                                     const int8_t* __restrict__ W2, const int32_t* __restrict__ b2, RQ rql,
                                                     const uint32_t* __restrict__ lut, const uint8_t* __restrict__ X,
                                                     uint32_t* __restrict__ cf, uint16_t* __restrict__ cdf,
                                                     int8_t* __restrict__ a_dbg) {
  extern __shared__ __align__(1024) uint8_t sm[];
  using S = SmemLayout;
  uint8_t* sB = sm + S::B;
  uint8_t* sA = sm + S::A;
  uint32_t* sLut = reinterpret_cast<uint32_t*>(sm + S::LUT);
  int32_t* sb2 = reinterpret_cast<int32_t*>(sm + S::B2);
  int32_t* sW1 = reinterpret_cast<int32_t*>(sm + S::W1);
  int32_t* sb1 = reinterpret_cast<int32_t*>(sm + S::B1);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + S::MBAR);
  uint32_t* thold = reinterpret_cast<uint32_t*>(sm + S::THOLD);
  int32_t* rowi = reinterpret_cast<int32_t*>(sm + S::ROWI);
  uint16_t* stage = reinterpret_cast<uint16_t*>(sm + S::STAGE);
  const int tid = threadIdx.x, warp = tid >> 5;
  constexpr int CW = C / 4, HW = H / 4;

  // B operand: W2 [256][H] -> canonical K-major 256 x 32 (K >= H zero-padded)
  for (int k = tid; k < 256 * 8; k += TILE) {
    const int r = k >> 3, w = k & 7;
    const uint32_t v = (w < HW) ? reinterpret_cast<const uint32_t*>(W2)[r * HW + w] : 0u;
    *reinterpret_cast<uint32_t*>(sB + tc::kmaj_off(r, 4 * w)) = v;
  }
  for (int k = tid; k < 1024; k += TILE) sLut[k] = lut[k];
  for (int k = tid; k < 256; k += TILE) sb2[k] = b2[k];
  for (int k = tid; k < H * CW; k += TILE) sW1[k] = reinterpret_cast<const int32_t*>(W1)[k];
  for (int k = tid; k < H; k += TILE) sb1[k] = b1[k];
  if (warp == 0) tc::tmem_alloc<256>(thold);
  if (tid == 0) tc::mbar_init(mbar, 1);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *thold;
  const uint32_t taddr = tbase + (uint32_t(warp * 32) << 16);
  const uint64_t adesc = tc::sdesc(tc::smem_u32(sA));
  const uint64_t bdesc = tc::sdesc(tc::smem_u32(sB));
  const uint32_t ntiles = (n + TILE - 1) / TILE;
  uint32_t phase = 0;

  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t row = tile * TILE + tid;
    const bool valid = row < n;
    // ---- hidden layer (C -> H) into the A operand ----
    int32_t fw[CW];
#pragma unroll
    for (int w = 0; w < CW; ++w) fw[w] = valid ? reinterpret_cast<const int32_t*>(F + size_t(row) * C)[w] : 0;
    uint32_t aw[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) aw[w] = 0;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      int32_t acc = sb1[h];
#pragma unroll
      for (int w = 0; w < CW; ++w) acc = __dp4a(fw[w], sW1[h * CW + w], acc);
      const uint32_t q = uint32_t(rq8(acc, rq1)) & 0xffu;
      aw[h >> 2] |= q << (8 * (h & 3));
    }
    if (a_dbg && valid) {
#pragma unroll
      for (int w = 0; w < HW; ++w) reinterpret_cast<uint32_t*>(a_dbg + size_t(row) * H)[w] = aw[w];
    }
    *reinterpret_cast<uint4*>(sA + tc::kmaj_off(tid, 0)) = make_uint4(aw[0], aw[1], aw[2], aw[3]);
    *reinterpret_cast<uint4*>(sA + tc::kmaj_off(tid, 16)) = make_uint4(aw[4], aw[5], aw[6], aw[7]);
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (tid == 0) {
      tc::mma_i8(tbase, adesc, bdesc, IDESC, 0u);
      tc::commit(mbar);
    }
    tc::mbar_wait(mbar, phase);
    phase ^= 1u;
    tc::fence_after();

    // ---- pass 1: Q8 logits (stored back into TMEM), max and first argmax ----
    int32_t lmax = INT32_MIN;
    int istar = 0;
#pragma unroll 1
    for (int ch = 0; ch < 8; ++ch) {
      uint32_t v[32];
      tc::tmem_ld32(taddr + ch * 32, v);
      tc::tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int i = ch * 32 + k;
        const int32_t l = lq8(int32_t(v[k]) + sb2[i], rql);
        v[k] = uint32_t(l);
        if (i < NCODE && l > lmax) {
          lmax = l;
          istar = i;
        }
      }
      tmem_st32(taddr + ch * 32, v);
    }
    tmem_wait_st();
    // ---- pass 2: e = LUT[delta >> 2] (0 beyond 16 nats), S = sum e ----
    uint32_t Ssum = 0;
#pragma unroll 1
    for (int ch = 0; ch < 8; ++ch) {
      uint32_t v[32];
      tc::tmem_ld32(taddr + ch * 32, v);
      tc::tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int i = ch * 32 + k;
        const uint32_t dl = uint32_t(lmax - int32_t(v[k]));
        const uint32_t e = (i < NCODE && dl < 4096u) ? sLut[dl >> 2] : 0u;
        v[k] = e;
        Ssum += e;
      }
      tmem_st32(taddr + ch * 32, v);
    }
    tmem_wait_st();
    // ---- pass 3: p = 1 + floor(e * 65281 / S), leftover to the first argmax ----
    const uint64_t inv = ~0ull / uint64_t(Ssum);
    uint32_t tot = 0;
    if constexpr (MODE == 0) {
      const int sym = valid ? int(X[row]) - 1 : 0;
      uint32_t cum = 0, fq = 0;
#pragma unroll 1
      for (int ch = 0; ch < 8; ++ch) {
        uint32_t v[32];
        tc::tmem_ld32(taddr + ch * 32, v);
        tc::tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int i = ch * 32 + k;
          const uint64_t num = uint64_t(v[k]) * 65281ull;
          uint64_t q = __umul64hi(num, inv);
          if (num - q * uint64_t(Ssum) >= uint64_t(Ssum)) ++q;
          const uint32_t p = (i < NCODE) ? uint32_t(1 + q) : 0u;
          tot += p;
          cum += (i < sym) ? p : 0u;
          fq = (i == sym) ? p : fq;
        }
      }
      const uint32_t left = 65536u - tot;
      if (istar < sym) cum += left;
      if (istar == sym) fq += left;
      if (valid) cf[row] = cum | (fq << 16);
    } else {
      uint16_t* srow = stage + tid * STG;
      uint32_t run = 0;
#pragma unroll 1
      for (int ch = 0; ch < 8; ++ch) {
        uint32_t v[32];
        tc::tmem_ld32(taddr + ch * 32, v);
        tc::tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 32; k += 2) {
          const int i = ch * 32 + k;
          uint32_t c2[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const uint64_t num = uint64_t(v[k + u]) * 65281ull;
            uint64_t q = __umul64hi(num, inv);
            if (num - q * uint64_t(Ssum) >= uint64_t(Ssum)) ++q;
            const uint32_t p = (i + u < NCODE) ? uint32_t(1 + q) : 0u;
            c2[u] = run;
            run += p;
          }
          *reinterpret_cast<uint32_t*>(srow + i) = (c2[0] & 0xffffu) | (c2[1] << 16);
        }
      }
      tot = run;
      rowi[2 * tid] = int32_t(65536u - tot);
      rowi[2 * tid + 1] = istar;
      __syncthreads();
      // coalesced write-out: one 512-byte row per iteration, leftover added after i*
      const uint32_t rows_here = (n - tile * TILE) < uint32_t(TILE) ? (n - tile * TILE) : uint32_t(TILE);
      for (uint32_t r = 0; r < rows_here; ++r) {
        const uint32_t i0 = 2u * tid;
        const uint32_t left = uint32_t(rowi[2 * r]);
        const int ist = rowi[2 * r + 1];
        const uint32_t pair = *reinterpret_cast<const uint32_t*>(stage + r * STG + i0);
        uint32_t c0 = (pair & 0xffffu) + (int(i0) > ist ? left : 0u);
        uint32_t c1 = (pair >> 16) + (int(i0 + 1) > ist ? left : 0u);
        if (i0 + 1 >= uint32_t(NCODE)) c1 = 0xffffu;
        reinterpret_cast<uint32_t*>(cdf + size_t(tile * TILE + r) * 256)[tid] = (c0 & 0xffffu) | (c1 << 16);
      }
    }
    tc::fence_before();
    __syncthreads();  // TMEM / sA / stage reused by the next tile
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

template <int C, int H, int MODE>
void launch_head(pcc_ctx c, const int8_t* F, uint32_t n, const DHead& L, const uint32_t* lut, const uint8_t* X,
                 uint32_t* cf, uint16_t* cdf, int8_t* a_dbg) {
  auto kern = k_head_tc<C, H, MODE>;
  static bool attr = false;
  if (!attr) {
    PCC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SmemLayout::END));
    attr = true;
  }
  const uint32_t ntiles = (n + TILE - 1) / TILE;
  const unsigned grid = std::max(1u, std::min(ntiles, unsigned(c->sm_count) * 2u));
  kern<<<grid, TILE, SmemLayout::END, c->stream>>>(F, n, L.W1, L.b1, L.rq1, L.W2, L.b2, L.rql, lut, X, cf, cdf, a_dbg);
  launched(c);
}

}  // namespace

void head_cdf_tc(pcc_ctx c, const int8_t* F, uint32_t n, int C, int H, const DHead& L, const uint32_t* lut, int mode,
                 const uint8_t* X, uint32_t* cf, uint16_t* cdf, int8_t* a_dbg) {
  if (n == 0) return;
  Prof p(c, mode == 0 ? "head_enc" : "head_dec", size_t(n) * (C + (mode == 0 ? 1 + 4 : 512)));
#define PCC_HEAD(CC)                                                         \
  if (C == CC && H == CC) {                                                  \
    if (mode == 0) launch_head<CC, CC, 0>(c, F, n, L, lut, X, cf, cdf, a_dbg); \
    else launch_head<CC, CC, 1>(c, F, n, L, lut, X, cf, cdf, a_dbg);          \
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
  static bool attr = false;
  if (!attr) {
    PCC_CUDA(cudaFuncSetAttribute(k_gemm_i8_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024));
    attr = true;
  }
  k_gemm_i8_test<<<1, 128, 80 * 1024, c->stream>>>(dA, dB, N, dD);
  launched(c);
}

}  // namespace pcc
