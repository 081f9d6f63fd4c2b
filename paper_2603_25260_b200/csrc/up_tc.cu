// up_tc.cu — GRED re-sparsification (Upsampling + Pruning, Eq.6/9/11) on the
// 5th-generation tensor cores, C = 32.
//
// Upsampling is "a linear transformation followed by a PReLU activation, performing an
// 8x channel expansion" over Concat(S, X) (reading Q6: the one-hot half is the int32 row
// E[X] = q_one * W_X[:, X]); Pruning "discards features of unoccupied child nodes".
// Per tile of 128 parents the A operand is the literal concatenation [S | q_one*onehot(X)]
// (K = 32 + 256, one-hot built in smem), times the model's Concat+Linear weight
// [256 x 288]: nine tcgen05.mma.kind::i8 (M = 128, N = 256, K = 32) into one TMEM
// accumulator.  Epilogue: 4 threads per parent (TMEM lane), thread quarter q owns child
// blocks c = 2q, 2q+1 (columns 64q..64q+63); for each occupied child c it adds the bias,
// PReLU-requantises the 32 outputs and writes the child row
// child_start[p] + rank(c) (children are contiguous and in Morton order, reading Q8).
// Bit-exact with the dp4a kernel and the oracle's up_prune.
#include "pcc_internal.cuh"
#include "tc.cuh"

namespace pcc {

namespace {

constexpr int UT = 128;  // parents per tile
constexpr int UNT = 512; // threads per CTA (4 per parent)
constexpr uint32_t IDESC_UP = tc::idesc_i8(128, 256);

__device__ __forceinline__ int32_t rq8(int32_t acc, RQ q) {
  int64_t v = int64_t(acc) * int64_t(acc >= 0 ? q.mp : q.mn);
  if (q.r > 0) v = (v + (int64_t(1) << (q.r - 1))) >> q.r;
  return int32_t(v < -128 ? -128 : (v > 127 ? 127 : v));
}

__device__ __forceinline__ void cp16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(tc::smem_u32(s)), "l"(g));
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

// smem: B = Wcat as 9 K-slabs of 256 x 32 (72 KB), A = 9 K-slabs of 128 x 32 (36 KB):
// slab 0 the parent rows S, slabs 1..8 the one-hot of X (q_one at column X-1).
constexpr int KSL = 9;
constexpr int SM_B = 0, SM_A = KSL * 8192, SM_BIAS = SM_A + KSL * 4096, SM_MBAR = SM_BIAS + 1024;
constexpr int SM_END = SM_MBAR + 64;

__global__ void __launch_bounds__(UNT, 2) k_up_tc(const int8_t* __restrict__ S, const uint8_t* __restrict__ Xp,
                                                  const uint32_t* __restrict__ cs, uint32_t np, uint32_t nc,
                                                  const int8_t* __restrict__ Wcat, const int32_t* __restrict__ bias,
                                                  RQ rq, int32_t q_one, int8_t* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sB = sm + SM_B;
  uint8_t* sA = sm + SM_A;
  int32_t* sbias = reinterpret_cast<int32_t*>(sm + SM_BIAS);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + SM_MBAR);
  uint32_t* thold = reinterpret_cast<uint32_t*>(sm + SM_MBAR + 8);
  const int t = threadIdx.x, warp = t >> 5;
  const int r = 32 * (warp & 3) + (t & 31);  // parent of the tile (= TMEM lane)
  const int q = warp >> 2;                   // child blocks 2q, 2q+1

  // Wcat [256][288]: 18 x 16-byte chunks per output row -> slab h/2, K half h%2
  for (int k = t; k < 256 * 18; k += UNT) {
    const int o = k / 18, h = k % 18;
    *reinterpret_cast<uint4*>(sB + (h >> 1) * 8192 + tc::kmaj_off(o, 16 * (h & 1))) =
        reinterpret_cast<const uint4*>(Wcat)[k];
  }
  for (int k = t; k < KSL * 4096 / 16; k += UNT) reinterpret_cast<uint4*>(sA)[k] = make_uint4(0u, 0u, 0u, 0u);
  for (int k = t; k < 256; k += UNT) sbias[k] = bias[k];
  if (warp == 0) tc::tmem_alloc<256>(thold);
  if (t == 0) tc::mbar_init(mbar, 1);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *thold;
  const uint32_t taddr = tbase + (uint32_t(32 * (warp & 3)) << 16);
  const uint32_t ntiles = (np + UT - 1) / UT;
  uint32_t phase = 0;
  if (blockIdx.x == 0 && t < 8) reinterpret_cast<uint32_t*>(out + size_t(nc) * 32)[t] = 0u;  // zero row

  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t p = tile * UT + r;
    const bool valid = p < np;
    const uint32_t x = valid ? uint32_t(Xp[p]) : 0u;
    const uint32_t c0 = valid ? cs[p] : 0u;
    uint8_t* hot = nullptr;  // this row's one-hot byte (set by quarter 0)
    if (t < 2 * UT) {  // slab 0: parent rows, two 16-byte halves each
      const int rr = t >> 1, h = t & 1;
      const uint32_t pp = tile * UT + rr;
      if (pp < np) cp16(sA + tc::kmaj_off(rr, 16 * h), S + size_t(pp) * 32 + 16 * h);
      else *reinterpret_cast<uint4*>(sA + tc::kmaj_off(rr, 16 * h)) = make_uint4(0u, 0u, 0u, 0u);
    }
    if (q == 0 && x != 0u) {  // Concat(S, X): q_one at one-hot column x-1 (reading Q6)
      hot = sA + (1 + (x - 1) / 32) * 4096 + tc::kmaj_off(r, (x - 1) % 32);
      *hot = uint8_t(int8_t(q_one));
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (t == 0) {
#pragma unroll
      for (int s = 0; s < KSL; ++s)
        tc::mma_i8(tbase, tc::sdesc(tc::smem_u32(sA + s * 4096)), tc::sdesc(tc::smem_u32(sB + s * 8192)), IDESC_UP,
                   s > 0 ? 1u : 0u);
      tc::commit(mbar);
    }
    tc::mbar_wait(mbar, phase);
    phase ^= 1u;
    tc::fence_after();
    if (hot) *hot = 0u;  // the MMAs have consumed the tile: restore the all-zero one-hot slabs
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      const int c = 2 * q + cc;
      const bool occ = (x >> c) & 1u;
      // warp-collective TMEM loads: issue only if some parent of this warp has child c
      if (__any_sync(0xffffffffu, occ)) {
        uint32_t v[32];
        tmem_ld16(taddr + uint32_t(32 * c), *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
        tmem_ld16(taddr + uint32_t(32 * c + 16), *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
        tc::tmem_wait_ld();
        if (occ) {
          uint32_t w[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int32_t* bb = sbias + 32 * c + 4 * k;
            const uint32_t b0 = uint32_t(rq8(int32_t(v[4 * k]) + bb[0], rq)) & 0xffu;
            const uint32_t b1 = uint32_t(rq8(int32_t(v[4 * k + 1]) + bb[1], rq)) & 0xffu;
            const uint32_t b2 = uint32_t(rq8(int32_t(v[4 * k + 2]) + bb[2], rq)) & 0xffu;
            const uint32_t b3 = uint32_t(rq8(int32_t(v[4 * k + 3]) + bb[3], rq)) & 0xffu;
            w[k] = b0 | (b1 << 8) | (b2 << 16) | (b3 << 24);
          }
          const uint32_t row = c0 + __popc(x & ((1u << c) - 1u));
          uint4* o4 = reinterpret_cast<uint4*>(out + size_t(row) * 32);
          o4[0] = make_uint4(w[0], w[1], w[2], w[3]);
          o4[1] = make_uint4(w[4], w[5], w[6], w[7]);
        }
      }
    }
    tc::fence_before();
    __syncthreads();  // TMEM and the A tile are reused by the next tile
    tc::fence_after();
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<256>(tbase);
}

}  // namespace

void up_prune_tc(pcc_ctx c, const int8_t* S, const uint8_t* Xp, const uint32_t* cs_p, uint32_t np, uint32_t nc,
                 const DUp& L, int8_t* out) {
  constexpr int smem = SM_END;  // ~109 KB: at most 2 CTAs/SM (also the TMEM limit, 2 x 256 cols)
  static bool attr = false;
  if (!attr) {
    PCC_CUDA(cudaFuncSetAttribute(k_up_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  const uint32_t ntiles = (np + UT - 1) / UT;
  const unsigned grid = std::max(1u, std::min(ntiles, unsigned(c->sm_count) * 2u));
  Prof p(c, "up", size_t(nc) * 32 + size_t(np) * (32 + 1 + 4));
  k_up_tc<<<grid, UNT, smem, c->stream>>>(S, Xp, cs_p, np, nc, L.Wcat, L.b, L.rq, L.q_one, out);
  launched(c);
}

}  // namespace pcc
