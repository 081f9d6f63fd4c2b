// up_tc.cu — GRED re-sparsification (Upsampling + Pruning, Eq.6/9/11) on the
// 5th-generation tensor cores, C = 32.
//
// Upsampling is "a linear transformation followed by a PReLU activation, performing an
// 8x channel expansion" over Concat(S, X) (reading Q6: the one-hot half is the int32 row
// E[X] = q_one * W_X[:, X]); Pruning "discards features of unoccupied child nodes".
// Transposed product on tcgen05.mma.kind::i8: D[o][p] = W_S[o] . S[p] with the 256 output
// channels as M (two M = 128 halves, A = W_S staged once per CTA) and a tile of 128
// parents as N (B = the parent rows, cp.async, double-buffered): TMEM lane = channel,
// column = parent.  A warp of lane quarter q reads channel block c of 16 parents per
// tcgen05.ld, so the occupancy test "does parent p have child c" is uniform across the
// warp, and a warp ballot turns it into a mask that the warp walks: no lane idles on a
// pruned child and a pruned child costs one uniform branch.  The one-hot half is
// q_one * W_X[o][X] (reading Q6) read from a transposed copy of W_X held in smem (65 KB,
// one conflict-free 32-byte row per kept child), the bias is a per-lane register; then
// the fast exact requant (rq.cuh) and one byte per lane of the child row
// child_start[p] + rank(c) (children contiguous, Morton order, reading Q8).
#include "pcc_internal.cuh"
#include "rq.cuh"
#include "tc.cuh"

namespace pcc {

namespace {

constexpr int UT = 128;  // parents per tile
constexpr int UNT = 512; // threads per CTA (4 per parent)
constexpr uint32_t IDESC_UP = tc::idesc_i8(128, UT);

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

// smem: A = W_S as two [128 x 32] canonical K-major halves (8 KB); per buffer: the parent
// tile [128 x 32] (4 KB), its codes and child starts; W_X transposed [255][256] int8.
constexpr int SM_A = 0, SM_S = 8192, SM_X = SM_S + 2 * 4096, SM_CS = SM_X + 2 * UT, SM_WX = SM_CS + 2 * UT * 4;
constexpr int SM_MBAR = SM_WX + NCODE * 256;
constexpr int SM_END = SM_MBAR + 64;

__global__ void __launch_bounds__(UNT, 2) k_up_tc(const int8_t* __restrict__ S, const uint8_t* __restrict__ Xp,
                                                  const uint32_t* __restrict__ cs, uint32_t np, uint32_t nc,
                                                  const int8_t* __restrict__ WS, const int8_t* __restrict__ WXt,
                                                  const int32_t* __restrict__ bias, int32_t q_one, RQ rq,
                                                  int8_t* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm + SM_A;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + SM_MBAR);
  uint32_t* thold = reinterpret_cast<uint32_t*>(sm + SM_MBAR + 8);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int qd = warp & 3;          // TMEM lane quarter: channels 32qd.. of a half
  const int hv = (warp >> 2) & 1;   // channel half -> child block c = 4hv + qd
  const int c = 4 * hv + qd;
  const int pr = warp >> 3;         // parents 64pr .. 64pr+63 of the tile
  const uint32_t below = (1u << c) - 1u;

  // W_S [256][32]: row o -> half o/128, row o%128 (two 16-byte chunks per row)
  for (int k = t; k < 512; k += UNT) {
    const int o = k >> 1, h = k & 1;
    *reinterpret_cast<uint4*>(sA + (o >> 7) * 4096 + tc::kmaj_off(o & 127, 16 * h)) =
        reinterpret_cast<const uint4*>(WS)[k];
  }
  for (int k = t; k < NCODE * 256 / 16; k += UNT)
    reinterpret_cast<uint4*>(sm + SM_WX)[k] = reinterpret_cast<const uint4*>(WXt)[k];
  const int8_t* sWX = reinterpret_cast<const int8_t*>(sm + SM_WX) + 32 * c + lane - 256;  // row X-1
  const int32_t bias_r = bias[32 * c + lane];
  if (warp == 0) tc::tmem_alloc<256>(thold);
  if (t == 0) tc::mbar_init(mbar, 1);
  const uint32_t ntiles = (np + UT - 1) / UT;
  if (blockIdx.x == 0 && t < 8) reinterpret_cast<uint32_t*>(out + size_t(nc) * 32)[t] = 0u;  // zero row

  // stage tile `tile` into buffer `b`: parent rows by cp.async, codes / child starts by threads 256..383
  auto stage = [&](uint32_t tile, int b) {
    uint8_t* sS = sm + SM_S + b * 4096;
    if (t < 2 * UT) {
      const int rr = t >> 1, h = t & 1;
      const uint32_t pp = tile * UT + rr;
      if (pp < np) cp16(sS + tc::kmaj_off(rr, 16 * h), S + size_t(pp) * 32 + 16 * h);
      else *reinterpret_cast<uint4*>(sS + tc::kmaj_off(rr, 16 * h)) = make_uint4(0u, 0u, 0u, 0u);
    } else if (t < 3 * UT) {
      const int rr = t - 2 * UT;
      const uint32_t pp = tile * UT + rr;
      sm[SM_X + b * UT + rr] = pp < np ? Xp[pp] : uint8_t(0);
      reinterpret_cast<uint32_t*>(sm + SM_CS)[b * UT + rr] = pp < np ? cs[pp] : 0u;
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  if (blockIdx.x < ntiles) stage(blockIdx.x, 0);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *thold;
  uint32_t phase = 0;
  int buf = 0;

  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, buf ^= 1) {
    if (t == 0) {
      const uint64_t bdesc = tc::sdesc(tc::smem_u32(sm + SM_S + buf * 4096));
      tc::mma_i8(tbase, tc::sdesc(tc::smem_u32(sA)), bdesc, IDESC_UP, 0u);
      tc::mma_i8(tbase + 128, tc::sdesc(tc::smem_u32(sA + 4096)), bdesc, IDESC_UP, 0u);
      tc::commit(mbar);
    }
    if (tile + gridDim.x < ntiles) stage(tile + gridDim.x, buf ^ 1);  // overlaps the MMA + epilogue
    tc::mbar_wait(mbar, phase);
    phase ^= 1u;
    tc::fence_after();
    const uint8_t* sX = sm + SM_X + buf * UT;
    const uint32_t* sCS = reinterpret_cast<const uint32_t*>(sm + SM_CS) + buf * UT;
#pragma unroll 1
    for (int j0 = 64 * pr; j0 < 64 * pr + 64; j0 += 16) {
      uint32_t v[16];
      tmem_ld16(tbase + (uint32_t(32 * qd) << 16) + uint32_t(128 * hv + j0), v);
      uint32_t xl = 0u, cl = 0u;
      if (lane < 16) {
        xl = sX[j0 + lane];
        cl = sCS[j0 + lane];
      }
      const uint32_t m = __ballot_sync(0xffffffffu, (xl >> c) & 1u);  // parents with child c
      tc::tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if ((m >> i) & 1u) {  // warp-uniform
          const uint32_t x = __shfl_sync(0xffffffffu, xl, i);
          const uint32_t row = __shfl_sync(0xffffffffu, cl, i) + __popc(x & below);
          const int32_t e = q_one * int32_t(sWX[x * 256]) + bias_r;
          out[size_t(row) * 32 + lane] = int8_t(rq8(int32_t(v[i]) + e, rq));
        }
      }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();  // TMEM and the staged tile are reused by the next tile
    tc::fence_after();
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<256>(tbase);
}

}  // namespace

void up_prune_tc(pcc_ctx c, const int8_t* S, const uint8_t* Xp, const uint32_t* cs_p, uint32_t np, uint32_t nc,
                 const DUp& L, int8_t* out) {
  constexpr int smem = SM_END;  // ~83 KB: 2 CTAs/SM (also the TMEM limit, 2 x 256 columns)
  static bool attr = false;
  if (!attr) {
    PCC_CUDA(cudaFuncSetAttribute(k_up_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  const uint32_t ntiles = (np + UT - 1) / UT;
  const unsigned grid = std::max(1u, std::min(ntiles, unsigned(c->sm_count) * 2u));
  Prof p(c, "up", size_t(nc) * 32 + size_t(np) * (32 + 1 + 4));
  k_up_tc<<<grid, UNT, smem, c->stream>>>(S, Xp, cs_p, np, nc, L.W, L.WXt, L.b, L.q_one, L.rq, out);
  launched(c);
}

}  // namespace pcc
