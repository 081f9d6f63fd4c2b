// down_tc.cu — GRED downsampling (K2S2 sparse conv, Eq.10) on the 5th-generation
// tensor cores, C = 32.
//
// The downsampled feature of parent p is Σ_c W_c · g[child_c(p)] over its occupied children
// c (W_c = the kernel tap of child position c, children contiguous from child_start[p] in
// Morton order, reading Q8).  As a block-diagonal product on tcgen05.mma.kind::i8: a tile
// is 128 consecutive parents (M = 128, TMEM lane = parent); row p of the A operand holds
// the child row g[child_start[p] + rank(c)] in K-slot c for every occupied child c (zero
// elsewhere), B[o][32c + i] = W_c[o][i], so D[p][o] = Σ_c W_c[o] · g[child_c] (N = 32,
// K = 256: eight MMAs).  Epilogue: one lane per parent, bias in registers, the signed
// one-multiply requant (rq.cuh) and two 16-byte stores.  Four independent 128-thread tile
// groups per CTA (own A tile, TMEM accumulator, mbarrier, named barrier) overlap one
// another's gathers, MMAs and epilogues; within a group the next tile's gather is in
// flight during the current epilogue.  Bit-exact with the dp4a kernel and the oracle.
#include "pcc_internal.cuh"
#include "rq.cuh"
#include "tc.cuh"

namespace pcc {

namespace {

constexpr int DG = 4;             // tile groups per CTA
constexpr int DNT = 128 * DG;     // threads per CTA (one per parent row of each group's tile)
constexpr uint32_t IDESC_DN = tc::idesc_i8(128, 32);

__device__ __forceinline__ void cp16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(tc::smem_u32(s)), "l"(g));
}
__device__ __forceinline__ void bar_group(int id) { asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory"); }

// smem: per group an A tile [128 x 256] (8 canonical slabs of 4 KB); B = 8 slabs [32 x 32];
// mbarriers + TMEM holder
constexpr int SM_A = 0, SM_B = DG * 32768, SM_MBAR = SM_B + 8192, SM_E = SM_MBAR + 128, SM_END = SM_E + NCODE * 32;

// EMB: the child rows are the embedding g = E[X_c - 1] of the children's codes (Eq.4, the
// first K2S2 step of a deep level, reading Q5): gathered straight from the 255 x 32 table
// instead of a materialised embedded level.
template <bool SIGNED, bool EMB>
__global__ void __launch_bounds__(DNT, 1) k_down_tc(const int8_t* __restrict__ g, const uint8_t* __restrict__ Xp,
                                                    const uint32_t* __restrict__ cs, uint32_t np,
                                                    const int8_t* __restrict__ W, const int32_t* __restrict__ bias,
                                                    RQ rq, int8_t* __restrict__ out, const uint8_t* __restrict__ Xc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int t = threadIdx.x, grp = t >> 7, r = t & 127;  // group, parent row of the tile (= TMEM lane)
  uint8_t* sA = sm + SM_A + grp * 32768;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + SM_MBAR) + grp;
  uint32_t* thold = reinterpret_cast<uint32_t*>(sm + SM_MBAR + 8 * DG);

  // B slab c, row o: W[c][o][0..31] (two 16-byte chunks)
  for (int k = t; k < 512; k += DNT) {
    const int co = k >> 1, h = k & 1;  // co = 32c + o
    *reinterpret_cast<uint4*>(sm + SM_B + (co >> 5) * 1024 + tc::kmaj_off(co & 31, 16 * h)) =
        reinterpret_cast<const uint4*>(W)[k];
  }
  for (int k = t; k < DG * 32768 / 16; k += DNT) reinterpret_cast<uint4*>(sm + SM_A)[k] = make_uint4(0u, 0u, 0u, 0u);
  if (EMB)  // the embedding table: every child row of the step is one of its 255 rows
    for (int k = t; k < NCODE * 2; k += DNT) reinterpret_cast<uint4*>(sm + SM_E)[k] = reinterpret_cast<const uint4*>(g)[k];
  if (t < 32) tc::tmem_alloc<32 * DG>(thold);
  if (r == 0) tc::mbar_init(mbar, 1);
  if (blockIdx.x == 0 && t < 8) reinterpret_cast<uint32_t*>(out + size_t(np) * 32)[t] = 0u;  // zero row
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tacc = *thold + uint32_t(32 * grp) + (uint32_t(32 * (r >> 5)) << 16);
  int32_t bs[32];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int4 b4 = reinterpret_cast<const int4*>(bias)[k];
    bs[4 * k] = b4.x, bs[4 * k + 1] = b4.y, bs[4 * k + 2] = b4.z, bs[4 * k + 3] = b4.w;
  }

  const uint32_t ntiles = (np + 127) / 128;
  const uint32_t stride = gridDim.x * DG;
  uint32_t tile = blockIdx.x * DG + grp;
  uint32_t phase = 0;
  // code and child start of row r of tile tl; EMB: the children's codes, packed (loaded
  // two tiles ahead with the rest, so the gather never waits on them)
  auto load = [&](uint32_t tl, uint32_t& xx, uint32_t& jj, uint64_t& cw) {
    const uint32_t p = tl * 128 + r;
    xx = 0u, jj = 0u, cw = 0ull;
    if (tl < ntiles && p < np) {
      xx = Xp[p], jj = cs[p];
      if (EMB) {
        const int nc = __popc(xx);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k < nc) cw |= uint64_t(Xc[jj + k]) << (8 * k);
      }
    }
  };
  auto gather = [&](uint32_t xx, uint32_t jj, uint64_t cw) {  // child rows into their K-slots of row r
    for (uint32_t m = xx; m; m &= m - 1u, ++jj, cw >>= 8) {
      const uint32_t c = __ffs(m) - 1;
      if (EMB) {  // from the shared-memory table (a 8 KB hot set would serialise in L2)
        const uint4* src = reinterpret_cast<const uint4*>(sm + SM_E + (uint32_t(cw & 0xffu) - 1u) * 32u);
        *reinterpret_cast<uint4*>(sA + c * 4096 + tc::kmaj_off(r, 0)) = src[0];
        *reinterpret_cast<uint4*>(sA + c * 4096 + tc::kmaj_off(r, 16)) = src[1];
      } else {
        cp16(sA + c * 4096 + tc::kmaj_off(r, 0), g + size_t(jj) * 32);
        cp16(sA + c * 4096 + tc::kmaj_off(r, 16), g + size_t(jj) * 32 + 16);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  uint32_t x, j0, xn, jn;
  uint64_t cw0, cwn;
  load(tile, x, j0, cw0);
  load(tile + stride, xn, jn, cwn);
  gather(x, j0, cw0);
  for (; tile < ntiles; tile += stride) {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    tc::fence_async_smem();
    tc::fence_before();
    bar_group(1 + grp);  // A tile complete (gathers + restored zeros), TMEM reads of the last tile done
    tc::fence_after();
    if (r == 0) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        tc::mma_i8(*thold + uint32_t(32 * grp), tc::sdesc(tc::smem_u32(sA + c * 4096)),
                   tc::sdesc(tc::smem_u32(sm + SM_B + c * 1024)), IDESC_DN, c > 0 ? 1u : 0u);
      tc::commit(mbar);
    }
    uint32_t x2, j2;
    uint64_t cw2;
    load(tile + 2 * stride, x2, j2, cw2);
    tc::mbar_wait(mbar, phase);
    phase ^= 1u;
    tc::fence_after();
    uint32_t acc[32];
    tc::tmem_ld32(tacc, acc);
    tc::tmem_wait_ld();
    // the MMAs have consumed the tile: zero the slots the next tile does not overwrite,
    // then start the next gather
    for (uint32_t m = x & ~xn; m; m &= m - 1u) {
      const uint32_t c = __ffs(m) - 1;
      *reinterpret_cast<uint4*>(sA + c * 4096 + tc::kmaj_off(r, 0)) = make_uint4(0u, 0u, 0u, 0u);
      *reinterpret_cast<uint4*>(sA + c * 4096 + tc::kmaj_off(r, 16)) = make_uint4(0u, 0u, 0u, 0u);
    }
    gather(xn, jn, cwn);
    const uint32_t p = tile * 128 + r;
    if (p < np) {
      uint32_t o4[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int32_t a0 = int32_t(acc[4 * k]) + bs[4 * k], a1 = int32_t(acc[4 * k + 1]) + bs[4 * k + 1];
        const int32_t a2 = int32_t(acc[4 * k + 2]) + bs[4 * k + 2], a3 = int32_t(acc[4 * k + 3]) + bs[4 * k + 3];
        if (SIGNED) {
          o4[k] = pack_sat4(rq_s(a0, rq), rq_s(a1, rq), rq_s(a2, rq), rq_s(a3, rq));
        } else {
          o4[k] = (uint32_t(rq8(a0, rq)) & 0xffu) | (uint32_t(rq8(a1, rq)) & 0xffu) << 8 |
                  (uint32_t(rq8(a2, rq)) & 0xffu) << 16 | (uint32_t(rq8(a3, rq)) & 0xffu) << 24;
        }
      }
      uint4* dst = reinterpret_cast<uint4*>(out + size_t(p) * 32);
      dst[0] = make_uint4(o4[0], o4[1], o4[2], o4[3]);
      dst[1] = make_uint4(o4[4], o4[5], o4[6], o4[7]);
    }
    x = xn, j0 = jn;
    xn = x2, jn = j2, cwn = cw2;
  }
  __syncthreads();
  if (t < 32) tc::tmem_dealloc<32 * DG>(*thold);
}

}  // namespace

void down_tc(pcc_ctx c, const int8_t* g, const uint8_t* Xp, const uint32_t* cs_p, uint32_t np, const DDown& L,
             int8_t* out, const uint8_t* Xc) {
  constexpr int smem = SM_END;  // ~136 KB: one CTA (four tile groups) per SM
  const uint32_t ntiles = (np + 127) / 128;
  const unsigned grid = std::max(1u, std::min((ntiles + DG - 1) / DG, unsigned(c->sm_count)));
  Prof p(c, "down", size_t(np) * (1 + 4 + 32));
#define PCC_DOWN(SG, EM)                                                                                 \
  do {                                                                                                   \
    PCC_SMEM_ATTR((k_down_tc<SG, EM>), smem);                                                            \
    k_down_tc<SG, EM><<<grid, DNT, smem, c->stream>>>(g, Xp, cs_p, np, L.W, L.b, L.rq, out, Xc);         \
  } while (0)
  if (L.rq.fast_s && Xc) PCC_DOWN(true, true);
  else if (L.rq.fast_s) PCC_DOWN(true, false);
  else if (Xc) PCC_DOWN(false, true);
  else PCC_DOWN(false, false);
#undef PCC_DOWN
  launched(c);
}

}  // namespace pcc
