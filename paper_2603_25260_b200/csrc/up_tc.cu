// up_tc.cu — GRED re-sparsification (Upsampling + Pruning, Eq.6/9/11) on the
// 5th-generation tensor cores, C = 32.
//
// Upsampling is "a linear transformation followed by a PReLU activation, performing an
// 8x channel expansion" over Concat(S, X) (reading Q6: the one-hot half is the int32 row
// E[X] = q_one * W_X[:, X]); Pruning "discards features of unoccupied child nodes".
// Child-major, block-diagonal product on tcgen05.mma.kind::i8: a tile is 128 consecutive
// child rows j (M = 128, TMEM lane = child).  Row j of the A operand is the parent row
// S[par(j)] placed in K-slot c(j) = key(j) & 7 of an otherwise zero [128 x 256] tile, and
// B[o][32c + i] = W_S[32c + o][i], so D[j][o] = W_S[32c(j) + o] . S[par(j)] is exactly the
// kept block of the 8x expansion (N = 32, K = 256: eight MMAs).  Every lane of the
// epilogue owns one kept child and its 32 outputs (no lane idles on a pruned block); the
// one-hot half q_one * W_X[o][X] (reading Q6) is one dp4a per output against a transposed
// copy of W_X in smem, the bias a padded smem row; requant in the signed one-multiply
// form (rq.cuh) and two 16-byte stores of the child row j.  Four independent 128-thread
// tile groups per CTA (own A tile, TMEM accumulator, mbarrier, named barrier) overlap
// one another's gathers, MMAs and epilogues; within a group a software pipeline keeps
// the index loads three tiles and the code loads two tiles ahead of the epilogue.
#include "pcc_internal.cuh"
#include "rq.cuh"
#include "tc.cuh"

namespace pcc {

namespace {

constexpr int UG = 4;             // tile groups per CTA
constexpr int UNT = 128 * UG;     // threads per CTA (one per child row of each group's tile)
constexpr uint32_t IDESC_UP = tc::idesc_i8(128, 32);
constexpr int WXS = 272;          // W_X^T row stride (256 + 16: spreads rows over banks)
constexpr int BST = 36;           // bias row stride in int32 (32 + 4: distinct bank groups)

__device__ __forceinline__ void cp16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(tc::smem_u32(s)), "l"(g));
}
__device__ __forceinline__ void cp4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(tc::smem_u32(s)), "l"(g));
}
__device__ __forceinline__ void bar_group(int id) { asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory"); }

// smem: per group an A tile [128 x 256] (8 canonical slabs of 4 KB); B = 8 slabs [32 x 32];
// W_X^T [255][272] int8; bias [8][36] int32; mbarriers + TMEM holder
constexpr int SM_A = 0, SM_B = UG * 32768, SM_WX = SM_B + 8192, SM_BIAS = SM_WX + NCODE * WXS;
constexpr int SM_RING = SM_BIAS + 8 * BST * 4;  // per group [3 slots][par | key low word][128] u32
constexpr int SM_MBAR = SM_RING + UG * 3 * 256 * 4, SM_END = SM_MBAR + 8 * UG + 16;

template <bool SIGNED>
__global__ void __launch_bounds__(UNT, 1) k_up_tc(const int8_t* __restrict__ S, const uint8_t* __restrict__ Xp,
                                                  const uint32_t* __restrict__ par, const uint64_t* __restrict__ key,
                                                  uint32_t nc, const int8_t* __restrict__ WS,
                                                  const int8_t* __restrict__ WXt, const int32_t* __restrict__ bias,
                                                  int32_t q_one, RQ rq, int8_t* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int t = threadIdx.x, g = t >> 7, r = t & 127;  // group, child row of the tile (= TMEM lane)
  uint8_t* sA = sm + SM_A + g * 32768;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + SM_MBAR) + g;
  uint32_t* thold = reinterpret_cast<uint32_t*>(sm + SM_MBAR + 8 * UG);
  const int32_t* sbias = reinterpret_cast<const int32_t*>(sm + SM_BIAS);
  const int8_t* sWX = reinterpret_cast<const int8_t*>(sm + SM_WX);

  // B slab c, row o: W_S row 32c + o (two 16-byte chunks)
  for (int k = t; k < 512; k += UNT) {
    const int o = k >> 1, h = k & 1;
    *reinterpret_cast<uint4*>(sm + SM_B + (o >> 5) * 1024 + tc::kmaj_off(o & 31, 16 * h)) =
        reinterpret_cast<const uint4*>(WS)[k];
  }
  for (int k = t; k < NCODE * 16; k += UNT)  // W_X^T rows, 16 chunks each
    *reinterpret_cast<uint4*>(sm + SM_WX + (k >> 4) * WXS + 16 * (k & 15)) = reinterpret_cast<const uint4*>(WXt)[k];
  for (int k = t; k < 256; k += UNT) reinterpret_cast<int32_t*>(sm + SM_BIAS)[(k >> 5) * BST + (k & 31)] = bias[k];
  for (int k = t; k < UG * 32768 / 16; k += UNT) reinterpret_cast<uint4*>(sm + SM_A)[k] = make_uint4(0u, 0u, 0u, 0u);
  if (t < 32) tc::tmem_alloc<32 * UG>(thold);
  if (r == 0) tc::mbar_init(mbar, 1);
  if (blockIdx.x == 0 && t < 8) reinterpret_cast<uint32_t*>(out + size_t(nc) * 32)[t] = 0u;  // zero row
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tacc = *thold + uint32_t(32 * g) + (uint32_t(32 * (r >> 5)) << 16);

  // one-hot masks for dp4a: byte b of qm[b] = q_one
  const int32_t qm0 = q_one & 0xff, qm1 = qm0 << 8, qm2 = qm0 << 16, qm3 = int32_t(uint32_t(qm0) << 24);
  const uint32_t ntiles = (nc + 127) / 128;
  const uint32_t stride = gridDim.x * UG;
  uint32_t tile = blockIdx.x * UG + g;
  uint32_t phase = 0;
  // Software pipeline per thread (row r of its group's tiles T, T+s, T+2s, ...): the
  // indices par/key of tile T+3s are copied (cp.async) into a 3-slot ring while tile T is
  // processed, the parent code X of tile T+2s is loaded into a register, and the gather of
  // tile T+s is in flight during the epilogue of T.  Each thread reads only its own ring
  // entries, so the ring needs no barrier.
  uint32_t* ring = reinterpret_cast<uint32_t*>(sm + SM_RING) + g * 768;
  auto valid = [&](uint32_t tl) { return tl < ntiles && tl * 128 + r < nc; };
  auto idx_load = [&](uint32_t tl, int slot) {
    if (valid(tl)) {
      cp4(ring + slot * 256 + r, par + tl * 128 + r);
      cp4(ring + slot * 256 + 128 + r, reinterpret_cast<const uint32_t*>(key + tl * 128 + r));
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  auto gather = [&](uint32_t pp, uint32_t c_) {  // the parent row into K-slot c_ of row r
    cp16(sA + c_ * 4096 + tc::kmaj_off(r, 0), S + size_t(pp) * 32);
    cp16(sA + c_ * 4096 + tc::kmaj_off(r, 16), S + size_t(pp) * 32 + 16);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  idx_load(tile, 0);
  idx_load(tile + stride, 1);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  bool v = valid(tile), vn = valid(tile + stride);
  uint32_t cc = v ? (ring[128 + r] & 7u) : 0u, x = v ? uint32_t(Xp[ring[r]]) : 0u;
  uint32_t cn = vn ? (ring[256 + 128 + r] & 7u) : 0u, xn = vn ? uint32_t(Xp[ring[256 + r]]) : 0u;
  if (v) gather(ring[r], cc);
  idx_load(tile + 2 * stride, 2);
  int slot = 0;
  for (; tile < ntiles; tile += stride) {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    tc::fence_async_smem();
    tc::fence_before();
    bar_group(1 + g);  // A tile complete (gathers + restored zeros), TMEM reads of the last tile done
    tc::fence_after();
    if (r == 0) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        tc::mma_i8(*thold + uint32_t(32 * g), tc::sdesc(tc::smem_u32(sA + c * 4096)),
                   tc::sdesc(tc::smem_u32(sm + SM_B + c * 1024)), IDESC_UP, c > 0 ? 1u : 0u);
      tc::commit(mbar);
    }
    const int s1 = slot == 2 ? 0 : slot + 1, s2 = s1 == 2 ? 0 : s1 + 1;
    // tile T+2s: indices landed (waited above) -> its code; then tile T+3s's indices into T's slot
    const bool v2 = valid(tile + 2 * stride);
    const uint32_t c2 = v2 ? (ring[s2 * 256 + 128 + r] & 7u) : 0u;
    const uint32_t x2 = v2 ? uint32_t(Xp[ring[s2 * 256 + r]]) : 0u;
    idx_load(tile + 3 * stride, slot);
    tc::mbar_wait(mbar, phase);
    phase ^= 1u;
    tc::fence_after();
    uint32_t acc[32];
    tc::tmem_ld32(tacc, acc);
    tc::tmem_wait_ld();
    // the MMAs have consumed the tile: restore the zero slot, start the next gather
    if (v && !(vn && cn == cc)) {
      *reinterpret_cast<uint4*>(sA + cc * 4096 + tc::kmaj_off(r, 0)) = make_uint4(0u, 0u, 0u, 0u);
      *reinterpret_cast<uint4*>(sA + cc * 4096 + tc::kmaj_off(r, 16)) = make_uint4(0u, 0u, 0u, 0u);
    }
    if (vn) gather(ring[s1 * 256 + r], cn);
    if (v) {
      const uint4* wx4 = reinterpret_cast<const uint4*>(sWX + (x - 1) * WXS + 32 * cc);
      const uint4 wa = wx4[0], wb = wx4[1];
      const uint32_t wxw[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
      const int4* b4 = reinterpret_cast<const int4*>(sbias + cc * BST);
      uint32_t o4[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int4 bb = b4[k];
        int32_t a0 = __dp4a(int32_t(wxw[k]), qm0, int32_t(acc[4 * k]) + bb.x);
        int32_t a1 = __dp4a(int32_t(wxw[k]), qm1, int32_t(acc[4 * k + 1]) + bb.y);
        int32_t a2 = __dp4a(int32_t(wxw[k]), qm2, int32_t(acc[4 * k + 2]) + bb.z);
        int32_t a3 = __dp4a(int32_t(wxw[k]), qm3, int32_t(acc[4 * k + 3]) + bb.w);
        if (SIGNED) {
          o4[k] = pack_sat4(rq_s(a0, rq), rq_s(a1, rq), rq_s(a2, rq), rq_s(a3, rq));
        } else {
          o4[k] = (uint32_t(rq8(a0, rq)) & 0xffu) | (uint32_t(rq8(a1, rq)) & 0xffu) << 8 |
                  (uint32_t(rq8(a2, rq)) & 0xffu) << 16 | (uint32_t(rq8(a3, rq)) & 0xffu) << 24;
        }
      }
      uint4* dst = reinterpret_cast<uint4*>(out + size_t(tile * 128 + r) * 32);
      dst[0] = make_uint4(o4[0], o4[1], o4[2], o4[3]);
      dst[1] = make_uint4(o4[4], o4[5], o4[6], o4[7]);
    }
    v = vn, cc = cn, x = xn;
    vn = v2, cn = c2, xn = x2;
    slot = s1;
  }
  __syncthreads();
  if (t < 32) tc::tmem_dealloc<32 * UG>(*thold);
}

}  // namespace

void up_prune_tc(pcc_ctx c, const int8_t* S, const uint8_t* Xp, const uint32_t* par_c, const uint64_t* key_c,
                 uint32_t nc, const DUp& L, int8_t* out) {
  constexpr int smem = SM_END;  // ~207 KB: one CTA (four tile groups) per SM
  PCC_SMEM_ATTR(k_up_tc<true>, smem);
  PCC_SMEM_ATTR(k_up_tc<false>, smem);
  const uint32_t ntiles = (nc + 127) / 128;
  const unsigned grid = std::max(1u, std::min((ntiles + UG - 1) / UG, unsigned(c->sm_count)));
  Prof p(c, "up", size_t(nc) * (4 + 8 + 2 * 32));
  if (L.rq.fast_s)
    k_up_tc<true><<<grid, UNT, smem, c->stream>>>(S, Xp, par_c, key_c, nc, L.W, L.WXt, L.b, L.q_one, L.rq, out);
  else
    k_up_tc<false><<<grid, UNT, smem, c->stream>>>(S, Xp, par_c, key_c, nc, L.W, L.WXt, L.b, L.q_one, L.rq, out);
  launched(c);
}

}  // namespace pcc
