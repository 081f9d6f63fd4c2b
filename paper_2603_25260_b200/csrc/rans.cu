// rans.cu — warp-interleaved rANS over the occupancy bytes (the paper entropy-codes X^l
// under p^l, without naming the coder; reading Q23/Q24: 32-bit state,
// L = 2^16, 16-bit words, M = 2^16, K <= 32 interleaved lanes per segment).
// One warp per segment; lane k owns symbols j = s*K + k.  Encoder runs steps in reverse
// and places each renormalisation word by ballot so the stream is in decoder order.
#include "pcc_internal.cuh"

namespace pcc {

namespace {

__device__ __forceinline__ int lanes_for(uint32_t n) {
  uint32_t k = (n + 2047u) / 2048u;
  return int(k < 1u ? 1u : (k > 32u ? 32u : k));
}

__global__ void __launch_bounds__(128) k_rans_enc(const EncSeg* __restrict__ segs, int nseg, const uint32_t* __restrict__ cf,
                                                  uint16_t* __restrict__ words, uint32_t* __restrict__ seg_W,
                                                  uint32_t* __restrict__ seg_state) {
  const int gw = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (gw >= nseg) return;
  const EncSeg sg = segs[gw];
  const uint32_t n = sg.n;
  const int K = lanes_for(n);
  const uint32_t steps = (n + uint32_t(K) - 1u) / uint32_t(K);
  uint32_t x = 1u << 16;
  uint32_t cnt = 0;
  uint16_t* end = words + sg.node + n;
  const unsigned above = ~((2u << lane) - 1u);  // lanes with a higher index
  for (uint32_t s = steps; s-- > 0;) {
    const uint32_t j = s * uint32_t(K) + uint32_t(lane);
    const bool act = lane < K && j < n;
    const uint32_t v = act ? cf[sg.node + j] : 0u;
    const uint32_t c = v & 0xffffu, f = v >> 16;
    const bool emit = act && x >= (f << 16);
    const unsigned m = __ballot_sync(0xffffffffu, emit);
    if (emit) {
      end[-1 - int(cnt + __popc(m & above))] = uint16_t(x & 0xffffu);
      x >>= 16;
    }
    cnt += __popc(m);
    if (act) x = ((x / f) << 16) + (x % f) + c;
  }
  if (lane == 0) seg_W[gw] = cnt;
  if (lane < K) seg_state[size_t(gw) * 32 + lane] = x;
}

__device__ __forceinline__ uint32_t ld_u32(const uint8_t* p) {
  return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
  const uint32_t s = uint32_t(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Decoder: one warp per segment (block = 1 warp), CDF rows of the K nodes of the next
// step prefetched into shared memory with cp.async (double buffer, 2 x 32 x 512 B).
__global__ void __launch_bounds__(32) k_rans_dec(const DecSeg* __restrict__ segs, int nseg, const uint8_t* __restrict__ bs,
                                                 const uint16_t* __restrict__ cdf, uint8_t* __restrict__ X,
                                                 uint32_t* __restrict__ err) {
  extern __shared__ __align__(16) uint16_t rows[];  // [2][32][256]
  const int gw = blockIdx.x;
  const int lane = threadIdx.x;
  if (gw >= nseg) return;
  const DecSeg sg = segs[gw];
  const uint8_t* lvl = bs + sg.byte;
  const uint32_t lvl_bytes = sg.level_bytes;
  // walk earlier (full, 65536-symbol, K = 32) chunks of this level payload
  uint32_t pos = 0;
  bool bad = false;
  for (uint32_t ch = 0; ch < sg.chunk && !bad; ++ch) {
    if (pos + 4 > lvl_bytes) { bad = true; break; }
    const uint32_t Wc = ld_u32(lvl + pos);
    const uint64_t sz = 4ull + 128ull + 4ull * ((uint64_t(Wc) + 1) / 2);
    if (pos + sz > lvl_bytes) { bad = true; break; }
    pos += uint32_t(sz);
  }
  const uint32_t n = sg.n;
  const int K = lanes_for(n);
  uint32_t W = 0;
  if (!bad) {
    if (uint64_t(pos) + 4 + 4 * K > lvl_bytes) bad = true;
    else {
      W = ld_u32(lvl + pos);
      const uint64_t sz = 4ull + 4ull * K + 4ull * ((uint64_t(W) + 1) / 2);
      if (W > n || pos + sz > lvl_bytes) bad = true;
      if (sg.last && pos + sz != lvl_bytes) bad = true;
    }
  }
  if (bad) {
    if (lane == 0) atomicOr(err, EF_CORRUPT);
    return;
  }
  uint32_t x = lane < K ? ld_u32(lvl + pos + 4 + 4 * lane) : (1u << 16);
  if (x < (1u << 16)) bad = true;
  const uint16_t* wp = reinterpret_cast<const uint16_t*>(lvl + pos + 4 + 4 * K);
  const uint32_t steps = (n + uint32_t(K) - 1u) / uint32_t(K);
  const uint16_t* base = cdf + size_t(sg.node) * 256;
  const unsigned lt = (1u << lane) - 1u;
  auto prefetch = [&](uint32_t s) {
    uint16_t* buf = rows + (s & 1u) * (32 * 256);
    for (int r = 0; r < K; ++r) {
      const uint32_t j = s * uint32_t(K) + uint32_t(r);
      if (j < n) cp_async16(buf + r * 256 + lane * 8, base + size_t(j) * 256 + lane * 8);
    }
    cp_commit();
  };
  prefetch(0);
  uint32_t used = 0;
  for (uint32_t s = 0; s < steps; ++s) {
    if (s + 1 < steps) {
      prefetch(s + 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncwarp();
    const uint32_t j = s * uint32_t(K) + uint32_t(lane);
    const bool act = lane < K && j < n;
    bool need = false;
    if (act) {
      const uint16_t* c = rows + (s & 1u) * (32 * 256) + lane * 256;
      const uint32_t slot = x & 0xffffu;
      int lo = 0, hi = NCODE - 1;
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int mid = (lo + hi + 1) >> 1;
        if (lo < hi) {
          if (uint32_t(c[mid]) <= slot) lo = mid; else hi = mid - 1;
        }
      }
      const uint32_t cum = c[lo];
      const uint32_t nxt = lo < NCODE - 1 ? uint32_t(c[lo + 1]) : 65536u;
      const uint32_t f = nxt - cum;
      X[sg.node + j] = uint8_t(lo + 1);
      x = f * (x >> 16) + slot - cum;
      need = x < (1u << 16);
    }
    const unsigned m = __ballot_sync(0xffffffffu, need);
    if (need) {
      const uint32_t wi = used + __popc(m & lt);
      if (wi < W) x = (x << 16) | uint32_t(wp[wi]);
      else bad = true;
    }
    used += __popc(m);
    __syncwarp();
  }
  if (used != W || (lane < K && x != (1u << 16))) bad = true;
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, EF_CORRUPT);
}

}  // namespace

void rans_encode(pcc_ctx c, const EncSeg* d_segs, int nseg, const uint32_t* cf, uint16_t* words, uint32_t* seg_W,
                 uint32_t* seg_state) {
  if (nseg == 0) return;
  const unsigned grid = unsigned((size_t(nseg) * 32 + 127) / 128);
  Prof p(c, "rans_enc", 0);
  k_rans_enc<<<grid, 128, 0, c->stream>>>(d_segs, nseg, cf, words, seg_W, seg_state);
  launched(c);
}

void rans_decode(pcc_ctx c, const DecSeg* d_segs, int nseg, const uint8_t* bs, const uint16_t* cdf, uint8_t* X,
                 uint32_t* err) {
  if (nseg == 0) return;
  const size_t smem = 2 * 32 * 256 * sizeof(uint16_t);
  static bool attr = false;
  if (!attr) {
    PCC_CUDA(cudaFuncSetAttribute(k_rans_dec, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  Prof p(c, "rans_dec", 0);
  k_rans_dec<<<nseg, 32, smem, c->stream>>>(d_segs, nseg, bs, cdf, X, err);
  launched(c);
}

}  // namespace pcc
