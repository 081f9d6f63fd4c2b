// rans.cu — warp-interleaved rANS over the occupancy bytes (the paper entropy-codes X^l
// under p^l, without naming the coder; reading Q23/Q24: 32-bit state,
// L = 2^16, 16-bit words, M = 2^16, K <= 32 interleaved lanes per segment).
// One warp per segment; lane k owns symbols j = s*K + k.  Encoder runs steps in reverse
// and places each renormalisation word by ballot so the stream is in decoder order.
#include "pcc_internal.cuh"
#include "tc.cuh"

namespace pcc {

namespace {

__device__ __forceinline__ int lanes_for(uint32_t n) {
  uint32_t k = (n + 511u) / 512u;
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

// Decoder: one warp per segment (block = 1 warp).  The CDF rows of the K nodes of a step
// do not depend on the rANS state, so they are prefetched DEC_STAGES steps ahead into
// shared memory with TMA bulk copies; the renormalisation words are consumed in stream order
// and are held in a 96-word register window (three words per lane) refilled 64 words
// ahead, so no step waits on a dependent global load.  DEC_STAGES = 2 by default (more
// resident CTAs per SM beat deeper prefetch on the bandwidth-bound levels).
template <int DEC_STAGES>
__global__ void __launch_bounds__(32) k_rans_dec(const DecSeg* __restrict__ segs, int nseg, const uint8_t* __restrict__ bs,
                                                 const uint16_t* __restrict__ cdf, const uint32_t* __restrict__ lut,
                                                 uint8_t* __restrict__ X, uint32_t* __restrict__ err, int stage_rows) {
  extern __shared__ __align__(128) uint16_t rows[];  // [DEC_STAGES][stage_rows][DROW_U16]
  __shared__ __align__(8) uint64_t dec_mbar[DEC_STAGES];
  __shared__ uint32_t slut[1025];  // the model's exp table, slut[1024] = 0 (delta >= 4096)
  const int gw = blockIdx.x;
  const int lane = threadIdx.x;
  if (gw >= nseg) return;
  for (int k = lane; k < 1024; k += 32) slut[k] = lut[k];
  if (lane == 0) slut[1024] = 0u;
  __syncwarp();
  const DecSeg sg = segs[gw];
  const uint8_t* lvl = bs + sg.byte;
  const uint32_t lvl_bytes = sg.level_bytes;
  // walk earlier (full, 16384-symbol, K = 32) chunks of this level payload
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
  if (bad || K > stage_rows) {
    if (lane == 0) atomicOr(err, EF_CORRUPT);
    return;
  }
  uint32_t x = lane < K ? ld_u32(lvl + pos + 4 + 4 * lane) : (1u << 16);
  if (x < (1u << 16)) bad = true;
  const uint16_t* wp = reinterpret_cast<const uint16_t*>(lvl + pos + 4 + 4 * K);
  auto ldw = [&](uint32_t k) -> uint32_t { return k < W ? uint32_t(wp[k]) : 0u; };
  uint32_t wbase = 0;  // window = words [wbase, wbase + 96)
  uint32_t w0 = ldw(lane), w1 = ldw(32 + lane), w2 = ldw(64 + lane);
  const uint32_t steps = (n + uint32_t(K) - 1u) / uint32_t(K);
  const uint16_t* base = cdf + size_t(sg.node) * DROW_U16;
  const unsigned lt = (1u << lane) - 1u;
  // The K rows of a step are contiguous (nodes s*K .. s*K+K-1): one TMA bulk copy per
  // step, issued by lane 0, completing on that stage's mbarrier.
  if (lane == 0)
    for (int st = 0; st < DEC_STAGES; ++st) tc::mbar_init(&dec_mbar[st], 1);
  __syncwarp();
  auto prefetch = [&](uint32_t s) {
    if (lane == 0 && s < steps) {
      const uint32_t j0 = s * uint32_t(K);
      const uint32_t nr = (n - j0) < uint32_t(K) ? (n - j0) : uint32_t(K);
      uint64_t* mb = &dec_mbar[s % DEC_STAGES];
      tc::mbar_expect_tx(mb, nr * uint32_t(DROW_BYTES));
      tc::bulk_g2s(rows + size_t(s % DEC_STAGES) * stage_rows * DROW_U16, base + size_t(j0) * DROW_U16,
                   nr * uint32_t(DROW_BYTES), mb);
    }
  };
#pragma unroll
  for (int p = 0; p < DEC_STAGES - 1; ++p) prefetch(uint32_t(p));
  uint32_t used = 0;
  for (uint32_t s = 0; s < steps; ++s) {
    prefetch(s + DEC_STAGES - 1);
    tc::mbar_wait(&dec_mbar[s % DEC_STAGES], (s / DEC_STAGES) & 1u);
    const uint32_t j = s * uint32_t(K) + uint32_t(lane);
    const bool act = lane < K && j < n;
    bool need = false;
    if (act) {
      const uint16_t* rw = rows + size_t(s % DEC_STAGES) * stage_rows * DROW_U16 + lane * DROW_U16;
      const uint32_t* hd = reinterpret_cast<const uint32_t*>(rw);
      const uint16_t* jx = rw + DROW_HDR / 2;
      const uint32_t slot = x & 0xffffu;
      const uint32_t S = hd[0], inv32 = hd[1];
      // C_i <= slot  <=>  i <= slot and E_i * 65281 < (slot - i + 1) * S (exact, 64-bit);
      // C_i is non-decreasing in i, so the block is the number of true coarse tests
      const uint64_t sS = uint64_t(S);
      int blk = 0;
#pragma unroll
      for (int k = 1; k < 16; ++k) {
        const uint32_t i = 16u * uint32_t(k);
        blk += (i <= slot && uint64_t(hd[1 + k]) * 65281ull < uint64_t(slot - i + 1u) * sS) ? 1 : 0;
      }
      // inside the block: its 16 LUT indices in two 16-byte loads, the 16 exponentials as
      // independent loads, then the running prefix and one exact test per symbol
      const uint4* jq = reinterpret_cast<const uint4*>(jx + 16 * blk);
      const uint4 ja = jq[0], jb = jq[1];
      const uint32_t jw[8] = {ja.x, ja.y, ja.z, ja.w, jb.x, jb.y, jb.z, jb.w};
      uint32_t ev[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) ev[t] = slut[(jw[t >> 1] >> (16 * (t & 1))) & 0xffffu];
      const uint32_t E0 = blk ? hd[1 + blk] : 0u;
      uint32_t Er = E0, Elo = E0, elo = ev[0];
      int cnt = 0;
#pragma unroll
      for (int t = 0; t < 15; ++t) {
        Er += ev[t];  // E_{16 blk + t + 1}
        const uint32_t i1 = uint32_t(16 * blk + t + 1);
        if (i1 < uint32_t(NCODE) && i1 <= slot && uint64_t(Er) * 65281ull < uint64_t(slot - i1 + 1u) * sS) {
          cnt = t + 1;
          Elo = Er;
          elo = ev[t + 1];
        }
      }
      const int lo = 16 * blk + cnt;
      // C_lo and C_{lo+1} exactly: q = floor(E K / S) from the 32-bit reciprocal estimate
      auto fl = [&](uint32_t Ev) -> uint32_t {
        const uint32_t qt = __umulhi(Ev, inv32);
        return qt + ((uint64_t(Ev) * 65281ull - uint64_t(qt) * sS) >= sS ? 1u : 0u);
      };
      const uint32_t cum = uint32_t(lo) + fl(Elo);
      const uint32_t nxt = lo < NCODE - 1 ? uint32_t(lo + 1) + fl(Elo + elo) : 65536u;
      const uint32_t f = nxt - cum;
      X[sg.node + j] = uint8_t(lo + 1);
      x = f * (x >> 16) + slot - cum;
      need = x < (1u << 16);
    }
    const unsigned m = __ballot_sync(0xffffffffu, need);
    const uint32_t off = used + __popc(m & lt) - wbase;  // < 64 + 32 since used - wbase < 32
    const uint32_t v0 = __shfl_sync(0xffffffffu, w0, off & 31);
    const uint32_t v1 = __shfl_sync(0xffffffffu, w1, off & 31);
    const uint32_t v2 = __shfl_sync(0xffffffffu, w2, off & 31);
    if (need) {
      if (used + __popc(m & lt) < W) x = (x << 16) | (off < 32 ? v0 : (off < 64 ? v1 : v2));
      else bad = true;
    }
    used += __popc(m);
    if (used - wbase >= 32) {  // slide the window by 32 words, load 64 ahead
      wbase += 32;
      w0 = w1;
      w1 = w2;
      w2 = ldw(wbase + 64 + lane);
    }
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

void rans_decode(pcc_ctx c, const DecSeg* d_segs, int nseg, const uint8_t* bs, const uint16_t* cdf,
                 const uint32_t* lut, uint8_t* X, uint32_t* err, int max_lanes, size_t nsym) {
  if (nseg == 0) return;
  const int stage_rows = max_lanes <= 8 ? 8 : (max_lanes <= 16 ? 16 : 32);
  PCC_SMEM_ATTR(k_rans_dec<2>, 2 * 32 * DROW_BYTES);
  PCC_SMEM_ATTR(k_rans_dec<3>, 3 * 32 * DROW_BYTES);
  PCC_SMEM_ATTR(k_rans_dec<4>, 4 * 32 * DROW_BYTES);
  // two stages: measured best on the B = 256 bench (2.55 ms vs 2.87 / 3.02 ms per step for
  // 3 / 4 stages): the decode is bandwidth-bound on the largest levels, where more CTAs
  // resident per SM beat deeper prefetch
  int st = 2;
  static const int forced = [] {
    const char* e = getenv("PCC_DEC_STAGES");  // development override (2..4)
    return e ? atoi(e) : 0;
  }();
  if (forced >= 2 && forced <= 4) st = forced;
  const size_t smem = size_t(st) * stage_rows * DROW_BYTES;
  Prof p(c, "rans_dec", nsym * (DROW_BYTES + 2));  // algorithmic: the row + one word per symbol
  if (st == 4) k_rans_dec<4><<<nseg, 32, smem, c->stream>>>(d_segs, nseg, bs, cdf, lut, X, err, stage_rows);
  else if (st == 3) k_rans_dec<3><<<nseg, 32, smem, c->stream>>>(d_segs, nseg, bs, cdf, lut, X, err, stage_rows);
  else k_rans_dec<2><<<nseg, 32, smem, c->stream>>>(d_segs, nseg, bs, cdf, lut, X, err, stage_rows);
  launched(c);
}

}  // namespace pcc
