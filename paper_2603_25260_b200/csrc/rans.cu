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

// Decoder rows carry S, 65281 * 2^32 / S, the maximum logit mu, the 15 block prefix masses
// and the node's hidden activations a (pcc_internal.cuh DROW_*).  The decoder recomputes
// the 16 logits of the one 16-symbol block its coarse test selects from a and the level's
// W2 / b2 held in shared memory (exact int32 dp4a), so a node costs 112 bytes of HBM
// instead of a full CDF row.  Shared-memory layouts keep a warp's 16 possible blocks on
// distinct bank groups (<= 2-way conflicts): W2 row i (32 bytes, zero padded beyond H) is
// two 16-byte chunks, chunk (i, h) at slot 8 (i >> 2) + ((2 (i & 3) + h + (i >> 4)) & 7);
// b2 of block blk is four 16-byte chunks, chunk c at 4 blk + ((c + (blk >> 1)) & 3).
__device__ __forceinline__ uint32_t w2_slot(uint32_t i, uint32_t h) {
  return ((i >> 2) << 3) + ((2u * (i & 3u) + h + (i >> 4)) & 7u);
}
__device__ __forceinline__ uint32_t b2_slot(uint32_t blk, uint32_t c) { return blk * 4u + ((c + (blk >> 1)) & 3u); }

// One warp per segment, DEC_WPC segments per CTA sharing the level's W2 / b2 / exp table.
// The rows of the K nodes of a step do not depend on the rANS state, so they are
// prefetched a step ahead into shared memory by TMA bulk copies (2 stages per warp, one
// mbarrier each); the renormalisation words are consumed in stream order from a 96-word
// register window (three words per lane) refilled 64 words ahead.
constexpr int DEC_WPC = 4;

template <int H, bool SAT>
__global__ void __launch_bounds__(32 * DEC_WPC) k_rans_dec(const DecSeg* __restrict__ segs, int nseg,
                                                          const uint8_t* __restrict__ bs, const uint8_t* __restrict__ rowsg,
                                                          const int8_t* __restrict__ W2, const int32_t* __restrict__ b2,
                                                          RQ rql, int32_t zsat_lo, int32_t zsat_hi,
                                                          const uint32_t* __restrict__ lut, uint8_t* __restrict__ X,
                                                          uint32_t* __restrict__ err, int stage_rows) {
  extern __shared__ __align__(128) uint8_t dsm[];  // [DEC_WPC][2][stage_rows][DROW_BYTES]
  __shared__ uint4 w2s[512];
  __shared__ uint4 b2s[64];
  __shared__ uint32_t slut[1025];  // the model's exp table, slut[1024] = 0 (delta >= 4096)
  __shared__ __align__(8) uint64_t dec_mbar[DEC_WPC][2];
  constexpr int HW = H / 4;
  for (int k = threadIdx.x; k < 512; k += blockDim.x) {
    const uint32_t i = uint32_t(k) >> 1, h = uint32_t(k) & 1u;
    uint32_t wv[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const uint32_t wi = 4u * h + uint32_t(w);  // word of the 32-byte row
      wv[w] = wi < uint32_t(HW) ? reinterpret_cast<const uint32_t*>(W2)[i * HW + wi] : 0u;
    }
    w2s[w2_slot(i, h)] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
  for (int k = threadIdx.x; k < 64; k += blockDim.x) {
    const uint32_t blk = uint32_t(k) >> 2, c = uint32_t(k) & 3u;
    b2s[b2_slot(blk, c)] = reinterpret_cast<const uint4*>(b2)[k];  // b2[16 blk + 4c .. +3]
  }
  for (int k = threadIdx.x; k < 1024; k += blockDim.x) slut[k] = lut[k];
  if (threadIdx.x == 0) slut[1024] = 0u;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * DEC_WPC + warp;
  if (gw >= nseg) return;
  uint8_t* stage = dsm + size_t(warp) * 2 * stage_rows * DROW_BYTES;
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
  const uint8_t* base = rowsg + size_t(sg.node) * DROW_BYTES;
  const unsigned lt = (1u << lane) - 1u;
  // The K rows of a step are contiguous (nodes s*K .. s*K+K-1): one TMA bulk copy per
  // step, issued by lane 0, completing on that stage's mbarrier.
  if (lane == 0) {
    tc::mbar_init(&dec_mbar[warp][0], 1);
    tc::mbar_init(&dec_mbar[warp][1], 1);
  }
  __syncwarp();
  auto prefetch = [&](uint32_t s) {
    if (lane == 0 && s < steps) {
      const uint32_t j0 = s * uint32_t(K);
      const uint32_t nr = (n - j0) < uint32_t(K) ? (n - j0) : uint32_t(K);
      uint64_t* mb = &dec_mbar[warp][s & 1u];
      tc::mbar_expect_tx(mb, nr * uint32_t(DROW_BYTES));
      tc::bulk_g2s(stage + size_t(s & 1u) * stage_rows * DROW_BYTES, base + size_t(j0) * DROW_BYTES,
                   nr * uint32_t(DROW_BYTES), mb);
    }
  };
  prefetch(0);
  const int64_t lhalf = rql.r > 0 ? (int64_t(1) << (rql.r - 1)) : 0;
  const bool fastl = !SAT && rql.fast_s;
  const int32_t nM = -rql.Sp;
  uint32_t used = 0;
  for (uint32_t s = 0; s < steps; ++s) {
    prefetch(s + 1);
    tc::mbar_wait(&dec_mbar[warp][s & 1u], (s >> 1) & 1u);
    const uint32_t j = s * uint32_t(K) + uint32_t(lane);
    const bool act = lane < K && j < n;
    bool need = false;
    if (act) {
      const uint8_t* rw = stage + size_t(s & 1u) * stage_rows * DROW_BYTES + lane * DROW_BYTES;
      const uint32_t* hd = reinterpret_cast<const uint32_t*>(rw);
      const uint32_t slot = x & 0xffffu;
      const uint32_t S = hd[0], inv32 = hd[1];
      const int32_t mu = int32_t(hd[2]);
      // C_i <= slot  <=>  i <= slot and E_i * 65281 < (slot - i + 1) * S (exact, 64-bit);
      // C_i is non-decreasing in i, so the block is the number of true coarse tests
      const uint64_t sS = uint64_t(S);
      int blk = 0;
#pragma unroll
      for (int k = 1; k < 16; ++k) {
        const uint32_t i = 16u * uint32_t(k);
        blk += (i <= slot && uint64_t(hd[2 + k]) * 65281ull < uint64_t(slot - i + 1u) * sS) ? 1 : 0;
      }
      // the block's 16 logits z_i = b2_i + a . W2_i (Eq.7), Q8 requant, delta = mu - l_i,
      // e_i = LUT[delta >> 2] (0 beyond 16 nats; i = 255 is not a symbol)
      const uint4 a0 = reinterpret_cast<const uint4*>(rw + DROW_A)[0];
      const uint4 a1 = reinterpret_cast<const uint4*>(rw + DROW_A)[1];
      const uint32_t aw[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const int64_t C2 = (int64_t(mu) << 32) + 0x7fffffff;
      uint32_t ev[16];
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const uint4 bb = b2s[b2_slot(uint32_t(blk), uint32_t(c4))];
        const uint32_t bv[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = 4 * c4 + u;
          const uint32_t i = uint32_t(16 * blk + t);
          const uint4 q0 = w2s[w2_slot(i, 0)];
          int32_t z = int32_t(bv[u]);
          z = __dp4a(int32_t(aw[0]), int32_t(q0.x), z);
          z = __dp4a(int32_t(aw[1]), int32_t(q0.y), z);
          if (HW > 2) {
            z = __dp4a(int32_t(aw[2]), int32_t(q0.z), z);
            z = __dp4a(int32_t(aw[3]), int32_t(q0.w), z);
          }
          if (HW > 4) {
            const uint4 q1 = w2s[w2_slot(i, 1)];
            z = __dp4a(int32_t(aw[4]), int32_t(q1.x), z);
            z = __dp4a(int32_t(aw[5]), int32_t(q1.y), z);
            z = __dp4a(int32_t(aw[6]), int32_t(q1.z), z);
            z = __dp4a(int32_t(aw[7]), int32_t(q1.w), z);
          }
          uint32_t dl;
          if (fastl) {
            dl = uint32_t(int32_t((int64_t(z) * nM + C2) >> 32));
          } else {
            int64_t lv = (int64_t(z) * int64_t(rql.mp) + lhalf) >> rql.r;
            if (SAT) {
              lv = z > zsat_hi ? (int64_t(1) << 24) : lv;
              lv = z < zsat_lo ? -(int64_t(1) << 24) : lv;
            }
            dl = uint32_t(mu - int32_t(lv));
          }
          ev[t] = i < uint32_t(NCODE) ? slut[min(dl, 4096u) >> 2] : 0u;
        }
      }
      const uint32_t E0 = blk ? hd[2 + blk] : 0u;
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

void rans_decode(pcc_ctx c, const DecSeg* d_segs, int nseg, const uint8_t* bs, const uint16_t* rows, int H,
                 const DHead& hd, const uint32_t* lut, uint8_t* X, uint32_t* err, int max_lanes, size_t nsym) {
  if (nseg == 0) return;
  const int stage_rows = max_lanes <= 8 ? 8 : (max_lanes <= 16 ? 16 : 32);
  const size_t smem = size_t(DEC_WPC) * 2 * stage_rows * DROW_BYTES;
  // the attribute is set once per device: to the largest launch (32 rows per stage)
  constexpr size_t smem_max = size_t(DEC_WPC) * 2 * 32 * DROW_BYTES;
  const unsigned grid = unsigned((nseg + DEC_WPC - 1) / DEC_WPC);
  // algorithmic bytes: the 112-byte row and one 16-bit word per symbol
  Prof p(c, "rans_dec", nsym * (DROW_BYTES + 2));
#define PCC_DEC(HH, SS)                                                                                         \
  if (H == HH && hd.can_saturate == SS) {                                                                      \
    PCC_SMEM_ATTR((k_rans_dec<HH, SS>), smem_max);                                                             \
    k_rans_dec<HH, SS><<<grid, 32 * DEC_WPC, smem, c->stream>>>(d_segs, nseg, bs,                              \
                                                                reinterpret_cast<const uint8_t*>(rows), hd.W2, \
                                                                hd.b2, hd.rql, hd.zsat_lo, hd.zsat_hi, lut, X, \
                                                                err, stage_rows);                              \
    launched(c);                                                                                               \
    return;                                                                                                    \
  }
  PCC_DEC(8, false)
  PCC_DEC(8, true)
  PCC_DEC(16, false)
  PCC_DEC(16, true)
  PCC_DEC(32, false)
  PCC_DEC(32, true)
#undef PCC_DEC
  throw Error{PCC_ERR_INVALID_ARG};
}

}  // namespace pcc
