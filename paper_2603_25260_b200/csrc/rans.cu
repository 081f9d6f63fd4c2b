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
// two 16-byte chunks, chunk (i, h) at slot 32 (i >> 4) + 8 ((i >> 2) & 3) + ((2 (i & 3) +
// h + (i >> 4)) & 7); b2 of block blk is four 16-byte chunks, chunk c at 4 blk + ((c +
// (blk >> 1)) & 3).
__device__ __forceinline__ uint32_t w2_slot(uint32_t i, uint32_t h) {
  return ((i >> 2) << 3) + ((2u * (i & 3u) + h + (i >> 4)) & 7u);
}
__device__ __forceinline__ uint32_t b2_slot(uint32_t blk, uint32_t c) { return blk * 4u + ((c + (blk >> 1)) & 3u); }

// Lane groups: a level's segments have K <= G lanes (G = the power of two >= the level's
// largest K), so a warp decodes 32 / G segments side by side — each group of G lanes is a
// mini-warp with its own state, word stream and 3G-word register window — and a level of
// short per-frame segments (K = 1..8) does not leave 31..24 lanes of every warp idle.
// Each lane prefetches its own node's row DEC_STAGES - 1 steps ahead with cp.async into its
// private stage slot (no cross-lane hand-off, no barrier).  DEC_WPC warps per CTA share
// the level's W2 / b2 / exp table.
constexpr int DEC_WPC = 4, DEC_STAGES = 3;

// LQ: the Q8 logit l(z) and delta = mu - l(z) (Eq.15, reading Q20): 0 = the signed
// one-multiply form (RQ::fast_s; the model cannot saturate), 1 = generic 64-bit shift,
// 2 = generic with the +-2^24 clamp.
template <int H, int LQ>
__global__ void __launch_bounds__(32 * DEC_WPC) k_rans_dec(const DecSeg* __restrict__ segs, int nseg, int lg,
                                                          const uint8_t* __restrict__ bs, const uint8_t* __restrict__ rowsg,
                                                          const int8_t* __restrict__ W2, const int32_t* __restrict__ b2,
                                                          RQ rql, int32_t zsat_lo, int32_t zsat_hi,
                                                          const uint32_t* __restrict__ lut, uint8_t* __restrict__ X,
                                                          uint32_t* __restrict__ err) {
  extern __shared__ __align__(128) uint8_t dsm[];  // [DEC_WPC][DEC_STAGES][32 lanes][DROW_BYTES]
  __shared__ uint4 w2s[512];
  __shared__ uint4 b2s[64];
  __shared__ uint32_t slut[1025];  // the model's exp table, slut[1024] = 0 (delta >= 4096)
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
  const int G = 1 << lg, g = lane >> lg, gl = lane & (G - 1);
  const unsigned gmask = lg == 5 ? 0xffffffffu : ((1u << G) - 1u);
  const unsigned ltg = (1u << gl) - 1u;  // lanes of the group below this one
  const int gw = (blockIdx.x * DEC_WPC + warp) * (32 >> lg) + g;  // this group's segment
  if ((blockIdx.x * DEC_WPC + warp) * (32 >> lg) >= nseg) return;  // whole warp idle
  uint8_t* slot = dsm + (size_t(warp) * DEC_STAGES * 32 + lane) * DROW_BYTES;  // stage st at + st*32*DROW_BYTES
  bool bad = false;
  uint32_t n = 0, W = 0, K = 1, pos = 0, node = 0;
  const uint8_t* lvl = nullptr;
  if (gw < nseg) {
    const DecSeg sg = segs[gw];
    lvl = bs + sg.byte;
    const uint32_t lvl_bytes = sg.level_bytes;
    n = sg.n;
    node = sg.node;
    K = uint32_t(lanes_for(n));
    // walk earlier (full, 16384-symbol, K = 32) chunks of this level payload
    for (uint32_t ch = 0; ch < sg.chunk && !bad; ++ch) {
      if (pos + 4 > lvl_bytes) { bad = true; break; }
      const uint32_t Wc = ld_u32(lvl + pos);
      const uint64_t sz = 4ull + 128ull + 4ull * ((uint64_t(Wc) + 1) / 2);
      if (pos + sz > lvl_bytes) { bad = true; break; }
      pos += uint32_t(sz);
    }
    if (!bad) {
      if (uint64_t(pos) + 4 + 4 * K > lvl_bytes) bad = true;
      else {
        W = ld_u32(lvl + pos);
        const uint64_t sz = 4ull + 4ull * K + 4ull * ((uint64_t(W) + 1) / 2);
        if (W > n || pos + sz > lvl_bytes) bad = true;
        if (sg.last && pos + sz != lvl_bytes) bad = true;
      }
    }
    if (K > uint32_t(G)) bad = true;
  }
  uint32_t x = 1u << 16;
  if (!bad && gw < nseg && uint32_t(gl) < K) {
    x = ld_u32(lvl + pos + 4 + 4 * gl);
    if (x < (1u << 16)) bad = true;
  }
  const uint32_t steps = (bad || gw >= nseg) ? 0u : (n + K - 1u) / K;
  const uint16_t* wp = lvl ? reinterpret_cast<const uint16_t*>(lvl + pos + 4 + 4 * K) : nullptr;
  auto ldw = [&](uint32_t k) -> uint32_t { return k < W ? uint32_t(wp[k]) : 0u; };
  uint32_t wbase = 0;  // the group's window = words [wbase, wbase + 3G)
  uint32_t w0 = steps ? ldw(gl) : 0u, w1 = steps ? ldw(G + gl) : 0u, w2 = steps ? ldw(2 * G + gl) : 0u;
  const uint8_t* rbase = rowsg + (size_t(node) + gl) * DROW_BYTES;
  auto prefetch = [&](uint32_t st) {  // this lane's row of step st into stage st % DEC_STAGES
    if (st < steps && st * K + gl < n && uint32_t(gl) < K) {
      const uint8_t* src = rbase + size_t(st) * K * DROW_BYTES;
      const uint32_t dst = tc::smem_u32(slot + (st % DEC_STAGES) * 32 * DROW_BYTES);
#pragma unroll
      for (int c16 = 0; c16 < DROW_BYTES / 16; ++c16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 16 * c16), "l"(src + 16 * c16));
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
#pragma unroll
  for (int p = 0; p < DEC_STAGES - 1; ++p) prefetch(uint32_t(p));
  const uint32_t steps_max = __reduce_max_sync(0xffffffffu, steps);
  const int64_t lhalf = rql.r > 0 ? (int64_t(1) << (rql.r - 1)) : 0;
  const int32_t nM = -rql.Sp;
  const uint32_t w2b = tc::smem_u32(w2s);
  uint32_t used = 0;
  for (uint32_t s = 0; s < steps_max; ++s) {
    prefetch(s + DEC_STAGES - 1);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(DEC_STAGES - 1) : "memory");
    const uint32_t j = s * K + uint32_t(gl);
    const bool act = s < steps && uint32_t(gl) < K && j < n;
    bool need = false;
    if (act) {
      const uint8_t* rw = slot + (s % DEC_STAGES) * 32 * DROW_BYTES;
      const uint32_t* hd = reinterpret_cast<const uint32_t*>(rw);
      const uint32_t slotv = x & 0xffffu;
      const uint32_t S = hd[0], inv32 = hd[1];
      const int32_t mu = int32_t(hd[2]);
      const uint64_t sS = uint64_t(S);
      // coarse block: C_{16k} ~= 16k + umulhi(E_{16k}, inv32) is C or C - 1 (inv32 is the
      // truncated reciprocal), and the C_{16k} are >= 16 apart, so only the last estimated
      // block can be one too far: one exact test (E * 65281 < (slot - i + 1) * S) fixes it
      int blk = 0;
#pragma unroll
      for (int k = 1; k < 16; ++k) {
        const uint32_t ce = uint32_t(16 * k) + __umulhi(hd[2 + k], inv32);
        blk += ce <= slotv ? 1 : 0;
      }
      if (blk > 0) {
        const uint32_t i = 16u * uint32_t(blk);
        if (!(i <= slotv && uint64_t(hd[2 + blk]) * 65281ull < uint64_t(slotv - i + 1u) * sS)) --blk;
      }
      // the block's 16 logits z_i = b2_i + a . W2_i (Eq.7), the Q8 requant, delta = mu - l_i
      // and e_i = LUT[delta >> 2] (0 beyond 16 nats; i = 255 is not a symbol)
      const uint4 a0 = reinterpret_cast<const uint4*>(rw + DROW_A)[0];
      const uint4 a1 = reinterpret_cast<const uint4*>(rw + DROW_A)[1];
      const uint32_t aw[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const int64_t C2 = (int64_t(mu) << 32) + 0x7fffffff;
      // the 8 chunk addresses of the block: chunk (t, h) = 8 (t >> 2) + ((2 (t & 3) + h + blk) & 7)
      uint32_t ca[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) ca[k] = w2b + 16u * (32u * uint32_t(blk) + ((uint32_t(k) + uint32_t(blk)) & 7u));
      uint32_t ev[16];
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const uint4 bb = b2s[b2_slot(uint32_t(blk), uint32_t(c4))];
        const uint32_t bv[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = 4 * c4 + u;
          uint4 q0, q1;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q0.x), "=r"(q0.y), "=r"(q0.z), "=r"(q0.w)
                       : "r"(ca[2 * (t & 3)] + 128u * uint32_t(t >> 2)));
          int32_t z = int32_t(bv[u]);
          z = __dp4a(int32_t(aw[0]), int32_t(q0.x), z);
          z = __dp4a(int32_t(aw[1]), int32_t(q0.y), z);
          if (HW > 2) {
            z = __dp4a(int32_t(aw[2]), int32_t(q0.z), z);
            z = __dp4a(int32_t(aw[3]), int32_t(q0.w), z);
          }
          if (HW > 4) {
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q1.x), "=r"(q1.y), "=r"(q1.z), "=r"(q1.w)
                         : "r"(ca[2 * (t & 3) + 1] + 128u * uint32_t(t >> 2)));
            z = __dp4a(int32_t(aw[4]), int32_t(q1.x), z);
            z = __dp4a(int32_t(aw[5]), int32_t(q1.y), z);
            z = __dp4a(int32_t(aw[6]), int32_t(q1.z), z);
            z = __dp4a(int32_t(aw[7]), int32_t(q1.w), z);
          }
          uint32_t dl;
          if (LQ == 0) {
            dl = uint32_t(int32_t((int64_t(z) * nM + C2) >> 32));
          } else {
            int64_t lv = (int64_t(z) * int64_t(rql.mp) + lhalf) >> rql.r;
            if (LQ == 2) {
              lv = z > zsat_hi ? (int64_t(1) << 24) : lv;
              lv = z < zsat_lo ? -(int64_t(1) << 24) : lv;
            }
            dl = uint32_t(mu - int32_t(lv));
          }
          ev[t] = slut[min(dl, 4096u) >> 2];
        }
      }
      if (blk == 15) ev[15] = 0u;  // index 255 is padding, not a symbol
      // fine search inside the block, the same estimate-then-fix scheme: C'_t = i + umulhi
      // (E_i, inv32) <= C_i <= C'_t + 1, the C_i strictly increasing
      const uint32_t E0 = blk ? hd[2 + blk] : 0u;
      uint32_t Er = E0, Elo = E0, elo = ev[0], eprev = 0u;
      int cnt = 0;
#pragma unroll
      for (int t = 0; t < 15; ++t) {
        Er += ev[t];  // E_{16 blk + t + 1}
        const uint32_t i1 = uint32_t(16 * blk + t + 1);
        const bool p = i1 + __umulhi(Er, inv32) <= slotv;  // monotone in t
        cnt += p ? 1 : 0;
        Elo = p ? Er : Elo;
        elo = p ? ev[t + 1] : elo;
        eprev = p ? ev[t] : eprev;  // the e last added into Elo
      }
      if (cnt > 0) {
        const uint32_t i = uint32_t(16 * blk + cnt);
        if (!(i <= slotv && uint64_t(Elo) * 65281ull < uint64_t(slotv - i + 1u) * sS)) {  // one too far
          Elo -= eprev;
          elo = eprev;
          --cnt;
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
      X[node + j] = uint8_t(lo + 1);
      x = f * (x >> 16) + slotv - cum;
      need = x < (1u << 16);
    }
    // the group's renormalisation words, in stream order, from its 3G-word window
    const unsigned gm = (__ballot_sync(0xffffffffu, need) >> (g << lg)) & gmask;
    const uint32_t rank = __popc(gm & ltg);
    const uint32_t off = used + rank - wbase;  // < 3G since used - wbase < G and rank < G
    const int src = (g << lg) + int(off & uint32_t(G - 1));
    const uint32_t v0 = __shfl_sync(0xffffffffu, w0, src);
    const uint32_t v1 = __shfl_sync(0xffffffffu, w1, src);
    const uint32_t v2 = __shfl_sync(0xffffffffu, w2, src);
    if (need) {
      const uint32_t sel = off >> lg;
      if (used + rank < W) x = (x << 16) | (sel == 0 ? v0 : (sel == 1 ? v1 : v2));
      else bad = true;
    }
    used += __popc(gm);
    if (used - wbase >= uint32_t(G)) {  // slide the window by G words, load 2G ahead
      wbase += uint32_t(G);
      w0 = w1;
      w1 = w2;
      w2 = ldw(wbase + 2u * uint32_t(G) + uint32_t(gl));
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  if (gw < nseg && (used != W || (uint32_t(gl) < K && x != (1u << 16)))) bad = true;
  const unsigned bm = (__ballot_sync(0xffffffffu, bad) >> (g << lg)) & gmask;
  if (bm && gl == 0) atomicOr(err, EF_CORRUPT);
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
  int lg = 0;  // lane-group size G = 2^lg >= the level's largest K
  while ((1 << lg) < max_lanes) ++lg;
  const int per_warp = 32 >> lg;
  const int warps = (nseg + per_warp - 1) / per_warp;
  const unsigned grid = unsigned((warps + DEC_WPC - 1) / DEC_WPC);
  constexpr size_t smem = size_t(DEC_WPC) * DEC_STAGES * 32 * DROW_BYTES;
  const int lq = hd.can_saturate ? 2 : (hd.rql.fast_s ? 0 : 1);
  // algorithmic bytes: the 112-byte row and one 16-bit word per symbol
  Prof p(c, "rans_dec", nsym * (DROW_BYTES + 2));
#define PCC_DEC(HH, LQ)                                                                                          \
  if (H == HH && lq == LQ) {                                                                                     \
    PCC_SMEM_ATTR((k_rans_dec<HH, LQ>), smem);                                                                   \
    k_rans_dec<HH, LQ><<<grid, 32 * DEC_WPC, smem, c->stream>>>(d_segs, nseg, lg, bs,                            \
                                                                reinterpret_cast<const uint8_t*>(rows), hd.W2,  \
                                                                hd.b2, hd.rql, hd.zsat_lo, hd.zsat_hi, lut, X,  \
                                                                err);                                           \
    launched(c);                                                                                                 \
    return;                                                                                                      \
  }
  PCC_DEC(8, 0)
  PCC_DEC(8, 1)
  PCC_DEC(8, 2)
  PCC_DEC(16, 0)
  PCC_DEC(16, 1)
  PCC_DEC(16, 2)
  PCC_DEC(32, 0)
  PCC_DEC(32, 1)
  PCC_DEC(32, 2)
#undef PCC_DEC
  throw Error{PCC_ERR_INVALID_ARG};
}

}  // namespace pcc
