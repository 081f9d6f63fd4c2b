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
  return int(k < 1u ? 1u : (k > 8u ? 8u : k));
}

// Lane groups of MAX_LANES = 8: a warp encodes 4 segments side by side (reading Q24': K <= 8).
__global__ void __launch_bounds__(128) k_rans_enc(const EncSeg* __restrict__ segs, int nseg, const uint32_t* __restrict__ cf,
                                                  uint16_t* __restrict__ words, uint32_t* __restrict__ seg_W,
                                                  uint32_t* __restrict__ seg_state) {
  constexpr int G = MAX_LANES;
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), gb = lane - gl;
  const int gw = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * (32 / G) + (lane / G);
  if (int((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * (32 / G) >= nseg) return;  // whole warp idle
  const bool seg = gw < nseg;
  const EncSeg sg = seg ? segs[gw] : EncSeg{0, 0};
  const uint32_t n = sg.n;
  const int K = seg ? lanes_for(n) : 1;
  const uint32_t steps = seg ? (n + uint32_t(K) - 1u) / uint32_t(K) : 0u;
  const uint32_t steps_max = __reduce_max_sync(0xffffffffu, steps);
  uint32_t x = 1u << 16;
  uint32_t cnt = 0;
  uint16_t* end = words + sg.node + n;
  const unsigned above = ~((2u << gl) - 1u) & 0xffu;  // lanes of the group with a higher index
  // the (cum, freq) words do not depend on the state: load them EP steps ahead in a
  // register ring so the serial state chain never waits on memory
  constexpr int EP = 8;
  auto ldcf = [&](uint32_t s) -> uint32_t {
    const uint32_t j = s * uint32_t(K) + uint32_t(gl);
    return (s < steps && gl < K && j < n) ? __ldg(cf + sg.node + j) : 0u;
  };
  uint32_t ring[EP];
#pragma unroll
  for (int e = 0; e < EP; ++e) ring[e] = steps_max > uint32_t(e) ? ldcf(steps_max - 1u - uint32_t(e)) : 0u;
  for (uint32_t s = steps_max; s-- > 0;) {
    const uint32_t j = s * uint32_t(K) + uint32_t(gl);
    const bool act = s < steps && gl < K && j < n;
    const uint32_t v = ring[0];
#pragma unroll
    for (int e = 0; e < EP - 1; ++e) ring[e] = ring[e + 1];
    ring[EP - 1] = s >= uint32_t(EP) ? ldcf(s - uint32_t(EP)) : 0u;
    const uint32_t c = v & 0xffffu, f = v >> 16;
    const bool emit = act && x >= (f << 16);
    const unsigned m = (__ballot_sync(0xffffffffu, emit) >> gb) & 0xffu;
    if (emit) {
      end[-1 - int(cnt + __popc(m & above))] = uint16_t(x & 0xffffu);
      x >>= 16;
    }
    cnt += __popc(m);
    if (act) x = ((x / f) << 16) + (x % f) + c;
  }
  if (seg && gl == 0) seg_W[gw] = cnt;
  if (seg && gl < K) seg_state[size_t(gw) * 32 + gl] = x;
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
    // walk earlier (full, 4096-symbol, K = 8) chunks of this level payload
    for (uint32_t ch = 0; ch < sg.chunk && !bad; ++ch) {
      if (pos + 4 > lvl_bytes) { bad = true; break; }
      const uint32_t Wc = ld_u32(lvl + pos);
      const uint64_t sz = 4ull + 4ull * MAX_LANES + 4ull * ((uint64_t(Wc) + 1) / 2);
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


// ---- T threads per rANS state (T = 2 or 4) ----------------------------------------
// The decode of one segment is a chain of <= 512 dependent steps per lane, and a step of
// k_rans_dec is ~700 instructions on one thread: at the small levels a warp runs alone on
// its SM partition and each step costs ~3000 cycles.  Here T threads share a state: thread
// q owns the U = 16 / T symbols U q .. U q + U - 1 of every 16-symbol block (its share of the
// coarse test, the block's logits and exponentials, the fine test), the T partial results
// meet by shuffles, and every thread of the state keeps the same x.  A warp holds 32 / T
// states; a segment's K <= 8 lanes (reading Q24') form a group of G T threads (G = the
// power of two >= the level's largest K).  W2 chunk (i, h) sits at slot 32 (i >> 4) + 8 ((i
// >> 2) & 3) + (((2 (i & 3) + h + 2 ((i >> 2) & 3)) & 7) ^ ((i >> 4) & 7)): the T threads of
// a state (rows U q + u of one block) read distinct bank groups, and a thread's chunk
// address in block blk is one LOP3 of a per-step base, a per-thread constant and blk.
__device__ __forceinline__ uint32_t w2_koff(uint32_t r, uint32_t h) {  // r = i & 15: 128 (r >> 2) + 16 c
  return 128u * (r >> 2) + 16u * ((2u * (r & 3u) + h + 2u * (r >> 2)) & 7u);
}
__device__ __forceinline__ uint32_t w2_slot_t(uint32_t i, uint32_t h) {
  return 32u * (i >> 4) + ((w2_koff(i & 15u, h) ^ (((i >> 4) & 7u) << 4)) >> 4);
}

template <int U>
__device__ __forceinline__ uint32_t pick(const uint32_t (&v)[U], uint32_t k) {
  uint32_t r = v[0];
#pragma unroll
  for (int u = 1; u < U; ++u) r = k == uint32_t(u) ? v[u] : r;
  return r;
}

// floor(E 65281 / S) exactly: the 32-bit reciprocal estimate is q or q - 1 (inv32 truncated)
__device__ __forceinline__ uint32_t qexact(uint32_t E, uint32_t inv32, uint64_t sS) {
  const uint32_t qt = __umulhi(E, inv32);
  return qt + ((uint64_t(E) * 65281ull - uint64_t(qt) * sS) >= sS ? 1u : 0u);
}

template <int H, int LQ, int T, int NS>
__global__ void __launch_bounds__(32 * DEC_WPC) k_rans_dec_t(const DecSeg* __restrict__ segs, int nseg, int lg,
                                                            const uint8_t* __restrict__ bs, const uint8_t* __restrict__ rowsg,
                                                            const int8_t* __restrict__ W2, const int32_t* __restrict__ b2,
                                                            RQ rql, int32_t zsat_lo, int32_t zsat_hi,
                                                            const uint32_t* __restrict__ lut, uint8_t* __restrict__ X,
                                                            uint32_t* __restrict__ err) {
  constexpr int SPW = 32 / T;  // states per warp
  constexpr int U = 16 / T;    // symbols of a 16-block per thread
  constexpr int HW = H / 4;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr uint32_t RSTRIDE = uint32_t(SPW) * DROW_BYTES;  // bytes between stages of one state
  extern __shared__ __align__(128) uint8_t dsm[];  // [DEC_WPC][NS][SPW states][DROW_BYTES]
  __shared__ __align__(512) uint4 w2s[512];
  __shared__ uint4 b2s[64];
  __shared__ uint32_t slut[1025];  // the model's exp table, slut[1024] = 0 (delta >= 4096)
  for (int k = threadIdx.x; k < 512; k += blockDim.x) {
    const uint32_t i = uint32_t(k) >> 1, h = uint32_t(k) & 1u;
    uint32_t wv[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const uint32_t wi = 4u * h + uint32_t(w);
      wv[w] = wi < uint32_t(HW) ? reinterpret_cast<const uint32_t*>(W2)[i * HW + wi] : 0u;
    }
    w2s[w2_slot_t(i, h)] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
  for (int k = threadIdx.x; k < 64; k += blockDim.x) {
    const uint32_t blk = uint32_t(k) >> 2, c = uint32_t(k) & 3u;
    b2s[b2_slot(blk, c)] = reinterpret_cast<const uint4*>(b2)[k];
  }
  for (int k = threadIdx.x; k < 1024; k += blockDim.x) slut[k] = lut[k];
  if (threadIdx.x == 0) slut[1024] = 0u;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = lane & (T - 1), sl = lane / T;                 // thread of the state, state slot
  const int G = 1 << lg, GT = G * T;
  const int g = sl >> lg, gl = sl & (G - 1);                   // group (segment) of the warp, lane k
  const int gb = g * GT, gt = lane - gb;                       // the group's first lane, index in it
  const int sb = lane - q;                                     // the state's first lane
  const unsigned gmask = GT == 32 ? FULL : ((1u << GT) - 1u);
  const unsigned smask = (T == 32 ? FULL : ((1u << T) - 1u)) << sb;  // the state's T lanes
  const int gw = (blockIdx.x * DEC_WPC + warp) * (SPW >> lg) + g;
  if ((blockIdx.x * DEC_WPC + warp) * (SPW >> lg) >= nseg) return;  // whole warp idle
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
    for (uint32_t ch = 0; ch < sg.chunk && !bad; ++ch) {  // earlier full (4096-symbol, K = 8) chunks
      if (pos + 4 > lvl_bytes) { bad = true; break; }
      const uint32_t Wc = ld_u32(lvl + pos);
      const uint64_t sz = 4ull + 4ull * MAX_LANES + 4ull * ((uint64_t(Wc) + 1) / 2);
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
  // the group's word window [wbase, wbase + 3 GT): word wbase + gt + m GT in wm; w3 is the
  // next slide's w2, loaded a whole slide ahead so no shuffle waits on a global load
  uint32_t wbase = 0;
  uint32_t w0 = steps ? ldw(gt) : 0u, w1 = steps ? ldw(GT + gt) : 0u, w2 = steps ? ldw(2 * GT + gt) : 0u;
  uint32_t w3 = steps ? ldw(3 * GT + gt) : 0u;
  // row prefetch: this thread's 16-byte chunks q, q + T, .. of its state's row, NS - 1 steps ahead
  const uint8_t* pf_src = rowsg + (size_t(node) + gl) * DROW_BYTES;
  const size_t pf_inc = size_t(K) * DROW_BYTES;
  const bool pf_lane = uint32_t(gl) < K;
  uint8_t* srow0 = dsm + (size_t(warp) * NS * SPW + sl) * DROW_BYTES;
  const uint32_t pf_dst0 = tc::smem_u32(srow0);
  uint32_t pf_st = 0, pf_stage = 0;
  auto prefetch = [&]() {
    if (pf_lane && pf_st < steps && pf_st * K + gl < n) {
      const uint32_t dst = pf_dst0 + pf_stage * RSTRIDE;
#pragma unroll
      for (int c16 = q; c16 < DROW_BYTES / 16; c16 += T)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 16 * c16), "l"(pf_src + 16 * c16));
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    pf_src += pf_inc;
    ++pf_st;
    pf_stage = pf_stage + 1 == NS ? 0u : pf_stage + 1;
  };
#pragma unroll
  for (int p = 0; p < NS - 1; ++p) prefetch();
  const uint32_t steps_max = __reduce_max_sync(FULL, steps);
  const int64_t lhalf = rql.r > 0 ? (int64_t(1) << (rql.r - 1)) : 0;
  const int32_t nM = -rql.Sp;
  const uint32_t w2b = tc::smem_u32(w2s);
  const bool lastq = q == T - 1;
  uint32_t ko[U][2];  // chunk offsets of this thread's rows U q + u within a block (w2_koff)
#pragma unroll
  for (int u = 0; u < U; ++u) {
    ko[u][0] = w2_koff(uint32_t(U * q + u), 0u);
    ko[u][1] = w2_koff(uint32_t(U * q + u), 1u);
  }
  uint32_t used = 0, rd_stage = 0;
  for (uint32_t s = 0; s < steps_max; ++s) {
    __syncwarp();  // the stage refilled below was last read at step s - 1 by every thread
    prefetch();
    asm volatile("cp.async.wait_group %0;\n" ::"n"(NS - 1) : "memory");
    __syncwarp();  // the T threads' chunks of the row are visible to all of them
    const uint32_t j = s * K + uint32_t(gl);
    const bool act = s < steps && uint32_t(gl) < K && j < n;
    // every thread computes (inactive states on stale rows: all reads stay in bounds), so
    // the ballots and shuffles below always see the whole warp
    const uint8_t* rw = srow0 + rd_stage * RSTRIDE;
    rd_stage = rd_stage + 1 == NS ? 0u : rd_stage + 1;
    const uint32_t* hd = reinterpret_cast<const uint32_t*>(rw);
    const uint4 h0 = *reinterpret_cast<const uint4*>(rw);
    const uint32_t Sv = h0.x, inv32 = h0.y;
    const int32_t mu = int32_t(h0.z);
    const uint64_t sS = uint64_t(Sv);
    // coarse thresholds C_{16k} = 16 k + floor(E_{16k} 65281 / S) exactly (independent of x),
    // thread q owning k = U q + 1 .. U q + U (k <= 15)
    uint32_t thr[U];
#pragma unroll
    for (int v = 0; v < U; ++v) {
      const uint32_t k = uint32_t(U * q + 1 + v);
      thr[v] = (v < U - 1 || !lastq) ? 16u * k + qexact(hd[2 + k], inv32, sS) : 0xffffffffu;
    }
    const uint32_t slotv = x & 0xffffu;
    // blk = #{k in 1..15 : C_{16k} <= slot} (the C are increasing): one ballot per owned k
    uint32_t blk = 0;
#pragma unroll
    for (int v = 0; v < U; ++v) blk += __popc(__ballot_sync(FULL, thr[v] <= slotv) & smask);
    const uint32_t E0 = blk ? hd[2 + blk] : 0u;
    const uint32_t Cb = 16u * blk + qexact(E0, inv32, sS);                               // C_{16 blk}
    const uint32_t Cn = blk < 15u ? 16u * (blk + 1u) + qexact(hd[3 + blk], inv32, sS) : 65536u;  // C_{16 blk + 16}
    // this thread's U logits z_i = b2_i + a . W2_i of the block (Eq.7), delta, e_i = LUT[delta >> 2]
    const uint4 a0 = reinterpret_cast<const uint4*>(rw + DROW_A)[0];
    const uint4 a1 = reinterpret_cast<const uint4*>(rw + DROW_A)[1];
    const uint32_t aw[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    const int64_t C2 = (int64_t(mu) << 32) + 0x7fffffff;
    const uint32_t Ab = w2b + 512u * blk, B16 = (blk & 7u) << 4;
    uint32_t ev[U];
#pragma unroll
    for (int c4 = 0; c4 < U / 4; ++c4) {
      const uint4 bb = b2s[b2_slot(blk, uint32_t(U * q / 4 + c4))];
      const uint32_t bv[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
      for (int u4 = 0; u4 < 4; ++u4) {
        const int u = 4 * c4 + u4;
        uint4 q0, q1;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q0.x), "=r"(q0.y), "=r"(q0.z), "=r"(q0.w)
                     : "r"(Ab | (ko[u][0] ^ B16)));
        int32_t z = int32_t(bv[u4]);
        z = __dp4a(int32_t(aw[0]), int32_t(q0.x), z);
        z = __dp4a(int32_t(aw[1]), int32_t(q0.y), z);
        if (HW > 2) {
          z = __dp4a(int32_t(aw[2]), int32_t(q0.z), z);
          z = __dp4a(int32_t(aw[3]), int32_t(q0.w), z);
        }
        if (HW > 4) {
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q1.x), "=r"(q1.y), "=r"(q1.z), "=r"(q1.w)
                       : "r"(Ab | (ko[u][1] ^ B16)));
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
        ev[u] = slut[min(dl, 4096u) >> 2];
      }
    }
    if (lastq) ev[U - 1] = blk == 15u ? 0u : ev[U - 1];  // index 255 is padding, not a symbol
    // prefix masses: P[u] = e_0 + .. + e_u of this thread, plus the lower threads' sums
    uint32_t P[U];
    P[0] = ev[0];
#pragma unroll
    for (int u = 1; u < U; ++u) P[u] = P[u - 1] + ev[u];
    uint32_t incl = P[U - 1];
#pragma unroll
    for (int o = 1; o < T; o <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL, incl, o, T);
      if (q >= o) incl += t;
    }
    const uint32_t base = E0 + incl - P[U - 1];
    // fine thresholds C_{i1} (i1 = 16 blk + t + 1, t = U q + u <= 14) exactly; the symbol's
    // offset in the block is c = #{t : C_{i1} <= slot}, lo = 16 blk + c
    uint32_t Cf[U];
    uint32_t c = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i1 = 16u * blk + uint32_t(U * q + u) + 1u;
      Cf[u] = (u < U - 1 || !lastq) ? i1 + qexact(base + P[u], inv32, sS) : 0xffffffffu;
      c += __popc(__ballot_sync(FULL, Cf[u] <= slotv) & smask);
    }
    // cum = C_lo, nxt = C_{lo+1}: fine thresholds of positions c - 1 and c, from their owners
    const uint32_t cm = c ? c - 1u : 0u;
    const uint32_t s_cum = pick<U>(Cf, cm % U), s_nxt = pick<U>(Cf, c % U);
    const uint32_t g_cum = T > 1 ? __shfl_sync(FULL, s_cum, sb + int(cm / U)) : s_cum;
    const uint32_t g_nxt = T > 1 ? __shfl_sync(FULL, s_nxt, sb + int(c / U)) : s_nxt;
    const uint32_t cum = c ? g_cum : Cb;
    const uint32_t nxt = c < 15u ? g_nxt : Cn;
    bool need = false;
    if (act) {
      if (q == 0) X[node + j] = uint8_t(16u * blk + c + 1u);
      x = (nxt - cum) * (x >> 16) + slotv - cum;
      need = x < (1u << 16);
    }
    // the group's renormalisation words, in stream order (lane order), from its window
    const unsigned gm = (__ballot_sync(FULL, need && q == 0) >> gb) & gmask;  // states' first lanes
    const uint32_t rank = __popc(gm & ((1u << (gl * T)) - 1u));
    const uint32_t off = used + rank - wbase;  // < 2 GT
    const int src = gb + int(off & uint32_t(GT - 1));
    const uint32_t v0 = __shfl_sync(FULL, w0, src);
    const uint32_t v1 = __shfl_sync(FULL, w1, src);
    if (need) {
      if (used + rank < W) x = (x << 16) | (off < uint32_t(GT) ? v0 : v1);
      else bad = true;
    }
    used += __popc(gm);
    if (used - wbase >= uint32_t(GT)) {  // slide the window by GT words
      wbase += uint32_t(GT);
      w0 = w1;
      w1 = w2;
      w2 = w3;
      w3 = ldw(wbase + 3u * uint32_t(GT) + uint32_t(gt));
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  if (gw < nseg && (used != W || (uint32_t(gl) < K && x != (1u << 16)))) bad = true;
  const unsigned bm = (__ballot_sync(FULL, bad) >> gb) & gmask;
  if (bm && gt == 0) atomicOr(err, EF_CORRUPT);
}

}  // namespace

void rans_encode(pcc_ctx c, const EncSeg* d_segs, int nseg, const uint32_t* cf, uint16_t* words, uint32_t* seg_W,
                 uint32_t* seg_state,
                 size_t nsym) {
  if (nseg == 0) return;
  const unsigned grid = unsigned((size_t(nseg) * MAX_LANES + 127) / 128);
  // algorithmic bytes: the (cum, freq) word read and one 16-bit word written per symbol
  Prof p(c, "rans_enc", nsym * (4 + 2));
  k_rans_enc<<<grid, 128, 0, c->stream>>>(d_segs, nseg, cf, words, seg_W, seg_state);
  launched(c);
}

void rans_decode(pcc_ctx c, const DecSeg* d_segs, int nseg, const uint8_t* bs, const uint16_t* rows, int H,
                 const DHead& hd, const uint32_t* lut, uint8_t* X, uint32_t* err, int max_lanes, size_t nsym,
                 size_t nstates) {
  if (nseg == 0) return;
  // threads per state (k_rans_dec_t): 4 while the level has few states (its decode is one
  // chain of <= 512 latency-bound steps per lane), 2 beyond 8192 states (there the issue rate
  // bounds it and 4 threads repeat more of the per-state work); PCC_RDEC=t4 / t2 force one,
  // PCC_RDEC=old runs k_rans_dec (one thread per state) for A/B
  static const int tps_env = [] {
    const char* e = getenv("PCC_RDEC");
    if (e && std::string(e) == "t4") return 4;
    if (e && std::string(e) == "t2") return 2;
    if (e && (std::string(e) == "old" || std::string(e) == "t1")) return 0;
    return -1;
  }();
  const int tps = tps_env >= 0 ? tps_env : (nstates <= 8192 ? 4 : 2);
  static const int ns = [] {  // row prefetch stages of k_rans_dec_t (PCC_RDEC_NS=3 for A/B)
    const char* e = getenv("PCC_RDEC_NS");
    return e && std::string(e) == "3" ? 3 : 6;
  }();
  int lg = 0;  // lane-group size G = 2^lg >= the level's largest K
  while ((1 << lg) < max_lanes) ++lg;
  const int T = tps ? tps : 1;
  const int per_warp = (32 / T) >> lg;
  const int warps = (nseg + per_warp - 1) / per_warp;
  const unsigned grid = unsigned((warps + DEC_WPC - 1) / DEC_WPC);
  const size_t smem = size_t(DEC_WPC) * (tps ? ns : DEC_STAGES) * (32 / T) * DROW_BYTES;
  const int lq = hd.can_saturate ? 2 : (hd.rql.fast_s ? 0 : 1);
  // algorithmic bytes: the 112-byte row and one 16-bit word per symbol
  Prof p(c, "rans_dec", nsym * (DROW_BYTES + 2));
#define PCC_DECT(HH, LQ, TT, NN)                                                                                 \
  PCC_SMEM_ATTR((k_rans_dec_t<HH, LQ, TT, NN>), smem);                                                           \
  k_rans_dec_t<HH, LQ, TT, NN><<<grid, 32 * DEC_WPC, smem, c->stream>>>(d_segs, nseg, lg, bs, rw, hd.W2, hd.b2,   \
                                                                        hd.rql, hd.zsat_lo, hd.zsat_hi, lut, X, err)
#define PCC_DEC(HH, LQ)                                                                                          \
  if (H == HH && lq == LQ) {                                                                                     \
    const uint8_t* rw = reinterpret_cast<const uint8_t*>(rows);                                                  \
    if (tps == 0) {                                                                                              \
      PCC_SMEM_ATTR((k_rans_dec<HH, LQ>), smem);                                                                 \
      k_rans_dec<HH, LQ><<<grid, 32 * DEC_WPC, smem, c->stream>>>(d_segs, nseg, lg, bs, rw, hd.W2, hd.b2, hd.rql, \
                                                                  hd.zsat_lo, hd.zsat_hi, lut, X, err);          \
    } else if (T == 4 && ns == 6) {                                                                              \
      PCC_DECT(HH, LQ, 4, 6);                                                                                    \
    } else if (T == 4) {                                                                                         \
      PCC_DECT(HH, LQ, 4, 3);                                                                                    \
    } else if (ns == 6) {                                                                                        \
      PCC_DECT(HH, LQ, 2, 6);                                                                                    \
    } else {                                                                                                     \
      PCC_DECT(HH, LQ, 2, 3);                                                                                    \
    }                                                                                                            \
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
#undef PCC_DECT
  throw Error{PCC_ERR_INVALID_ARG};
}

}  // namespace pcc
