// rawcoder.cu — the raw prefix X_0..X_{R-1} "encode[d] ... based on their symbol
// frequencies" (reading Q13', NEXT-4), when the model sets MF_RAW_FREQ.
//
// Adaptive frequency model: counts n_i = 1 for the 255 symbols, total T; after a symbol,
// n_i += RAW_INC and T += RAW_INC, and when T > RAW_LIMIT every count is halved rounding
// up.  Q16 cumulative bounds by cumulative floors (as reading Q21): C_i = i +
// floor(K_i * 65281 / T), K_i = sum_{u<i} n_u, C_255 = 65536.  One rANS lane of the O9
// coder; region = u32 W | u32 x | W u16 words (decoder order) | pad to 4 bytes.
//
// One warp per frame.  Lane l holds the counts of symbol indices 8l..8l+7 in registers
// (index 255 does not exist and stays 0); prefix sums by a warp scan.  The decoder finds
// the symbol with the division-free test C_j <= slot <=> K_j * 65281 < (slot - j + 1) * T.
#include "pcc_internal.cuh"

namespace pcc {
namespace {

constexpr uint32_t RAW_INC = 32, RAW_LIMIT = 1u << 15;

struct WarpFreq {
  uint32_t n[8];   // counts of symbol indices 8*lane + k
  uint32_t T;      // total (all lanes hold it)
  __device__ void init(int lane) {
#pragma unroll
    for (int k = 0; k < 8; ++k) n[k] = (8 * lane + k < NCODE) ? 1u : 0u;
    T = NCODE;
  }
  // K before this lane's first symbol (exclusive warp scan of the lane sums)
  __device__ uint32_t lane_base(int lane) const {
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += n[k];
    uint32_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    return inc - s;
  }
  // C_i for i = 8*lane + k (k in 0..8) given the lane base
  __device__ uint32_t bound(uint32_t base, int lane, int k) const {
    uint32_t K = base;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (u < k) K += n[u];
    return uint32_t(8 * lane + k) + uint32_t((uint64_t(K) * 65281u) / T);
  }
  __device__ void update(int lane, int i) {
    if ((i >> 3) == lane) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if ((i & 7) == k) n[k] += RAW_INC;
    }
    T += RAW_INC;
    if (T > RAW_LIMIT) {
      uint32_t s = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        n[k] = (n[k] + 1) >> 1;
        s += n[k];
      }
      T = __reduce_add_sync(0xffffffffu, s);
    }
  }
};

// Encoder: symbols of frame f = code[nb[d] + foff[d][f] .. ] for d = 0..R-1 in order.
// Writes the region into out + f * cap and its byte size into sz[f].  cf: scratch
// u32 [frames][max_sym] of (cum | freq << 16).
__global__ void k_raw_enc(const uint8_t* __restrict__ code, const uint64_t* __restrict__ nb,
                          const uint32_t* __restrict__ foff, int B, int R, uint32_t max_sym,
                          uint32_t* __restrict__ cf, uint16_t* __restrict__ stack, uint8_t* __restrict__ out,
                          uint32_t cap, uint32_t* __restrict__ sz) {
  const int f = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (f >= B) return;
  WarpFreq fm;
  fm.init(lane);
  uint32_t* mycf = cf + size_t(f) * max_sym;
  uint32_t j = 0;
  for (int d = 0; d < R; ++d) {
    const uint32_t a = foff[d * (B + 1) + f], cnt = foff[d * (B + 1) + f + 1] - a;
    const uint8_t* X = code + nb[d] + a;
    for (uint32_t k = 0; k < cnt; ++k, ++j) {
      const int i = int(X[k]) - 1;
      const uint32_t base = fm.lane_base(lane);
      uint32_t lo = 0, hi = 0;
      if ((i >> 3) == lane) {
        lo = fm.bound(base, lane, i & 7);
        hi = fm.bound(base, lane, (i & 7) + 1);
      }
      lo = __shfl_sync(0xffffffffu, lo, i >> 3);
      hi = __shfl_sync(0xffffffffu, hi, i >> 3);
      if (lane == 0) mycf[j] = lo | ((hi - lo) << 16);
      fm.update(lane, i);
    }
  }
  __syncwarp();
  if (lane != 0) return;
  // one rANS lane, symbols in reverse; words pushed on a stack emitted reversed
  uint32_t x = 1u << 16, W = 0;
  uint16_t* st = stack + size_t(f) * max_sym;
  for (uint32_t t = j; t-- > 0;) {
    const uint32_t c = mycf[t] & 0xFFFFu, fr = mycf[t] >> 16;
    if (uint64_t(x) >= (uint64_t(fr) << 16)) {
      st[W++] = uint16_t(x & 0xFFFFu);
      x >>= 16;
    }
    x = ((x / fr) << 16) + (x % fr) + c;
  }
  uint8_t* o = out + size_t(f) * cap;
  reinterpret_cast<uint32_t*>(o)[0] = W;
  reinterpret_cast<uint32_t*>(o)[1] = x;
  uint16_t* w = reinterpret_cast<uint16_t*>(o + 8);
  for (uint32_t k = 0; k < W; ++k) w[k] = st[W - 1 - k];
  if (W & 1u) w[W] = 0;
  sz[f] = 8u + 4u * ((W + 1u) / 2u);
}

// Plain reading Q13: region = the raw bytes themselves; only the size is needed.
__global__ void k_raw_plain_size(const uint32_t* __restrict__ foff, int B, int R, uint32_t* __restrict__ sz) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= B) return;
  uint32_t s = 0;
  for (int d = 0; d < R; ++d) s += foff[d * (B + 1) + f + 1] - foff[d * (B + 1) + f];
  sz[f] = s;
}

// Decoder: region of frame f at bs + raw_off[f], raw_len[f] bytes.  Writes the decoded
// symbols to sym + f * max_sym and the node count of every depth 0..R into
// cnt[f * (R + 1) + d] (the same contract as the plain k_raw_count).
__global__ void k_raw_dec(const uint8_t* __restrict__ bs, const uint64_t* __restrict__ raw_off,
                          const uint32_t* __restrict__ raw_len, int B, int R, uint32_t max_sym,
                          const uint32_t* __restrict__ NL, uint8_t* __restrict__ sym, uint32_t* __restrict__ cnt,
                          uint32_t* __restrict__ err) {
  const int f = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (f >= B) return;
  const uint8_t* p = bs + raw_off[f];
  const uint32_t len = raw_len[f];
  bool bad = len < 8;
  uint32_t W = 0, x = 0;
  if (!bad) {
    W = uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
    x = uint32_t(p[4]) | uint32_t(p[5]) << 8 | uint32_t(p[6]) << 16 | uint32_t(p[7]) << 24;
    bad = uint64_t(len) != 8ull + 4ull * ((uint64_t(W) + 1) / 2) || x < (1u << 16);
  }
  const uint8_t* w = p + 8;
  WarpFreq fm;
  fm.init(lane);
  uint8_t* out = sym + size_t(f) * max_sym;
  uint32_t nd = 1, pos = 0, j = 0;
  for (int d = 0; d < R && !bad; ++d) {
    if (lane == 0) cnt[f * (R + 1) + d] = nd;
    uint32_t nx = 0;
    for (uint32_t k = 0; k < nd; ++k, ++j) {
      const uint32_t slot = x & 0xFFFFu;
      const uint32_t base = fm.lane_base(lane);
      // #{ boundaries C_b <= slot, b = 1..255 } = the symbol index (C strictly increasing)
      uint32_t le = 0, K = base;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        K += fm.n[q];
        const int b = 8 * lane + q + 1;  // boundary C_b (upper bound of index b-1)
        if (b <= NCODE && int(slot) - b >= 0 &&
            uint64_t(K) * 65281u < uint64_t(int(slot) - b + 1) * fm.T)
          ++le;
      }
      const int i = int(__reduce_add_sync(0xffffffffu, le));
      uint32_t lo = 0, hi = 0;
      if ((i >> 3) == lane) {
        lo = fm.bound(base, lane, i & 7);
        hi = fm.bound(base, lane, (i & 7) + 1);
      }
      lo = __shfl_sync(0xffffffffu, lo, i >> 3);
      hi = __shfl_sync(0xffffffffu, hi, i >> 3);
      x = (hi - lo) * (x >> 16) + slot - lo;
      if (x < (1u << 16)) {
        if (pos >= W) {
          bad = true;
          break;
        }
        x = (x << 16) | (uint32_t(w[2 * pos]) | uint32_t(w[2 * pos + 1]) << 8);
        ++pos;
      }
      if (lane == 0) out[j] = uint8_t(i + 1);
      nx += __popc(uint32_t(i + 1));
      fm.update(lane, i);
    }
    nd = nx;
    if (nd > NL[f]) bad = true;
  }
  if (!bad && (pos != W || x != (1u << 16))) bad = true;
  if (lane == 0) {
    cnt[f * (R + 1) + R] = bad ? 0 : nd;
    if (bad) atomicOr(err, EF_CORRUPT);
  }
}

inline unsigned cdiv(size_t a, size_t b) { return unsigned((a + b - 1) / b); }

}  // namespace

uint32_t raw_max_symbols(int R) {
  uint32_t s = 0, p = 1;
  for (int d = 0; d < R; ++d, p *= 8) s += p;
  return s;
}

void raw_encode(pcc_ctx c, bool freq, const uint8_t* code, const uint64_t* d_nb, const uint32_t* d_foff, int B, int R,
                uint8_t* region, uint32_t cap, uint32_t* sz) {
  Prof p(c, "container", 0);
  if (!freq) {
    k_raw_plain_size<<<cdiv(B, 128), 128, 0, c->stream>>>(d_foff, B, R, sz);
  } else {
    const uint32_t ms = raw_max_symbols(R);
    uint32_t* cf = wsT<uint32_t>(c, "raw_cf", size_t(B) * ms);
    uint16_t* st = wsT<uint16_t>(c, "raw_stack", size_t(B) * ms);
    k_raw_enc<<<cdiv(size_t(B) * 32, 128), 128, 0, c->stream>>>(code, d_nb, d_foff, B, R, ms, cf, st, region, cap, sz);
  }
  launched(c);
}

void raw_decode(pcc_ctx c, const uint8_t* bs, const uint64_t* raw_off, const uint32_t* raw_len, int B, int R,
                const uint32_t* d_NL, uint8_t* sym, uint32_t* cnt, uint32_t* err) {
  Prof p(c, "container", 0);
  k_raw_dec<<<cdiv(size_t(B) * 32, 128), 128, 0, c->stream>>>(bs, raw_off, raw_len, B, R, raw_max_symbols(R), d_NL, sym,
                                                             cnt, err);
  launched(c);
}

}  // namespace pcc
