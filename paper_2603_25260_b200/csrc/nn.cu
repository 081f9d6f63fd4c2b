// nn.cu — integer-only network layers (Eq.4-15), SIMT int8 path (dp4a).
//
// All layers: int8 activations/weights, zero-points 0 (reading Q16), exact int32
// accumulation (Eq.13; any summation order gives the same int32, reading O6), and the
// fixed-point requant q = clip((acc*m + 2^(r-1)) >> r) with PReLU fused as a sign-
// selected multiplier (Eq.14; readings Q15, Q18).
#include "pcc_internal.cuh"
#include "rq.cuh"

namespace pcc {

namespace {

__device__ __forceinline__ uint32_t pack4(int32_t a, int32_t b, int32_t c, int32_t d) {
  return (uint32_t(a) & 0xffu) | (uint32_t(b) & 0xffu) << 8 | (uint32_t(c) & 0xffu) << 16 | (uint32_t(d) & 0xffu) << 24;
}

template <int WORDS>
__device__ __forceinline__ void load_row(const int8_t* p, int32_t* x) {
  if constexpr (WORDS % 4 == 0) {
#pragma unroll
    for (int w = 0; w < WORDS; w += 4) {
      int4 v = *reinterpret_cast<const int4*>(p + 4 * w);
      x[w] = v.x; x[w + 1] = v.y; x[w + 2] = v.z; x[w + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int w = 0; w < WORDS; w += 2) {
      int2 v = *reinterpret_cast<const int2*>(p + 4 * w);
      x[w] = v.x; x[w + 1] = v.y;
    }
  }
}

template <int COUT>
__device__ __forceinline__ void store_row(int8_t* p, const int32_t* q) {
  uint32_t w[COUT / 4];
#pragma unroll
  for (int k = 0; k < COUT / 4; ++k) w[k] = pack4(q[4 * k], q[4 * k + 1], q[4 * k + 2], q[4 * k + 3]);
  if constexpr (COUT % 16 == 0) {
#pragma unroll
    for (int k = 0; k < COUT / 4; k += 4)
      *reinterpret_cast<uint4*>(p + 4 * k) = make_uint4(w[k], w[k + 1], w[k + 2], w[k + 3]);
  } else {
#pragma unroll
    for (int k = 0; k < COUT / 4; k += 2) *reinterpret_cast<uint2*>(p + 4 * k) = make_uint2(w[k], w[k + 1]);
  }
}

// ---- embedding lookup (Eq.4 Downsampling input, reading Q5; Q14 for E0) ------------
__global__ void k_embed(const int8_t* __restrict__ E, const uint8_t* __restrict__ X, uint32_t n, int C,
                        int8_t* __restrict__ out) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;  // one thread per 4 bytes
  const uint32_t wpr = C / 4;
  if (t >= (n + 1) * wpr) return;
  const uint32_t i = t / wpr, w = t % wpr;
  int32_t v = 0;
  if (i < n) v = reinterpret_cast<const int32_t*>(E + size_t(X[i] - 1) * C)[w];
  reinterpret_cast<int32_t*>(out + size_t(i) * C)[w] = v;
}

// ---- K3S1 sparse conv (Eq.5/8/10 ResBlock convs; P:337 indexed linear transforms) ----
// Thread per output row; the input row is Concat(in0 [C0], in1 [CIN-C0]) of the
// neighbour (reading Q7 "virtual concat"); absent neighbours index the zero row n.
template <int CIN, int COUT, int C0, int SKIP>
__global__ void __launch_bounds__(128) k_conv3(const int8_t* __restrict__ in0, const int8_t* __restrict__ in1, uint32_t n,
                                               const int32_t* __restrict__ nbr, const int8_t* __restrict__ W,
                                               const int32_t* __restrict__ bias, RQ rq,
                                               const int8_t* __restrict__ skip0, const int8_t* __restrict__ skip1,
                                               int32_t k_s, const int8_t* __restrict__ P, int8_t* __restrict__ out) {
  extern __shared__ int32_t smem[];
  constexpr int WIN = CIN / 4, W0 = C0 / 4, W1 = WIN - W0;
  int32_t* Ws = smem;                        // [27][COUT][WIN]
  int32_t* Ps = smem + 27 * COUT * WIN;      // [COUT][2*COUT/4] (SKIP == 2)
  for (int k = threadIdx.x; k < 27 * COUT * WIN; k += blockDim.x) Ws[k] = reinterpret_cast<const int32_t*>(W)[k];
  if (SKIP == 2)
    for (int k = threadIdx.x; k < COUT * (2 * COUT / 4); k += blockDim.x) Ps[k] = reinterpret_cast<const int32_t*>(P)[k];
  __syncthreads();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = i < n;
  int32_t acc[COUT];
#pragma unroll
  for (int o = 0; o < COUT; ++o) acc[o] = 0;
  for (int dl = 0; dl < 27; ++dl) {
    const int32_t j = active ? nbr[size_t(i) * 27 + dl] : int32_t(n);
    if (__all_sync(0xffffffffu, j == int32_t(n))) continue;
    int32_t x[WIN];
    load_row<W0>(in0 + size_t(j) * C0, x);
    if constexpr (W1 > 0) load_row<W1>(in1 + size_t(j) * (CIN - C0), x + W0);
    const int32_t* wr = Ws + dl * COUT * WIN;
#pragma unroll
    for (int o = 0; o < COUT; ++o) {
      int32_t a = acc[o];
#pragma unroll
      for (int w = 0; w < WIN; ++w) a = __dp4a(x[w], wr[o * WIN + w], a);
      acc[o] = a;
    }
  }
  if (i > n) return;
  int32_t q[COUT];
  if (i == n) {
#pragma unroll
    for (int o = 0; o < COUT; ++o) q[o] = 0;
  } else {
    if constexpr (SKIP == 1) {  // identity skip scaled by k_s (reading Q7)
      int32_t s[COUT / 4];
      load_row<COUT / 4>(skip0 + size_t(i) * COUT, s);
#pragma unroll
      for (int o = 0; o < COUT; ++o) acc[o] += k_s * int32_t(int8_t(uint32_t(s[o / 4]) >> (8 * (o % 4))));
    }
    if constexpr (SKIP == 2) {  // 1x1 projection of the 2C concat in the same accumulator
      int32_t s[2 * COUT / 4];
      load_row<COUT / 4>(skip0 + size_t(i) * COUT, s);
      load_row<COUT / 4>(skip1 + size_t(i) * COUT, s + COUT / 4);
#pragma unroll
      for (int o = 0; o < COUT; ++o) {
        int32_t a = acc[o];
#pragma unroll
        for (int w = 0; w < 2 * COUT / 4; ++w) a = __dp4a(s[w], Ps[o * (2 * COUT / 4) + w], a);
        acc[o] = a;
      }
    }
#pragma unroll
    for (int o = 0; o < COUT; ++o) q[o] = rq8(acc[o] + bias[o], rq);
  }
  store_row<COUT>(out + size_t(i) * COUT, q);
}

// ---- K2S2 down step (Eq.4, reading Q4): parent-side gather of <= 8 children --------
template <int C>
__global__ void __launch_bounds__(128) k_down(const int8_t* __restrict__ g, const uint8_t* __restrict__ Xp,
                                              const uint32_t* __restrict__ cs, uint32_t np, const int8_t* __restrict__ W,
                                              const int32_t* __restrict__ bias, RQ rq, int8_t* __restrict__ out) {
  // per-child blocks padded by 4 words so lanes with different child index c read
  // different banks
  constexpr int CB = C * C / 4 + 4;
  __shared__ int32_t Ws[8 * CB];
  for (int k = threadIdx.x; k < 8 * C * C / 4; k += blockDim.x)
    Ws[(k / (C * C / 4)) * CB + k % (C * C / 4)] = reinterpret_cast<const int32_t*>(W)[k];
  __syncthreads();
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > np) return;
  int32_t q[C];
  if (p == np) {
#pragma unroll
    for (int o = 0; o < C; ++o) q[o] = 0;
  } else {
    int32_t acc[C];
#pragma unroll
    for (int o = 0; o < C; ++o) acc[o] = 0;
    uint32_t x = Xp[p], j = cs[p];
    for (int c = 0; c < 8; ++c) {
      if (!((x >> c) & 1u)) continue;
      int32_t v[C / 4];
      load_row<C / 4>(g + size_t(j) * C, v);
      ++j;
      const int32_t* wr = Ws + c * CB;
#pragma unroll
      for (int o = 0; o < C; ++o) {
        int32_t a = acc[o];
#pragma unroll
        for (int w = 0; w < C / 4; ++w) a = __dp4a(v[w], wr[o * (C / 4) + w], a);
        acc[o] = a;
      }
    }
#pragma unroll
    for (int o = 0; o < C; ++o) q[o] = rq8(acc[o] + bias[o], rq);
  }
  store_row<C>(out + size_t(p) * C, q);
}

// ---- Upsampling + Pruning (Eq.6/9/11): thread per KEPT child row ------------------
// out[j] = prq(W_S[c] * S[par(j)] + q_one*W_X[c][X_par] + b[c]) with c = key(j) & 7.
// Only the unpruned 8x-expansion blocks are computed (identical result: Pruning
// "discards features of unoccupied child nodes").
template <int C>
__global__ void __launch_bounds__(128) k_up(const int8_t* __restrict__ S, const uint8_t* __restrict__ Xp,
                                            const uint32_t* __restrict__ par, const uint64_t* __restrict__ key_c,
                                            uint32_t nc, const int8_t* __restrict__ W, const int32_t* __restrict__ E,
                                            const int32_t* __restrict__ bias, RQ rq, int8_t* __restrict__ out) {
  // per-child blocks padded by 4 words so lanes with different child index c read
  // different banks
  constexpr int CB = C * C / 4 + 4;
  __shared__ int32_t Ws[8 * CB];
  for (int k = threadIdx.x; k < 8 * C * C / 4; k += blockDim.x)
    Ws[(k / (C * C / 4)) * CB + k % (C * C / 4)] = reinterpret_cast<const int32_t*>(W)[k];
  __syncthreads();
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j > nc) return;
  int32_t q[C];
  if (j == nc) {
#pragma unroll
    for (int o = 0; o < C; ++o) q[o] = 0;
  } else {
    const uint32_t p = par[j];
    const int c = int(key_c[j] & 7u);
    const int x = Xp[p];
    int32_t v[C / 4];
    load_row<C / 4>(S + size_t(p) * C, v);
    const int4* er4 = reinterpret_cast<const int4*>(E + size_t(x - 1) * (8 * C) + c * C);  // 16-B aligned rows
    const int4* br4 = reinterpret_cast<const int4*>(bias + c * C);
    int32_t eb[C];
#pragma unroll
    for (int k = 0; k < C / 4; ++k) {
      const int4 e4 = er4[k], b4 = br4[k];
      eb[4 * k] = e4.x + b4.x;
      eb[4 * k + 1] = e4.y + b4.y;
      eb[4 * k + 2] = e4.z + b4.z;
      eb[4 * k + 3] = e4.w + b4.w;
    }
    const int32_t* wr = Ws + c * CB;
#pragma unroll
    for (int o = 0; o < C; ++o) {
      int32_t a = eb[o];
#pragma unroll
      for (int w = 0; w < C / 4; ++w) a = __dp4a(v[w], wr[o * (C / 4) + w], a);
      q[o] = rq8(a, rq);
    }
  }
  store_row<C>(out + size_t(j) * C, q);
}

// ---- Predictor (Eq.7) + integer softmax to Q16 (Eq.15; readings Q20-Q22) -----------
// Warp per node.  Lane l owns symbols i = 8l .. 8l+7 (i = 255 is padding).
template <int C, int H, int MODE>
__global__ void __launch_bounds__(256) k_head_cdf(const int8_t* __restrict__ F, uint32_t n,
                                                  const int8_t* __restrict__ W1, const int32_t* __restrict__ b1, RQ rq1,
                                                  const int8_t* __restrict__ W2, const int32_t* __restrict__ b2, RQ rql,
                                                  const uint32_t* __restrict__ lut, const uint8_t* __restrict__ X,
                                                  uint32_t* __restrict__ cf, uint16_t* __restrict__ cdf,
                                                  int8_t* __restrict__ a_dbg) {
  constexpr int HW = H / 4, CW = C / 4;
  __shared__ int32_t W2s[HW * 256];   // word (w, i) at w*256 + (i&7)*32 + (i>>3)
  __shared__ int32_t W1s[H * CW];
  __shared__ int32_t b2s[256];
  __shared__ uint32_t luts[1024];
  for (int k = threadIdx.x; k < 256 * HW; k += blockDim.x) {
    const int i = k / HW, w = k % HW;  // W2 is [256][H] row-major
    W2s[w * 256 + (i & 7) * 32 + (i >> 3)] = reinterpret_cast<const int32_t*>(W2)[k];
  }
  for (int k = threadIdx.x; k < H * CW; k += blockDim.x) W1s[k] = reinterpret_cast<const int32_t*>(W1)[k];
  for (int k = threadIdx.x; k < 256; k += blockDim.x) b2s[k] = b2[k];
  for (int k = threadIdx.x; k < 1024; k += blockDim.x) luts[k] = lut[k];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint32_t node = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); node < n; node += warps) {
    // hidden layer a = prq(W1 F + b1)  (C -> H)
    int32_t fw = lane < CW ? reinterpret_cast<const int32_t*>(F + size_t(node) * C)[lane] : 0;
    int32_t ah = 0;
    if (lane < H) {
      int32_t acc = b1[lane];
#pragma unroll
      for (int w = 0; w < CW; ++w) acc = __dp4a(__shfl_sync(0xffffffffu, fw, w), W1s[lane * CW + w], acc);
      ah = rq8(acc, rq1);
    } else {
#pragma unroll
      for (int w = 0; w < CW; ++w) (void)__shfl_sync(0xffffffffu, fw, w);
    }
    if (a_dbg && lane < H) a_dbg[size_t(node) * H + lane] = int8_t(ah);
    int32_t aw[HW];
#pragma unroll
    for (int w = 0; w < HW; ++w)
      aw[w] = int32_t(pack4(__shfl_sync(0xffffffffu, ah, 4 * w), __shfl_sync(0xffffffffu, ah, 4 * w + 1),
                            __shfl_sync(0xffffffffu, ah, 4 * w + 2), __shfl_sync(0xffffffffu, ah, 4 * w + 3)));
    // logits z_i and Q8 requant l_i = clamp(round(z m / 2^r), +-2^24)
    int32_t l[8];
    int32_t lmax = INT32_MIN;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int i = 8 * lane + t;
      int32_t z = b2s[i];
#pragma unroll
      for (int w = 0; w < HW; ++w) z = __dp4a(aw[w], W2s[w * 256 + t * 32 + lane], z);
      int64_t v = int64_t(z) * int64_t(rql.mp);
      if (rql.r > 0) v = (v + (int64_t(1) << (rql.r - 1))) >> rql.r;
      v = v < -(int64_t(1) << 24) ? -(int64_t(1) << 24) : (v > (int64_t(1) << 24) ? (int64_t(1) << 24) : v);
      l[t] = int32_t(v);
      if (i < NCODE) lmax = max(lmax, l[t]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    // e_i = LUT[delta >> 2] (0 beyond 16 nats), S = sum e
    uint32_t e[8], jv[8];
    uint32_t s = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const uint32_t dl = uint32_t(lmax - l[t]);
      jv[t] = min(dl, 4096u) >> 2;  // decoder row entry (1024: e = 0)
      e[t] = (8 * lane + t < NCODE && dl < 4096u) ? luts[dl >> 2] : 0u;
      s += e[t];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    // reading Q21: C_i = i + floor(E_i * 65281 / S), E_i = sum_{j<i} e_j (exact: reciprocal
    // inv = floor((2^64-1)/S), then one integer correction)
    uint32_t ls = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) ls += e[t];
    uint32_t inc = ls;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    const uint64_t inv = ~0ull / uint64_t(s);
    auto Cq = [&](uint32_t E, int i) -> uint32_t {  // C_i for prefix mass E
      const uint64_t num = uint64_t(E) * 65281ull;
      uint64_t qq = __umul64hi(num, inv);
      if (num - qq * uint64_t(s) >= uint64_t(s)) ++qq;
      return uint32_t(i) + uint32_t(qq);
    };
    uint32_t E = inc - ls;  // mass before this lane's symbols
    if constexpr (MODE == 0) {
      const int sym = int(X[node]) - 1;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int i = 8 * lane + t;
        if (i == sym) {
          const uint32_t c0 = Cq(E, i), c1 = Cq(E + e[t], i + 1);
          cf[node] = c0 | ((c1 - c0) << 16);
        }
        E += e[t];
      }
    } else {
      // decoder row (pcc_internal.cuh DROW_*): S, inv32, mu, E_{16k} (k = 1..15), a
      uint8_t* row = reinterpret_cast<uint8_t*>(cdf) + size_t(node) * DROW_BYTES;
      uint32_t* hdr = reinterpret_cast<uint32_t*>(row);
      if (lane == 0) {
        hdr[0] = s;
        hdr[1] = uint32_t((65281ull << 32) / uint64_t(s));
        hdr[2] = uint32_t(lmax);
        hdr[18] = hdr[19] = 0u;
      } else if ((lane & 1) == 0) {
        hdr[2 + lane / 2] = E;  // mass before symbol 8 lane = 16 (lane / 2)
      }
      if (lane < 8) {
        uint32_t av = 0u;
#pragma unroll
        for (int w = 0; w < HW; ++w) av = (w == lane) ? uint32_t(aw[w]) : av;
        reinterpret_cast<uint32_t*>(row + DROW_A)[lane] = av;
      }
      (void)jv;
    }
  }
}

inline unsigned cdiv(size_t a, size_t b) { return unsigned((a + b - 1) / b); }

template <int CIN, int COUT, int C0, int SKIP>
void launch_conv3(pcc_ctx c, const int8_t* in0, const int8_t* in1, uint32_t n, const int32_t* nbr, const DConv& L,
                  const int8_t* s0, const int8_t* s1, int32_t k_s, const int8_t* P, int8_t* out) {
  const size_t smem = (27 * COUT * (CIN / 4) + (SKIP == 2 ? COUT * (2 * COUT / 4) : 0)) * sizeof(int32_t);
  auto kern = k_conv3<CIN, COUT, C0, SKIP>;
  PCC_SMEM_ATTR(kern, 200 * 1024);
  Prof p(c, "conv", size_t(n) * (CIN + COUT + 27 * 4 + (SKIP ? (SKIP == 2 ? 2 * COUT : COUT) : 0)));
  kern<<<cdiv(size_t(n) + 1, 128), 128, smem, c->stream>>>(in0, in1, n, nbr, L.W, L.b, L.rq, s0, s1, k_s, P, out);
  launched(c);
}

template <int C>
void conv3_c(pcc_ctx c, const int8_t* in0, const int8_t* in1, uint32_t n, const int32_t* nbr, const DConv& L,
             int skip_mode, const int8_t* s0, const int8_t* s1, int32_t k_s, const int8_t* P, int8_t* out) {
  if (in1) {
    if (skip_mode == 0) launch_conv3<2 * C, C, C, 0>(c, in0, in1, n, nbr, L, s0, s1, k_s, P, out);
    else throw Error{PCC_ERR_INVALID_ARG};
  } else {
    if (skip_mode == 0) launch_conv3<C, C, C, 0>(c, in0, nullptr, n, nbr, L, s0, s1, k_s, P, out);
    else if (skip_mode == 1) launch_conv3<C, C, C, 1>(c, in0, nullptr, n, nbr, L, s0, s1, k_s, P, out);
    else launch_conv3<C, C, C, 2>(c, in0, nullptr, n, nbr, L, s0, s1, k_s, P, out);
  }
}

}  // namespace

void embed(pcc_ctx c, const int8_t* E, const uint8_t* X, uint32_t n, int C, int8_t* out) {
  size_t t = size_t(n + 1) * (C / 4);
  Prof p(c, "embed", size_t(n) * (1 + C));
  k_embed<<<cdiv(t, 256), 256, 0, c->stream>>>(E, X, n, C, out);
  launched(c);
}

void conv3(pcc_ctx c, const int8_t* in0, const int8_t* in1, int C, uint32_t n, const int32_t* nbr, const DConv& L,
           int skip_mode, const int8_t* s0, const int8_t* s1, int32_t k_s, const int8_t* P, int8_t* out) {
  // C = 32: gather -> tcgen05 kind::i8 per kernel offset (conv_tc.cu); PCC_CONV=simt
  // keeps the dp4a kernel (A/B baseline, bit-exact with it).
  static const bool simt = [] {
    const char* e = getenv("PCC_CONV");
    return e && std::string(e) == "simt";
  }();
  if (C == 32 && !simt) {
    conv3_tc(c, in0, in1, n, nbr, L, skip_mode, s0, s1, k_s, P, out);
    return;
  }
  switch (C) {
    case 8: conv3_c<8>(c, in0, in1, n, nbr, L, skip_mode, s0, s1, k_s, P, out); break;
    case 16: conv3_c<16>(c, in0, in1, n, nbr, L, skip_mode, s0, s1, k_s, P, out); break;
    case 32: conv3_c<32>(c, in0, in1, n, nbr, L, skip_mode, s0, s1, k_s, P, out); break;
    default: throw Error{PCC_ERR_INVALID_ARG};
  }
}

void down(pcc_ctx c, const int8_t* g, const uint8_t* Xp, const uint32_t* cs_p, uint32_t np, int C, const DDown& L,
          int8_t* out) {
  const unsigned grid = cdiv(size_t(np) + 1, 128);
  Prof p(c, "down", size_t(np) * (1 + 4 + C));
  switch (C) {
    case 8: k_down<8><<<grid, 128, 0, c->stream>>>(g, Xp, cs_p, np, L.W, L.b, L.rq, out); break;
    case 16: k_down<16><<<grid, 128, 0, c->stream>>>(g, Xp, cs_p, np, L.W, L.b, L.rq, out); break;
    case 32: k_down<32><<<grid, 128, 0, c->stream>>>(g, Xp, cs_p, np, L.W, L.b, L.rq, out); break;
    default: throw Error{PCC_ERR_INVALID_ARG};
  }
  launched(c);
}

void up_prune(pcc_ctx c, const int8_t* S, const uint8_t* Xp, const uint32_t* par_c, const uint64_t* key_c, uint32_t nc,
              int C, const DUp& L, int8_t* out) {
  const unsigned grid = cdiv(size_t(nc) + 1, 128);
  Prof p(c, "up", size_t(nc) * (4 + 8 + 2 * C));
  switch (C) {
    case 8: k_up<8><<<grid, 128, 0, c->stream>>>(S, Xp, par_c, key_c, nc, L.W, L.E, L.b, L.rq, out); break;
    case 16: k_up<16><<<grid, 128, 0, c->stream>>>(S, Xp, par_c, key_c, nc, L.W, L.E, L.b, L.rq, out); break;
    case 32: k_up<32><<<grid, 128, 0, c->stream>>>(S, Xp, par_c, key_c, nc, L.W, L.E, L.b, L.rq, out); break;
    default: throw Error{PCC_ERR_INVALID_ARG};
  }
  launched(c);
}

template <int C, int H>
static void head_ch(pcc_ctx c, const int8_t* F, uint32_t n, const DHead& L, const uint32_t* lut, int mode,
                    const uint8_t* X, uint32_t* cf, uint16_t* cdf, int8_t* a_dbg) {
  const unsigned grid = std::max(1u, std::min(cdiv(n, 8), unsigned(c->sm_count) * 8u));
  Prof p(c, mode == 0 ? "head_enc" : "head_dec", size_t(n) * (C + (mode == 0 ? 1 + 4 : DROW_BYTES)));
  if (mode == 0)
    k_head_cdf<C, H, 0><<<grid, 256, 0, c->stream>>>(F, n, L.W1, L.b1, L.rq1, L.W2, L.b2, L.rql, lut, X, cf, cdf, a_dbg);
  else
    k_head_cdf<C, H, 1><<<grid, 256, 0, c->stream>>>(F, n, L.W1, L.b1, L.rq1, L.W2, L.b2, L.rql, lut, X, cf, cdf, a_dbg);
  launched(c);
}

void head_cdf(pcc_ctx c, const int8_t* F, uint32_t n, int C, int H, const DHead& L, const uint32_t* lut, int mode,
              const uint8_t* X, uint32_t* cf, uint16_t* cdf, int8_t* a_dbg) {
  if (n == 0) return;
  if (C == 8 && H == 8) head_ch<8, 8>(c, F, n, L, lut, mode, X, cf, cdf, a_dbg);
  else if (C == 16 && H == 16) head_ch<16, 16>(c, F, n, L, lut, mode, X, cf, cdf, a_dbg);
  else if (C == 32 && H == 32) head_ch<32, 32>(c, F, n, L, lut, mode, X, cf, cdf, a_dbg);
  else throw Error{PCC_ERR_INVALID_ARG};
}

}  // namespace pcc
