// runtime.cu — C ABI (include/pcc.h), model upload, workspace arena, level scheduler
// (Eq.2 level-wise autoregression: the encoder knows every level and runs the
// shallow chain then the four deep levels; the decoder is level-serial and parallel
// within a level), and the bitstream container (reading O11).
#include <algorithm>
#include <cstring>
#include <string>

#include "pcc_internal.cuh"
#include "rq.cuh"

using namespace pcc;

// ============================================================================
// arena / bookkeeping
// ============================================================================
namespace pcc {

void* ws(pcc_ctx c, const char* name, size_t bytes) {
  auto& b = c->bufs[name];
  if (b.cap < bytes) {
    if (b.p) PCC_CUDA(cudaFree(b.p));
    b.p = nullptr;
    size_t cap = std::max<size_t>(bytes + bytes / 4, 256);
    if (cudaMalloc(&b.p, cap) != cudaSuccess) {
      b.cap = 0;
      throw Error{PCC_ERR_OOM};
    }
    b.cap = cap;
  }
  return b.p;
}

void* pinned(pcc_ctx c, size_t bytes) {
  // a ring of pinned staging; callers synchronise before reuse
  if (c->pinned_cap < bytes) {
    if (c->pinned) cudaFreeHost(c->pinned);
    c->pinned = nullptr;
    size_t cap = std::max<size_t>(bytes * 2, 1 << 20);
    PCC_CUDA(cudaMallocHost(&c->pinned, cap));
    c->pinned_cap = cap;
  }
  return c->pinned;
}

// Called after every launch: counts it and surfaces a failed launch (bad configuration,
// shared-memory limit) immediately instead of as a wrong result later.
void* pinned_ring(pcc_ctx c, size_t bytes) {
  if (c->pinned1_cap < bytes) {
    if (c->pinned1) cudaFreeHost(c->pinned1);
    c->pinned1 = nullptr;
    size_t cap = std::max<size_t>(bytes * 2, 1 << 16);
    PCC_CUDA(cudaMallocHost(&c->pinned1, cap));
    c->pinned1_cap = cap;
  }
  return c->pinned1;
}

void launched(pcc_ctx c, int n) {
  c->launches += uint64_t(n);
  PCC_CUDA(cudaPeekAtLastError());
}

static cudaEvent_t ev_get(pcc_ctx c) {
  if (!c->pool.empty()) {
    cudaEvent_t e = c->pool.back();
    c->pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  PCC_CUDA(cudaEventCreate(&e));
  return e;
}

Prof::Prof(pcc_ctx c_, const char* cat_, uint64_t bytes_) : c(c_), cat(cat_), bytes(bytes_) {
  if (!c->prof) return;
  a = ev_get(c);
  b = ev_get(c);
  cudaEventRecord(a, c->stream);
}

Prof::~Prof() {
  if (!a) return;
  cudaEventRecord(b, c->stream);
  c->recs.push_back(pcc_ctx_s::Rec{cat, a, b, bytes});
}

void prof_collect(pcc_ctx c) {
  if (c->recs.empty()) return;
  cudaStreamSynchronize(c->stream);
  for (auto& r : c->recs) {
    float ms = 0;
    cudaEventElapsedTime(&ms, r.a, r.b);
    auto& t = c->tot[r.cat];
    t.ms += ms;
    t.launches += 1;
    t.bytes += r.bytes;
    c->pool.push_back(r.a);
    c->pool.push_back(r.b);
  }
  c->recs.clear();
}

void dbg_copy(pcc_ctx c, const std::string& name, const void* dptr, size_t bytes) {
  if (!c->debug) return;
  std::vector<uint8_t>& v = c->dbg[name];
  v.resize(bytes);
  if (bytes) {
    PCC_CUDA(cudaStreamSynchronize(c->stream));
    PCC_CUDA(cudaMemcpy(v.data(), dptr, bytes, cudaMemcpyDeviceToHost));
  }
}

}  // namespace pcc

namespace {

inline unsigned cdiv(size_t a, size_t b) { return unsigned((a + b - 1) / b); }

// Predictor + softmax: by default the one-thread-per-node kernel with N = 128 half
// accumulators and 4 tile groups per SM (head3_tc.cu); PCC_HEAD=t3g3 the same with 3 groups,
// t1 the full-width one-thread-per-node kernel (head1_tc.cu, 2 groups), t2 two threads per
// node (head2_tc.cu), q4 the round-1 kernel (4 threads per node), simt the dp4a warp-per-node
// kernel (A/B baselines; all bit-exact).  Measured per 1024-frame cfg2 step (dec / enc ms):
// head3 g4 9.5 / 10.4, g3 10.1 / 11.5, head1 9.7 / 11.7, head2 10.5 / 11.6, q4 12.9 / 12.5.
void head_any(pcc_ctx c, const int8_t* F, uint32_t n, int C, int H, const DHead& L, const uint32_t* lut, int mode,
              const uint8_t* X, uint32_t* cf, uint16_t* cdf, int8_t* a_dbg) {
  static const int which = [] {
    const char* e = getenv("PCC_HEAD");
    if (e && std::string(e) == "simt") return 2;
    if (e && std::string(e) == "q4") return 1;
    if (e && std::string(e) == "t2") return 3;
    if (e && std::string(e) == "t3g3") return 4;
    if (e && std::string(e) == "t1") return 6;
    if (e && std::string(e) == "t3") return 5;
    return 7;  // default: head4 (both layers and biases on tcgen05), head3 if a bias is too large
  }();
  if (which == 7 && L.bias_fold) {
    head_cdf_tc4(c, F, n, C, H, L, lut, mode, X, cf, cdf, a_dbg);
    return;
  }
  if (which == 4 || which == 5 || which == 7) {
    head_cdf_tc3(c, F, n, C, H, L, lut, mode, X, cf, cdf, a_dbg, which == 4 ? 3 : 4);
    return;
  }
  if (which == 2) head_cdf(c, F, n, C, H, L, lut, mode, X, cf, cdf, a_dbg);
  else if (which == 1) head_cdf_tc(c, F, n, C, H, L, lut, mode, X, cf, cdf, a_dbg);
  else if (which == 3) head_cdf_tc2(c, F, n, C, H, L, lut, mode, X, cf, cdf, a_dbg);
  else head_cdf_tc1(c, F, n, C, H, L, lut, mode, X, cf, cdf, a_dbg);  // which == 6
}

// b = 127 sum_{j<31} d_j + d_31 with |d_j| <= 127 and d_31 = b mod 127 in [0, 126], one
// row of 32 digits per bias; false when some |b| is too large for 31 digits
bool bias_digits(const std::vector<int32_t>& b, std::vector<int8_t>& D) {
  D.assign(b.size() * 32, 0);
  for (size_t i = 0; i < b.size(); ++i) {
    const int64_t v = b[i];
    const int64_t rem = ((v % 127) + 127) % 127;
    int64_t q = (v - rem) / 127;
    if (q > 31 * 127 || q < -31 * 127) return false;
    for (int j = 0; j < 31; ++j) {
      const int64_t d = q > 127 ? 127 : (q < -127 ? -127 : q);
      D[i * 32 + j] = int8_t(d);
      q -= d;
    }
    D[i * 32 + 31] = int8_t(rem);
  }
  return true;
}

inline int lanes_for(uint32_t n) {
  uint32_t k = (n + 511u) / 512u;
  return int(k < 1u ? 1u : (k > 8u ? 8u : k));
}

// ============================================================================
// model file -> device
// ============================================================================
struct Rd {
  const uint8_t* p;
  size_t n, pos = 0;
  void need(size_t k) {
    if (pos + k > n) throw Error{PCC_ERR_INVALID_ARG};
  }
  uint32_t u32() {
    need(4);
    uint32_t v;
    std::memcpy(&v, p + pos, 4);
    pos += 4;
    return v;
  }
  int32_t i32() { return int32_t(u32()); }
  const uint8_t* take(size_t k) {
    need(k);
    const uint8_t* q = p + pos;
    pos += k;
    return q;
  }
  RQ rq() {
    RQ t;
    t.mp = i32();
    t.mn = i32();
    t.r = i32();
    // reading O5: m in [0, 2^31), r in [0, 62] (m >= 0 keeps every requant monotone)
    if (t.r < 0 || t.r > 62 || t.mp < 0 || t.mn < 0) throw Error{PCC_ERR_INVALID_ARG};
    rq_prepare(t);
    return t;
  }
};

struct Stage {  // host image of the device model buffer
  std::vector<uint8_t> img;
  size_t put(const void* src, size_t bytes) {
    size_t off = (img.size() + 255) & ~size_t(255);
    img.resize(off + bytes);
    if (bytes) std::memcpy(img.data() + off, src, bytes);
    return off;
  }
};

uint64_t fnv1a(const uint8_t* p, size_t n) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ull;
  }
  return h;
}

// For l(z) = floor((z*m + h) / 2^r), h = 2^(r-1) (0 if r = 0), m >= 0, clamped to
// [-T, T] with T = 2^24 (reading Q20): the int32 thresholds such that z > hi <=> l(z) >= T
// and z < lo <=> l(z) <= -T.  Strictly between them |l| < T, so a kernel may compute
// l from the low 32 bits of the 64-bit shift and skip the 64-bit clamp (exact).
void logit_saturation(const RQ& q, int32_t& lo, int32_t& hi) {
  const __int128 T = __int128(1) << 24;
  const __int128 two_r = __int128(1) << q.r;
  const __int128 h = q.r > 0 ? (__int128(1) << (q.r - 1)) : 0;
  auto ceil_div = [](__int128 a, __int128 b) {  // b > 0
    __int128 qq = a / b;
    if (qq * b < a) ++qq;  // C++ division truncates toward zero
    return qq;
  };
  __int128 zhi, zlo;  // zhi = min z with l >= T; zlo = max z with l <= -T
  if (q.mp == 0) {
    zhi = __int128(INT32_MAX) + 1;
    zlo = __int128(INT32_MIN) - 1;
  } else {
    zhi = ceil_div(T * two_r - h, q.mp);
    zlo = ceil_div((1 - T) * two_r - h, q.mp) - 1;
  }
  __int128 hx = zhi - 1, lx = zlo + 1;  // exclusive forms: z > hx, z < lx
  if (hx > INT32_MAX) hx = INT32_MAX;
  if (hx < INT32_MIN) hx = INT32_MIN;
  if (lx < INT32_MIN) lx = INT32_MIN;
  if (lx > INT32_MAX) lx = INT32_MAX;
  hi = int32_t(hx);
  lo = int32_t(lx);
}

// Pointers are staged as offsets and rebased after the single cudaMalloc.
template <class T>
T* off_ptr(size_t off) {
  return reinterpret_cast<T*>(off);
}
template <class T>
T* rebase(T* p, uint8_t* base) {
  return reinterpret_cast<T*>(base + reinterpret_cast<size_t>(p));
}

pcc_model load_model(const uint8_t* bytes, size_t len, int device) {
  if (len < 72 || std::memcmp(bytes, "PCCM", 4) != 0) throw Error{PCC_ERR_INVALID_ARG};
  uint64_t h;
  std::memcpy(&h, bytes + len - 8, 8);
  if (fnv1a(bytes, len - 8) != h) throw Error{PCC_ERR_MODEL_MISMATCH};
  Rd r{bytes, len - 8};
  r.pos = 4;
  if (r.u32() != 1) throw Error{PCC_ERR_VERSION};
  auto* m = new pcc_model_s();
  try {
    m->device = device;
    m->hash = h;
    m->C = int(r.u32());
    m->H = int(r.u32());
    m->R = int(r.u32());
    m->n_deep = int(r.u32());
    m->min_depth = int(r.u32());
    m->max_depth = int(r.u32());
    const int C = m->C, H = m->H;
    // n_deep = 0: the GRED-off Table 4 "Baseline" (every level shallow); R <= 6 keeps the
    // raw prefix (<= 37449 nodes) inside the container's u16 raw_bytes field
    if (!(C == 8 || C == 16 || C == 32) || H != C || m->n_deep < 0 || m->n_deep > 4 || m->R < 1 || m->R > 6 ||
        m->max_depth > MAX_DEPTH || m->min_depth < m->R + 1 + m->n_deep || m->max_depth < m->min_depth)
      throw Error{PCC_ERR_INVALID_ARG};
    r.pos = 40;
    if (r.u32() != 1024) throw Error{PCC_ERR_INVALID_ARG};
    m->flags = r.u32();
    if (m->flags & ~MF_ALL) throw Error{PCC_ERR_INVALID_ARG};
    r.pos = 64;
    Stage st;
    {
      // exp table (reading Q20) must be a softmax table: LUT[0] in (65281, 2^24] and
      // non-increasing, so S = sum e lies in (65281, 255 * 2^24]: u32 row sums, no division
      // by zero, and inv32 = floor(65281 * 2^32 / S) < 2^32 (the decoder rows)
      if (len < 64 + 4096 + 8) throw Error{PCC_ERR_INVALID_ARG};
      uint32_t lut[1024];
      std::memcpy(lut, bytes + 64, 4096);
      if (lut[0] <= 65281u || lut[0] > (1u << 24)) throw Error{PCC_ERR_INVALID_ARG};
      for (int j = 1; j < 1024; ++j)
        if (lut[j] > lut[j - 1]) throw Error{PCC_ERR_INVALID_ARG};
    }
    size_t o_lut = st.put(r.take(4096), 4096);
    size_t o_E0 = st.put(r.take(size_t(NCODE) * C), size_t(NCODE) * C);
    auto conv = [&](int cin) {
      DConv cv;
      size_t w = st.put(r.take(size_t(27) * C * cin), size_t(27) * C * cin);
      size_t b = st.put(r.take(size_t(4) * C), size_t(4) * C);
      cv.W = off_ptr<const int8_t>(w);
      cv.b = off_ptr<const int32_t>(b);
      return cv;
    };
    auto up = [&]() {
      DUp u;
      const uint8_t* W = r.take(size_t(8) * C * (C + NCODE));
      std::vector<int8_t> WS(size_t(8) * C * C);
      for (int o = 0; o < 8 * C; ++o)
        for (int i = 0; i < C; ++i) WS[size_t(o) * C + i] = int8_t(W[size_t(o) * (C + NCODE) + i]);
      const uint8_t* b = r.take(size_t(4) * 8 * C);
      u.rq = r.rq();
      const int32_t q_one = r.i32();
      if (q_one < -128 || q_one > 127) throw Error{PCC_ERR_INVALID_ARG};  // an int8 activation
      std::vector<int32_t> E(size_t(NCODE) * 8 * C);  // E[v][o] = q_one * W[o][C + v] (exact)
      for (int v = 0; v < NCODE; ++v)
        for (int o = 0; o < 8 * C; ++o) E[size_t(v) * 8 * C + o] = q_one * int32_t(int8_t(W[size_t(o) * (C + NCODE) + C + v]));
      std::vector<int8_t> WXt(size_t(NCODE) * 8 * C);
      for (int v = 0; v < NCODE; ++v)
        for (int o = 0; o < 8 * C; ++o) WXt[size_t(v) * 8 * C + o] = int8_t(W[size_t(o) * (C + NCODE) + C + v]);
      u.q_one = q_one;
      u.W = off_ptr<const int8_t>(st.put(WS.data(), WS.size()));
      u.E = off_ptr<const int32_t>(st.put(E.data(), E.size() * 4));
      u.b = off_ptr<const int32_t>(st.put(b, size_t(4) * 8 * C));
      u.WXt = off_ptr<const int8_t>(st.put(WXt.data(), WXt.size()));
      return u;
    };
    auto head = [&]() {
      DHead hd;
      hd.W1 = off_ptr<const int8_t>(st.put(r.take(size_t(H) * C), size_t(H) * C));
      const uint8_t* b1p = r.take(size_t(4) * H);
      std::vector<int32_t> hd_b1_host(H);
      std::memcpy(hd_b1_host.data(), b1p, size_t(4) * H);
      hd.b1 = off_ptr<const int32_t>(st.put(b1p, size_t(4) * H));
      hd.rq1 = r.rq();
      std::vector<int8_t> W2(size_t(256) * H, 0);
      std::memcpy(W2.data(), r.take(size_t(NCODE) * H), size_t(NCODE) * H);
      std::vector<int32_t> b2(256, 0);
      std::memcpy(b2.data(), r.take(size_t(4) * NCODE), size_t(4) * NCODE);
      hd.rql = r.rq();
      logit_saturation(hd.rql, hd.zsat_lo, hd.zsat_hi);
      {  // |z_i| <= |b2_i| + 128 * sum_h |W2_ih| since |a_h| <= 128
        int64_t zb = 0;
        for (int i = 0; i < NCODE; ++i) {
          int64_t s = std::abs(int64_t(b2[i]));
          for (int h2 = 0; h2 < H; ++h2) s += 128 * std::abs(int64_t(W2[size_t(i) * H + h2]));
          zb = std::max(zb, s);
        }
        hd.can_saturate = zb > hd.zsat_hi || -zb < hd.zsat_lo;
      }
      hd.W2 = off_ptr<const int8_t>(st.put(W2.data(), W2.size()));
      hd.b2 = off_ptr<const int32_t>(st.put(b2.data(), b2.size() * 4));
      {  // bias digits for head4_tc.cu: b = 127 sum_{j<31} d_j + d_31, d_31 = b mod 127
        std::vector<int32_t> b1(32, 0);
        std::memcpy(b1.data(), hd_b1_host.data(), size_t(4) * H);
        std::vector<int8_t> D1, D2;
        hd.bias_fold = bias_digits(b1, D1) && bias_digits(b2, D2);
        hd.B1d = off_ptr<const int8_t>(st.put(D1.data(), D1.size()));
        hd.B2d = off_ptr<const int8_t>(st.put(D2.data(), D2.size()));
      }
      return hd;
    };
    for (int d = m->R; d < m->max_depth - m->n_deep; ++d) {
      DShallow s;
      s.a = conv(C);
      s.a.rq = r.rq();
      s.b = conv(C);
      s.k_s = r.i32();
      s.b.rq = r.rq();
      s.up = up();
      s.head = head();
      m->shallow.push_back(s);
    }
    for (int j = 1; j <= m->n_deep; ++j) {
      DDeep dp{};
      dp.E = off_ptr<const int8_t>(st.put(r.take(size_t(NCODE) * C), size_t(NCODE) * C));
      for (int s = 0; s < j - 1; ++s) {
        dp.down[s].W = off_ptr<const int8_t>(st.put(r.take(size_t(8) * C * C), size_t(8) * C * C));
        dp.down[s].b = off_ptr<const int32_t>(st.put(r.take(size_t(4) * C), size_t(4) * C));
        dp.down[s].rq = r.rq();
      }
      if (m->flags & MF_XFP_OFF) {  // ResBlock(G_D) in the shallow layout (P:528 ablation)
        dp.a = conv(C);
        dp.a.rq = r.rq();
        dp.b = conv(C);
        dp.k_s = r.i32();
        dp.b.rq = r.rq();
        dp.P = nullptr;
      } else {
        dp.a = conv(2 * C);
        dp.a.rq = r.rq();
        dp.b.W = off_ptr<const int8_t>(st.put(r.take(size_t(27) * C * C), size_t(27) * C * C));
        dp.P = off_ptr<const int8_t>(st.put(r.take(size_t(C) * 2 * C), size_t(C) * 2 * C));
        dp.b.b = off_ptr<const int32_t>(st.put(r.take(size_t(4) * C), size_t(4) * C));
        dp.b.rq = r.rq();
        dp.k_s = 0;
      }
      for (int s = 0; s < j; ++s) dp.up[s] = up();
      dp.head = head();
      m->deep.push_back(dp);
    }
    if (r.pos != r.n) throw Error{PCC_ERR_INVALID_ARG};
    m->file.assign(bytes, bytes + len);
    PCC_CUDA(cudaSetDevice(device));
    PCC_CUDA(cudaMalloc(&m->dmem, st.img.size()));
    PCC_CUDA(cudaMemcpy(m->dmem, st.img.data(), st.img.size(), cudaMemcpyHostToDevice));
    uint8_t* base = static_cast<uint8_t*>(m->dmem);
    m->lut = reinterpret_cast<const uint32_t*>(base + o_lut);
    m->E0 = reinterpret_cast<const int8_t*>(base + o_E0);
    auto rb_head = [&](DHead& hd) {
      hd.W1 = rebase(hd.W1, base); hd.b1 = rebase(hd.b1, base); hd.W2 = rebase(hd.W2, base); hd.b2 = rebase(hd.b2, base);
      hd.B1d = rebase(hd.B1d, base); hd.B2d = rebase(hd.B2d, base);
    };
    auto rb_up = [&](DUp& u) {
      u.W = rebase(u.W, base); u.E = rebase(u.E, base); u.b = rebase(u.b, base); u.WXt = rebase(u.WXt, base);
    };
    for (auto& s : m->shallow) {
      s.a.W = rebase(s.a.W, base); s.a.b = rebase(s.a.b, base);
      s.b.W = rebase(s.b.W, base); s.b.b = rebase(s.b.b, base);
      rb_up(s.up);
      rb_head(s.head);
    }
    for (int j = 1; j <= m->n_deep; ++j) {
      DDeep& dp = m->deep[j - 1];
      dp.E = rebase(dp.E, base);
      for (int s = 0; s < j - 1; ++s) { dp.down[s].W = rebase(dp.down[s].W, base); dp.down[s].b = rebase(dp.down[s].b, base); }
      dp.a.W = rebase(dp.a.W, base); dp.a.b = rebase(dp.a.b, base);
      dp.b.W = rebase(dp.b.W, base); dp.b.b = rebase(dp.b.b, base);
      if (dp.P) dp.P = rebase(dp.P, base);
      for (int s = 0; s < j; ++s) rb_up(dp.up[s]);
      rb_head(dp.head);
    }
  } catch (...) {
    if (m->dmem) cudaFree(m->dmem);
    delete m;
    throw;
  }
  return m;
}

void check_device(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device || device < 0) throw Error{PCC_ERR_CUDA};
  cudaDeviceProp p;
  PCC_CUDA(cudaGetDeviceProperties(&p, device));
  if (p.major != 10) throw Error{PCC_ERR_CUDA};  // sm_100 only: no fallback path exists
}

void check_depth(pcc_model m, int L) {
  if (L < m->R + 1 + m->n_deep || L < m->min_depth || L > m->max_depth || L > MAX_DEPTH)
    throw Error{PCC_ERR_UNSUPPORTED_DEPTH};
}

template <class T>
T* buf(pcc_ctx c, const std::string& name, size_t count) {
  return wsT<T>(c, name.c_str(), count);
}

std::string nm(const char* a, int x) { return std::string(a) + "/" + std::to_string(x); }
std::string nm(const char* a, int x, int y) { return std::string(a) + "/" + std::to_string(x) + "/" + std::to_string(y); }

// ============================================================================
// per-level context network (Eq.4-11), shared by encoder and decoder
// ============================================================================
struct Net {
  pcc_ctx c;
  pcc_model m;
  int L, R, D, C;
  const OctreeOut& o;
  uint64_t* key() { return static_cast<uint64_t*>(c->bufs.at("key").p); }
  uint8_t* code() { return static_cast<uint8_t*>(c->bufs.at("code").p); }
  uint32_t* cs() { return static_cast<uint32_t*>(c->bufs.at("cs").p); }
  uint32_t* par() { return static_cast<uint32_t*>(c->bufs.at("par").p); }
  const uint8_t* X(int d) { return code() + o.nb[d]; }
  size_t rows(int d) { return size_t(o.N[d]) + 1; }
  int8_t* F(int d) { return buf<int8_t>(c, nm("F", d), rows(d) * C); }
  int32_t* nbr(int d) { return buf<int32_t>(c, nm("nbr", d), size_t(o.N[d]) * 27); }

  void dbgF(const std::string& name, const int8_t* p, uint32_t n, int width) { dbg_copy(c, name, p, size_t(n) * width); }

  // Upsampling + Pruning from depth k to k+1 (Eq.6/9/11).  C = 32: the tcgen05 kernel
  // (up_tc.cu; 2.1 vs 4.5 ms per B=256 step for the dp4a kernel); PCC_UP=simt selects the
  // dp4a kernel (bit-exact, same contract; also the path for C != 32).
  void up(int k, const int8_t* S, const DUp& L, int8_t* dst) {
    static const bool simt = [] {
      const char* e = getenv("PCC_UP");
      return e && std::string(e) == "simt";
    }();
    if (C == 32 && !simt)
      up_prune_tc(c, S, X(k), par() + o.nb[k + 1], key() + o.nb[k + 1], o.N[k + 1], L, dst);
    else
      up_prune(c, S, X(k), par() + o.nb[k + 1], key() + o.nb[k + 1], o.N[k + 1], C, L, dst);
  }

  // depth of the last kernel map built in this call (-1: none): kernel maps are needed at
  // consecutive depths R-1..D, so every one after the first is derived from its parent's
  // (kmap.cu k_kmap_derive); PCC_KMAP=hash hashes every depth (A/B baseline)
  int kmap_last = -1;
  void kmap(int d) {
    static const bool hash_all = [] {
      const char* e = getenv("PCC_KMAP");
      return e && std::string(e) == "hash";
    }();
    if (!hash_all && d >= 1 && kmap_last == d - 1)
      kernel_map_derive(c, key() + o.nb[d], par() + o.nb[d], o.N[d], nbr(d - 1), o.N[d - 1], X(d - 1),
                        cs() + o.nb[d - 1], nbr(d));
    else
      kernel_map(c, key() + o.nb[d], o.N[d], d, nbr(d));
    kmap_last = d;
    if (c->debug) dbg_copy(c, nm("nbr", d), nbr(d), size_t(o.N[d]) * 27 * 4);
  }

  // Returns the feature map of the depth-d nodes that the predictor of coded level d
  // consumes (Eq.7 input F^l): shallow F_d (Eq.8-9) or deep F'_d (Eq.4, 10-11).
  const int8_t* level(int d) {
    if (d <= D) {
      const DShallow& s = m->shallow[d - m->R];
      const uint32_t n = o.N[d - 1];
      if (d == R) {  // reading Q14: F_{R-1} = E0[X_{R-1}]
        embed(c, m->E0, X(d - 1), n, C, F(d - 1));
        dbgF(nm("F", d - 1), F(d - 1), n, C);
      }
      kmap(d - 1);
      int8_t* h = buf<int8_t>(c, "t_h", rows(d - 1) * C);
      int8_t* S = buf<int8_t>(c, "t_S", rows(d - 1) * C);
      conv3(c, F(d - 1), nullptr, C, n, nbr(d - 1), s.a, 0, nullptr, nullptr, 0, nullptr, h);  // Eq.8 conv_a + PReLU
      dbgF(nm("ha", d), h, n, C);
      conv3(c, h, nullptr, C, n, nbr(d - 1), s.b, 1, F(d - 1), nullptr, s.k_s, nullptr, S);   // conv_b + k_s*F skip
      dbgF(nm("S", d), S, n, C);
      up(d - 1, S, s.up, F(d));  // Eq.9
      dbgF(nm("F", d), F(d), o.N[d], C);
      return F(d);
    }
    const int j = d - D;
    const DDeep& dp = m->deep[j - 1];
    if (j == 1) kmap(D);
    // Eq.4: G_D = Downsampling(X_{d-1}): embed on depth d-1 then K2S2 steps down to D
    int8_t* ga = buf<int8_t>(c, "t_ga", rows(d - 1) * C);
    int8_t* gb = buf<int8_t>(c, "t_gb", rows(d - 1) * C);
    // C = 32: the tcgen05 kernel (down_tc.cu), whose first step gathers the embedding
    // E[X_{d-1}] of the children directly (the embedded level is materialised only for a
    // debug dump or when no down step follows); PCC_DOWN=simt selects the dp4a kernel
    static const bool simt = [] {
      const char* e = getenv("PCC_DOWN");
      return e && std::string(e) == "simt";
    }();
    const bool fuse = C == 32 && !simt && j > 1 && !c->debug;
    if (!fuse) {
      embed(c, dp.E, X(d - 1), o.N[d - 1], C, ga);
      dbgF(nm("G", d, d - 1), ga, o.N[d - 1], C);
    }
    for (int s = 0; s < j - 1; ++s) {
      const int k = d - 1 - s;  // depth k -> k-1
      if (C == 32 && !simt)
        down_tc(c, fuse && s == 0 ? dp.E : ga, X(k - 1), cs() + o.nb[k - 1], o.N[k - 1], dp.down[s], gb,
                fuse && s == 0 ? X(d - 1) : nullptr);
      else
        down(c, ga, X(k - 1), cs() + o.nb[k - 1], o.N[k - 1], C, dp.down[s], gb);
      std::swap(ga, gb);
      dbgF(nm("G", d, k - 1), ga, o.N[k - 1], C);
    }
    const uint32_t nD = o.N[D];
    int8_t* hx = buf<int8_t>(c, "t_hx", rows(D) * C);
    int8_t* Hk = buf<int8_t>(c, "t_H", rows(D) * C);
    if (m->flags & MF_XFP_OFF) {
      // "Baseline + GRED" (Table 4): H = ResBlock(G_D), no cross-scale concat
      conv3(c, ga, nullptr, C, nD, nbr(D), dp.a, 0, nullptr, nullptr, 0, nullptr, hx);
      dbgF(nm("hx", d), hx, nD, C);
      conv3(c, hx, nullptr, C, nD, nbr(D), dp.b, 1, ga, nullptr, dp.k_s, nullptr, Hk);
    } else {
      // Eq.10: H = ResBlock(Concat(F_D, G_D)), virtual concat, 1x1 projection skip
      conv3(c, F(D), ga, C, nD, nbr(D), dp.a, 0, nullptr, nullptr, 0, nullptr, hx);
      dbgF(nm("hx", d), hx, nD, C);
      conv3(c, hx, nullptr, C, nD, nbr(D), dp.b, 2, F(D), ga, 0, dp.P, Hk);
    }
    dbgF(nm("H", d), Hk, nD, C);
    // Eq.11: up/prune chain D -> d (H at k = D only, reading Q3)
    size_t mx = 0;
    for (int k = D + 1; k <= d; ++k) mx = std::max(mx, rows(k));
    int8_t* ua = buf<int8_t>(c, "t_ua", mx * C);
    int8_t* ub = buf<int8_t>(c, "t_ub", mx * C);
    const int8_t* cur = Hk;
    for (int k = D; k < d; ++k) {
      int8_t* dst = (k - D) % 2 == 0 ? ua : ub;
      up(k, cur, dp.up[k - D], dst);
      dbgF(nm("Fp", d, k + 1), dst, o.N[k + 1], C);
      cur = dst;
    }
    return cur;
  }

  const DHead& head_of(int d) { return d <= D ? m->shallow[d - m->R].head : m->deep[d - D - 1].head; }
};

// ============================================================================
// encoder output packing (reading O11)
// ============================================================================
__global__ void k_pack_sizes(const PackItem* __restrict__ items, int n, const EncSeg* __restrict__ segs,
                             const uint32_t* __restrict__ seg_W, const uint32_t* __restrict__ raw_sz,
                             uint32_t* __restrict__ sizes) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const PackItem it = items[i];
  if (it.kind == 0) {
    sizes[i] = it.bytes + ((raw_sz[it.frame] + 3u) & ~3u);  // header + level sizes + padded raw region
  } else {
    const uint32_t ns = segs[it.seg].n;
    uint32_t k = (ns + 511u) / 512u;
    k = k < 1u ? 1u : (k > 32u ? 32u : k);
    sizes[i] = 4u + 4u * k + 4u * ((seg_W[it.seg] + 1u) / 2u);
  }
}

__global__ void k_pack_write(const PackItem* __restrict__ items, int n, const uint32_t* __restrict__ item_off,
                             const uint32_t* __restrict__ sizes, const EncSeg* __restrict__ segs,
                             const uint32_t* __restrict__ seg_W, const uint32_t* __restrict__ seg_state,
                             const uint16_t* __restrict__ words, int L, int R, int n_deep, uint32_t flags,
                             uint64_t hash, const uint32_t* __restrict__ foff, int B, const uint64_t* __restrict__ nb,
                             const uint8_t* __restrict__ code, const uint32_t* __restrict__ raw_sz,
                             const uint8_t* __restrict__ raw_region, uint32_t raw_cap, uint8_t* __restrict__ out) {
  const int i = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const PackItem it = items[i];
  uint8_t* o = out + item_off[i];
  if (it.kind == 0) {
    const int f = int(it.frame);
    const uint32_t raw = raw_sz[f];
    const uint32_t NL = foff[L * (B + 1) + f + 1] - foff[L * (B + 1) + f];
    if (lane == 0) {
      o[0] = 'P'; o[1] = 'C'; o[2] = 'C'; o[3] = '1';
      o[4] = 2; o[5] = 0;  // container version 2: 4096-symbol segments (reading Q24')
      o[6] = uint8_t(L); o[7] = uint8_t(R); o[8] = uint8_t(n_deep); o[9] = uint8_t(flags);
      o[10] = uint8_t(raw); o[11] = uint8_t(raw >> 8);
      for (int b = 0; b < 4; ++b) o[12 + b] = uint8_t(NL >> (8 * b));
      for (int b = 0; b < 8; ++b) o[16 + b] = uint8_t(hash >> (8 * b));
    }
    // level payload sizes: sum of this frame's segment items per level
    for (int d = R + lane; d < L; d += 32) {
      uint32_t s = 0;
      for (uint32_t k = 1; k < it.nitems; ++k)
        if (items[i + k].level == uint32_t(d)) s += sizes[i + k];
      uint8_t* q = o + 24 + 4 * (d - R);
      q[0] = uint8_t(s); q[1] = uint8_t(s >> 8); q[2] = uint8_t(s >> 16); q[3] = uint8_t(s >> 24);
    }
    // raw prefix X_0..X_{R-1}: plain bytes (reading Q13) or the frequency-coded region
    // (MF_RAW_FREQ), zero-padded to 4 bytes
    uint8_t* rp = o + 24 + 4 * (L - R);
    uint32_t pos = 0;
    if (raw_region) {
      const uint8_t* src = raw_region + size_t(f) * raw_cap;
      for (uint32_t k = lane; k < raw; k += 32) rp[k] = src[k];
      pos = raw;
    } else {
      for (int d = 0; d < R; ++d) {
        const uint32_t a = foff[d * (B + 1) + f], cnt = foff[d * (B + 1) + f + 1] - a;
        for (uint32_t k = lane; k < cnt; k += 32) rp[pos + k] = code[nb[d] + a + k];
        pos += cnt;
      }
    }
    for (uint32_t k = pos + lane; k < ((pos + 3u) & ~3u); k += 32) rp[k] = 0;
  } else {
    const EncSeg sg = segs[it.seg];
    const uint32_t W = seg_W[it.seg];
    uint32_t K = (sg.n + 511u) / 512u;
    K = K < 1u ? 1u : (K > 32u ? 32u : K);
    uint32_t* o32 = reinterpret_cast<uint32_t*>(o);
    if (lane == 0) o32[0] = W;
    if (uint32_t(lane) < K) o32[1 + lane] = seg_state[size_t(it.seg) * 32 + lane];
    uint16_t* o16 = reinterpret_cast<uint16_t*>(o + 4 + 4 * K);
    const uint16_t* src = words + sg.node + sg.n - W;
    for (uint32_t k = lane; k < W; k += 32) o16[k] = src[k];
    if ((W & 1u) && lane == 0) o16[W] = 0;
  }
}

// ============================================================================
// decoder raw prefix (reading O4/Q13): per frame, counts then node arrays
// ============================================================================
__global__ void k_raw_count(const uint8_t* __restrict__ bs, const uint64_t* __restrict__ raw_off,
                            const uint32_t* __restrict__ raw_len, int B, int R, uint32_t* __restrict__ cnt,
                            uint32_t* __restrict__ err) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= B) return;
  const uint8_t* p = bs + raw_off[f];
  uint32_t nd = 1, pos = 0;
  bool bad = false;
  for (int d = 0; d < R; ++d) {
    cnt[f * (R + 1) + d] = nd;
    uint32_t nx = 0;
    if (pos + nd > raw_len[f]) { bad = true; break; }
    for (uint32_t k = 0; k < nd; ++k) {
      const uint8_t x = p[pos + k];
      if (x == 0) bad = true;
      nx += __popc(uint32_t(x));
    }
    pos += nd;
    nd = nx;
  }
  if (!bad && pos != raw_len[f]) bad = true;
  cnt[f * (R + 1) + R] = bad ? 0 : nd;
  if (bad) atomicOr(err, EF_CORRUPT);
}

// src: the bitstream with per-frame raw offsets (plain bytes), or, when stride != 0, the
// frequency decoder's symbols at src + f * stride
__global__ void k_raw_write(const uint8_t* __restrict__ bs, const uint64_t* __restrict__ raw_off, uint32_t stride, int B,
                            int R, const uint32_t* __restrict__ foff, const uint64_t* __restrict__ nb,
                            uint64_t* __restrict__ key, uint8_t* __restrict__ code, uint32_t* __restrict__ cs,
                            uint32_t* __restrict__ par) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= B) return;
  const uint8_t* p = stride ? bs + size_t(f) * stride : bs + raw_off[f];
  key[nb[0] + f] = uint64_t(f);
  uint32_t pos = 0;
  for (int d = 0; d < R; ++d) {
    const uint32_t a = foff[d * (B + 1) + f], n = foff[d * (B + 1) + f + 1] - a;
    const uint32_t a1 = foff[(d + 1) * (B + 1) + f];
    uint32_t j = 0;
    for (uint32_t k = 0; k < n; ++k) {
      const uint8_t x = p[pos + k];
      code[nb[d] + a + k] = x;
      cs[nb[d] + a + k] = a1 + j;
      const uint64_t kk = key[nb[d] + a + k] << 3;
      for (int c = 0; c < 8; ++c)
        if ((x >> c) & 1) {
          key[nb[d + 1] + a1 + j] = kk | uint64_t(c);
          par[nb[d + 1] + a1 + j] = a + k;
          ++j;
        }
    }
    pos += n;
  }
}

__global__ void k_gather_hdr(const uint8_t* __restrict__ bs, const uint64_t* __restrict__ off,
                             const uint64_t* __restrict__ len, int B, uint8_t* __restrict__ hdr, int hdr_bytes) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  int f = t / hdr_bytes, k = t % hdr_bytes;
  if (f >= B) return;
  hdr[t] = uint64_t(k) < len[f] ? bs[off[f] + k] : 0;
}

template <class T>
T* upload(pcc_ctx c, const char* name, const std::vector<T>& v) {
  T* d = wsT<T>(c, name, v.size() + 1);
  if (!v.empty()) {
    T* h = static_cast<T*>(pinned(c, v.size() * sizeof(T)));
    std::memcpy(h, v.data(), v.size() * sizeof(T));
    PCC_CUDA(cudaMemcpyAsync(d, h, v.size() * sizeof(T), cudaMemcpyHostToDevice, c->stream));
    PCC_CUDA(cudaStreamSynchronize(c->stream));  // pinned staging is reused
  }
  return d;
}

// ============================================================================
// encode
// ============================================================================
void encode_batch(pcc_ctx c, pcc_model m, const int32_t* d_xyz, const size_t* offs, int B, int L, uint8_t* d_out,
                  size_t out_cap, size_t* out_offs) {
  if (!c || !m || !offs || B < 1 || (!d_xyz && offs[B] > 0) || !out_offs) throw Error{PCC_ERR_INVALID_ARG};
  check_depth(m, L);
  for (int f = 0; f < B; ++f) {
    if (offs[f + 1] < offs[f]) throw Error{PCC_ERR_INVALID_ARG};
    if (offs[f + 1] == offs[f]) throw Error{PCC_ERR_EMPTY};
  }
  if (offs[B] >= (1ull << 32)) throw Error{PCC_ERR_INVALID_ARG};
  PCC_CUDA(cudaSetDevice(c->device));
  c->dbg.clear();
  cudaStream_t s = c->stream;
  const int R = m->R, C = m->C;
  OctreeOut o;
  build_octree(c, d_xyz, offs, B, L, o);
  if (c->debug)
    for (int d = 0; d <= L; ++d) {
      dbg_copy(c, nm("key", d), static_cast<uint64_t*>(c->bufs.at("key").p) + o.nb[d], size_t(o.N[d]) * 8);
      if (d < L) dbg_copy(c, nm("code", d), static_cast<uint8_t*>(c->bufs.at("code").p) + o.nb[d], o.N[d]);
    }
  const size_t tot = o.nb[L + 1];
  uint32_t* cf = buf<uint32_t>(c, "cf", tot);
  Net net{c, m, L, R, L - 1 - m->n_deep, C, o};
  for (int d = R; d < L; ++d) {
    const int8_t* Fd = net.level(d);
    int8_t* a_dbg = c->debug ? buf<int8_t>(c, "t_adbg", size_t(o.N[d]) * m->H) : nullptr;
    head_any(c, Fd, o.N[d], C, m->H, net.head_of(d), m->lut, 0, net.X(d), cf + o.nb[d], nullptr, a_dbg);
    if (c->debug) {
      dbg_copy(c, nm("a", d), a_dbg, size_t(o.N[d]) * m->H);
      dbg_copy(c, nm("cf", d), cf + o.nb[d], size_t(o.N[d]) * 4);
    }
  }
  // rANS segments (frame-major, level, chunk) and output items
  std::vector<EncSeg> segs;
  std::vector<PackItem> items;
  for (int f = 0; f < B; ++f) {
    const size_t i0 = items.size();
    items.push_back(PackItem{0, uint32_t(f), 0, 0, uint32_t(24 + 4 * (L - R)), 0});
    for (int d = R; d < L; ++d) {
      const uint32_t a = o.foff[size_t(d) * (B + 1) + f], nfd = o.foff[size_t(d) * (B + 1) + f + 1] - a;
      for (uint32_t s0 = 0; s0 < nfd; s0 += SEG_SYMS) {
        segs.push_back(EncSeg{uint32_t(o.nb[d] + a + s0), std::min<uint32_t>(SEG_SYMS, nfd - s0)});
        items.push_back(PackItem{1, uint32_t(f), uint32_t(segs.size() - 1), uint32_t(d), 0, 0});
      }
    }
    items[i0].nitems = uint32_t(items.size() - i0);
  }
  const int nseg = int(segs.size()), nit = int(items.size());
  EncSeg* d_segs = upload(c, "segs", segs);
  PackItem* d_items = upload(c, "items", items);
  uint16_t* words = buf<uint16_t>(c, "words", tot);
  uint32_t* seg_W = buf<uint32_t>(c, "seg_W", nseg);
  uint32_t* seg_state = buf<uint32_t>(c, "seg_state", size_t(nseg) * 32);
  size_t nsym = 0;
  for (const EncSeg& sg : segs) nsym += sg.n;
  rans_encode(c, d_segs, nseg, cf, words, seg_W, seg_state, nsym);
  uint32_t* sizes = buf<uint32_t>(c, "item_sizes", nit + 1);
  uint32_t* ioff = buf<uint32_t>(c, "item_off", nit + 1);
  uint64_t* d_nb = upload(c, "nb", o.nb);
  uint32_t* d_foff = static_cast<uint32_t*>(c->bufs.at("foff").p);
  // raw prefix region per frame (plain bytes, or the P:601 frequency coder)
  const bool rawfreq = (m->flags & MF_RAW_FREQ) != 0;
  const uint32_t raw_cap = (8u + 2u * raw_max_symbols(R) + 4u + 3u) & ~3u;
  uint8_t* raw_region = rawfreq ? buf<uint8_t>(c, "raw_region", size_t(B) * raw_cap) : nullptr;
  uint32_t* raw_sz = buf<uint32_t>(c, "raw_sz", B);
  raw_encode(c, rawfreq, static_cast<uint8_t*>(c->bufs.at("code").p), d_nb, d_foff, B, R, raw_region, raw_cap, raw_sz);
  {
    Prof p(c, "pack", 0);
    k_pack_sizes<<<cdiv(nit, 128), 128, 0, s>>>(d_items, nit, d_segs, seg_W, raw_sz, sizes);
    launched(c);
  }
  scan_u32(c, sizes, ioff, size_t(nit));
  uint32_t* h_off = static_cast<uint32_t*>(pinned(c, (nit + 1) * sizeof(uint32_t)));
  PCC_CUDA(cudaMemcpyAsync(h_off, ioff, (nit + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  PCC_CUDA(cudaStreamSynchronize(s));
  const size_t total = h_off[nit];
  {
    size_t k = 0;
    for (int f = 0; f < B; ++f) {
      out_offs[f] = h_off[k];
      k += items[k].nitems;
    }
    out_offs[B] = total;
  }
  if (total > out_cap || !d_out) throw Error{PCC_ERR_CAPACITY};
  Prof pw(c, "pack", total);
  k_pack_write<<<cdiv(size_t(nit) * 32, 128), 128, 0, s>>>(d_items, nit, ioff, sizes, d_segs, seg_W, seg_state, words, L,
                                                          R, m->n_deep, m->flags, m->hash, d_foff, B, d_nb,
                                                          static_cast<uint8_t*>(c->bufs.at("code").p), raw_sz,
                                                          raw_region, raw_cap, d_out);
  launched(c);
  PCC_CUDA(cudaStreamSynchronize(s));
  PCC_CUDA(cudaGetLastError());
}

// ============================================================================
// decode
// ============================================================================
struct Hdr {
  int L, R, nd;
  uint32_t raw, NL;
  uint64_t hash;
  std::vector<uint32_t> lb;
};

void decode_batch(pcc_ctx c, pcc_model m, const uint8_t* d_bs, const size_t* bs_offs, int B, int32_t* d_xyz,
                  size_t cap_points, size_t* out_offs) {
  if (!c || !m || !d_bs || !bs_offs || B < 1 || !out_offs) throw Error{PCC_ERR_INVALID_ARG};
  PCC_CUDA(cudaSetDevice(c->device));
  c->dbg.clear();
  cudaStream_t s = c->stream;
  for (int f = 0; f < B; ++f) {
    if (bs_offs[f + 1] < bs_offs[f] || (bs_offs[f] & 3)) throw Error{PCC_ERR_INVALID_ARG};
  }
  // 1. headers -> host (bookkeeping only)
  const int HB = 24 + 4 * MAX_DEPTH;
  std::vector<uint64_t> off(B), len(B);
  for (int f = 0; f < B; ++f) {
    off[f] = bs_offs[f];
    len[f] = bs_offs[f + 1] - bs_offs[f];
  }
  uint64_t* d_off = upload(c, "d_hoff", off);
  uint64_t* d_len = upload(c, "d_hlen", len);
  uint8_t* d_hdr = buf<uint8_t>(c, "d_hdr", size_t(B) * HB);
  {
    Prof p(c, "container", 0);
    k_gather_hdr<<<cdiv(size_t(B) * HB, 256), 256, 0, s>>>(d_bs, d_off, d_len, B, d_hdr, HB);
    launched(c);
  }
  std::vector<uint8_t> hh(size_t(B) * HB);
  PCC_CUDA(cudaMemcpyAsync(hh.data(), d_hdr, hh.size(), cudaMemcpyDeviceToHost, s));
  PCC_CUDA(cudaStreamSynchronize(s));
  std::vector<Hdr> hd(B);
  for (int f = 0; f < B; ++f) {
    const uint8_t* h = hh.data() + size_t(f) * HB;
    if (len[f] < 24) throw Error{PCC_ERR_TRUNCATED};
    if (std::memcmp(h, "PCC1", 4) != 0) throw Error{PCC_ERR_BAD_MAGIC};
    if ((h[4] | h[5] << 8) != 2) throw Error{PCC_ERR_VERSION};
    Hdr& x = hd[f];
    x.L = h[6]; x.R = h[7]; x.nd = h[8];
    x.raw = uint32_t(h[10]) | uint32_t(h[11]) << 8;
    std::memcpy(&x.NL, h + 12, 4);
    std::memcpy(&x.hash, h + 16, 8);
    if (x.hash != m->hash || x.R != m->R || x.nd != m->n_deep || h[9] != m->flags) throw Error{PCC_ERR_MODEL_MISMATCH};
    check_depth(m, x.L);
    if (x.L != hd[0].L) throw Error{PCC_ERR_INVALID_ARG};  // a batch shares one bit depth
    if (len[f] < size_t(24 + 4 * (x.L - x.R))) throw Error{PCC_ERR_TRUNCATED};
    x.lb.resize(x.L - x.R);
    uint64_t total = 24 + 4 * (x.L - x.R) + ((x.raw + 3) & ~3u);
    for (int d = 0; d < x.L - x.R; ++d) {
      std::memcpy(&x.lb[d], h + 24 + 4 * d, 4);
      total += x.lb[d];
    }
    if (total > len[f]) throw Error{PCC_ERR_TRUNCATED};
    if (x.NL == 0) throw Error{PCC_ERR_CORRUPT};
  }
  const int L = hd[0].L, R = m->R, C = m->C;
  uint64_t NLtot = 0;
  for (int f = 0; f < B; ++f) NLtot += hd[f].NL;
  {
    uint64_t acc = 0;
    for (int f = 0; f < B; ++f) {
      out_offs[f] = acc;
      acc += hd[f].NL;
    }
    out_offs[B] = acc;
  }
  if (NLtot > cap_points || !d_xyz) throw Error{PCC_ERR_CAPACITY};
  if (NLtot >= (1ull << 31)) throw Error{PCC_ERR_INVALID_ARG};
  // node array capacity: sum_d min(B 8^d, N_L)
  uint64_t cap = 0;
  for (int d = 0; d <= L; ++d) {
    uint64_t b = uint64_t(B);
    for (int k = 0; k < d && b < NLtot; ++k) b *= 8;
    cap += std::min<uint64_t>(b, NLtot);
  }
  buf<uint64_t>(c, "key", cap);
  buf<uint8_t>(c, "code", cap + 8);
  buf<uint32_t>(c, "cs", cap + 1);
  buf<uint32_t>(c, "par", cap);
  uint32_t* d_foff = buf<uint32_t>(c, "foff", size_t(L + 2) * (B + 1));
  uint32_t* err = buf<uint32_t>(c, "err", 4);
  PCC_CUDA(cudaMemsetAsync(err, 0, 16, s));
  // 2. raw prefix
  std::vector<uint64_t> raw_off(B);
  std::vector<uint32_t> raw_len(B);
  for (int f = 0; f < B; ++f) {
    raw_off[f] = bs_offs[f] + 24 + 4 * (L - R);
    raw_len[f] = hd[f].raw;
  }
  uint64_t* d_raw_off = upload(c, "d_raw_off", raw_off);
  uint32_t* d_raw_len = upload(c, "d_raw_len", raw_len);
  uint32_t* d_cnt = buf<uint32_t>(c, "raw_cnt", size_t(B) * (R + 1));
  const bool rawfreq = (m->flags & MF_RAW_FREQ) != 0;
  uint8_t* raw_sym = nullptr;
  if (rawfreq) {  // P:601 frequency-coded raw prefix: decode the symbols first
    std::vector<uint32_t> nl(B);
    for (int f = 0; f < B; ++f) nl[f] = hd[f].NL;
    uint32_t* d_nl = upload(c, "d_raw_nl", nl);
    raw_sym = buf<uint8_t>(c, "raw_sym", size_t(B) * raw_max_symbols(R));
    raw_decode(c, d_bs, d_raw_off, d_raw_len, B, R, d_nl, raw_sym, d_cnt, err);
  } else {
    Prof p(c, "container", 0);
    k_raw_count<<<cdiv(B, 128), 128, 0, s>>>(d_bs, d_raw_off, d_raw_len, B, R, d_cnt, err);
    launched(c);
  }
  std::vector<uint32_t> hc(size_t(B) * (R + 1));
  uint32_t herr = 0;
  PCC_CUDA(cudaMemcpyAsync(hc.data(), d_cnt, hc.size() * 4, cudaMemcpyDeviceToHost, s));
  PCC_CUDA(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, s));
  PCC_CUDA(cudaStreamSynchronize(s));
  if (herr) throw Error{PCC_ERR_CORRUPT};
  OctreeOut o;
  o.N.assign(R + 1, 0);
  o.nb.assign(R + 2, 0);
  o.foff.assign(size_t(R + 1) * (B + 1), 0);
  for (int d = 0; d <= R; ++d) {
    uint32_t acc = 0;
    for (int f = 0; f < B; ++f) {
      o.foff[size_t(d) * (B + 1) + f] = acc;
      const uint32_t nfd = hc[size_t(f) * (R + 1) + d];
      if (nfd > hd[f].NL) throw Error{PCC_ERR_CORRUPT};
      acc += nfd;
    }
    o.foff[size_t(d) * (B + 1) + B] = acc;
    o.N[d] = acc;
    o.nb[d + 1] = o.nb[d] + acc;
  }
  if (o.nb[R + 1] > cap) throw Error{PCC_ERR_CORRUPT};
  PCC_CUDA(cudaMemcpyAsync(d_foff, upload(c, "foff_stage", o.foff), o.foff.size() * 4, cudaMemcpyDeviceToDevice, s));
  uint64_t* d_nb = upload(c, "nb", o.nb);
  {
    Prof praw(c, "container", 0);
    k_raw_write<<<cdiv(B, 128), 128, 0, s>>>(rawfreq ? raw_sym : d_bs, d_raw_off, rawfreq ? raw_max_symbols(R) : 0u, B,
                                             R, d_foff, d_nb,
                                             static_cast<uint64_t*>(c->bufs.at("key").p),
                                             static_cast<uint8_t*>(c->bufs.at("code").p),
                                             static_cast<uint32_t*>(c->bufs.at("cs").p),
                                             static_cast<uint32_t*>(c->bufs.at("par").p));
    launched(c);
  }
  // 3. level-serial neural decoding (Eq.2)
  Net net{c, m, L, R, L - 1 - m->n_deep, C, o};
  // pinned staging for every level's segment list (upper bound: per level, one segment
  // per frame plus one per SEG_SYMS nodes)
  const size_t seg_ring_cap = size_t(L - R) * ((size_t(B) + NLtot / SEG_SYMS + 2) * sizeof(DecSeg) + 256);
  uint8_t* seg_ring = static_cast<uint8_t*>(pinned_ring(c, seg_ring_cap));
  size_t seg_ring_used = 0;
  std::vector<uint64_t> lvl_base(B);
  for (int f = 0; f < B; ++f) lvl_base[f] = bs_offs[f] + 24 + 4 * (L - R) + ((hd[f].raw + 3) & ~3u);
  for (int d = R; d < L; ++d) {
    const int8_t* Fd = net.level(d);
    const uint32_t nd = o.N[d];
    uint16_t* cdf = buf<uint16_t>(c, "cdf", size_t(nd) * DROW_U16);
    int8_t* a_dbg = c->debug ? buf<int8_t>(c, "t_adbg", size_t(nd) * m->H) : nullptr;
    head_any(c, Fd, nd, C, m->H, net.head_of(d), m->lut, 1, nullptr, nullptr, cdf, a_dbg);
    if (c->debug) {
      dbg_copy(c, nm("a", d), a_dbg, size_t(nd) * m->H);
      dbg_copy(c, nm("cdf", d), cdf, size_t(nd) * DROW_BYTES);
    }
    std::vector<DecSeg> segs;
    for (int f = 0; f < B; ++f) {
      const uint32_t a = o.foff[size_t(d) * (B + 1) + f], nfd = o.foff[size_t(d) * (B + 1) + f + 1] - a;
      uint32_t ch = 0;
      for (uint32_t s0 = 0; s0 < nfd; s0 += SEG_SYMS, ++ch) {
        const uint32_t cnt = std::min<uint32_t>(SEG_SYMS, nfd - s0);
        segs.push_back(DecSeg{lvl_base[f], ch, a + s0, cnt, hd[f].lb[d - R], s0 + cnt == nfd ? 1u : 0u});
      }
      lvl_base[f] += hd[f].lb[d - R];
    }
    // the segment list goes up through its own slice of a per-call pinned ring, so no
    // level waits for its upload (the level's single sync is the expansion readback)
    const size_t seg_bytes = segs.size() * sizeof(DecSeg);
    if (seg_ring_used + seg_bytes > seg_ring_cap) throw Error{PCC_ERR_INVALID_ARG};
    std::memcpy(seg_ring + seg_ring_used, segs.data(), seg_bytes);
    DecSeg* d_segs = wsT<DecSeg>(c, "dsegs", segs.size() + 1);
    PCC_CUDA(cudaMemcpyAsync(d_segs, seg_ring + seg_ring_used, seg_bytes, cudaMemcpyHostToDevice, s));
    seg_ring_used += (seg_bytes + 255) & ~size_t(255);
    int kmax = 1;
    size_t nstates = 0;
    for (const DecSeg& sg : segs) {
      kmax = std::max(kmax, lanes_for(sg.n));
      nstates += size_t(lanes_for(sg.n));
    }
    rans_decode(c, d_segs, int(segs.size()), d_bs, cdf, m->H, net.head_of(d), m->lut,
                static_cast<uint8_t*>(c->bufs.at("code").p) + o.nb[d], err, kmax, nd, nstates);
    if (c->debug) dbg_copy(c, nm("code", d), static_cast<uint8_t*>(c->bufs.at("code").p) + o.nb[d], nd);
    expand_level(c, d, B, o, uint32_t(std::min<uint64_t>(NLtot, 0xffffffffu)), err);
  }
  for (int f = 0; f < B; ++f)
    if (o.foff[size_t(L) * (B + 1) + f + 1] - o.foff[size_t(L) * (B + 1) + f] != hd[f].NL) throw Error{PCC_ERR_CORRUPT};
  keys_to_xyz(c, static_cast<uint64_t*>(c->bufs.at("key").p) + o.nb[L], o.N[L], L, d_xyz);
  if (c->debug)
    for (int d = 0; d <= L; ++d)
      dbg_copy(c, nm("key", d), static_cast<uint64_t*>(c->bufs.at("key").p) + o.nb[d], size_t(o.N[d]) * 8);
  PCC_CUDA(cudaStreamSynchronize(s));
  PCC_CUDA(cudaGetLastError());
}

// Frames coded together carry their index above the 3L Morton bits of a u64 key.  At
// most 2^fb - 1 frames share a launch, so no key (frame 2^fb - 1's corner voxel would be
// all ones) equals the kernel-map hash's EMPTY sentinel ~0.
int frames_per_chunk(int frames, int fb_max) {
  if (fb_max >= 30) return frames;
  return std::max(1, std::min(frames, (1 << fb_max) - 1));
}

template <class F>
pcc_status guard(pcc_ctx c, F&& f) {
  try {
    if (c) c->launches = 0;
    f();
    return PCC_OK;
  } catch (const Error& e) {
    if (c && c->stream) cudaStreamSynchronize(c->stream);
    cudaGetLastError();
    return e.st;
  } catch (...) {
    return PCC_ERR_CUDA;
  }
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

pcc_status pcc_model_load(const void* bytes, size_t len, int device, pcc_model* out) {
  if (!bytes || !out) return PCC_ERR_INVALID_ARG;
  return guard(nullptr, [&] {
    check_device(device);
    *out = load_model(static_cast<const uint8_t*>(bytes), len, device);
  });
}

pcc_status pcc_model_random_file(const pcc_model_config* cfg, void* buf, size_t cap, size_t* len) {
  if (!cfg || !len) return PCC_ERR_INVALID_ARG;
  return guard(nullptr, [&] {
    if (!model_config_valid(*cfg)) throw Error{PCC_ERR_INVALID_ARG};
    const std::vector<uint8_t> f = random_model_file(*cfg);
    *len = f.size();
    if (!buf || cap < f.size()) throw Error{PCC_ERR_CAPACITY};
    std::memcpy(buf, f.data(), f.size());
  });
}

pcc_status pcc_model_create_random(const pcc_model_config* cfg, int device, pcc_model* out) {
  if (!cfg || !out) return PCC_ERR_INVALID_ARG;
  return guard(nullptr, [&] {
    if (!model_config_valid(*cfg)) throw Error{PCC_ERR_INVALID_ARG};
    check_device(device);
    const std::vector<uint8_t> f = random_model_file(*cfg);
    *out = load_model(f.data(), f.size(), device);
  });
}

pcc_status pcc_model_save(pcc_model m, void* buf, size_t cap, size_t* len) {
  if (!m || !len) return PCC_ERR_INVALID_ARG;
  *len = m->file.size();
  if (!buf || cap < m->file.size()) return PCC_ERR_CAPACITY;
  std::memcpy(buf, m->file.data(), m->file.size());
  return PCC_OK;
}

pcc_status pcc_model_flags(pcc_model m, uint32_t* out) {
  if (!m || !out) return PCC_ERR_INVALID_ARG;
  *out = m->flags;
  return PCC_OK;
}

pcc_status pcc_model_hash(pcc_model m, uint64_t* out) {
  if (!m || !out) return PCC_ERR_INVALID_ARG;
  *out = m->hash;
  return PCC_OK;
}

pcc_status pcc_model_info(pcc_model m, int* C, int* H, int* R, int* n_deep, int* min_depth, int* max_depth) {
  if (!m) return PCC_ERR_INVALID_ARG;
  if (C) *C = m->C;
  if (H) *H = m->H;
  if (R) *R = m->R;
  if (n_deep) *n_deep = m->n_deep;
  if (min_depth) *min_depth = m->min_depth;
  if (max_depth) *max_depth = m->max_depth;
  return PCC_OK;
}

void pcc_model_destroy(pcc_model m) {
  if (!m) return;
  if (m->dmem) cudaFree(m->dmem);
  delete m;
}

pcc_status pcc_ctx_create(int device, void* stream, pcc_ctx* out) {
  if (!out) return PCC_ERR_INVALID_ARG;
  return guard(nullptr, [&] {
    check_device(device);
    PCC_CUDA(cudaSetDevice(device));
    auto* c = new pcc_ctx_s();
    c->device = device;
    c->stream = static_cast<cudaStream_t>(stream);
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    *out = c;
  });
}

void pcc_ctx_destroy(pcc_ctx c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& kv : c->bufs)
    if (kv.second.p) cudaFree(kv.second.p);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->pinned1) cudaFreeHost(c->pinned1);
  delete c;
}

size_t pcc_encode_bound(size_t n, int bit_depth) {
  if (bit_depth < 1) return 0;
  const size_t levels = size_t(bit_depth);
  const size_t segs = (n + SEG_SYMS - 1) / SEG_SYMS + 1;
  return 24 + 4 * levels + 600 + levels * (2 * n + 4 + segs * (4 + 4 * 32 + 4));
}

pcc_status pcc_build_octree(pcc_ctx c, const int32_t* d_xyz, size_t n, int bit_depth, uint8_t* d_codes,
                            size_t codes_cap, uint32_t* h_level_counts) {
  if (!c || !d_xyz || !h_level_counts) return PCC_ERR_INVALID_ARG;
  return guard(c, [&] {
    if (bit_depth < 1 || bit_depth > MAX_DEPTH) throw Error{PCC_ERR_UNSUPPORTED_DEPTH};
    if (n == 0) throw Error{PCC_ERR_EMPTY};
    PCC_CUDA(cudaSetDevice(c->device));
    size_t offs[2] = {0, n};
    OctreeOut o;
    build_octree(c, d_xyz, offs, 1, bit_depth, o);
    for (int d = 0; d <= bit_depth; ++d) h_level_counts[d] = o.N[d];
    if (d_codes) {
      const size_t need = o.nb[bit_depth];
      if (need > codes_cap) throw Error{PCC_ERR_CAPACITY};
      PCC_CUDA(cudaMemcpyAsync(d_codes, c->bufs.at("code").p, need, cudaMemcpyDeviceToDevice, c->stream));
    }
    if (c->debug)
      for (int d = 0; d <= bit_depth; ++d) {
        dbg_copy(c, nm("key", d), static_cast<uint64_t*>(c->bufs.at("key").p) + o.nb[d], size_t(o.N[d]) * 8);
        if (d < bit_depth) dbg_copy(c, nm("code", d), static_cast<uint8_t*>(c->bufs.at("code").p) + o.nb[d], o.N[d]);
        if (d >= 1) dbg_copy(c, nm("par", d), static_cast<uint32_t*>(c->bufs.at("par").p) + o.nb[d], size_t(o.N[d]) * 4);
      }
    PCC_CUDA(cudaStreamSynchronize(c->stream));
  });
}

// HRCS statistic: octree of the batch, then per depth one hash build + one
// 26-probe counting pass (kmap.cu k_hrcs).  Batches split like encode (frame bits).
pcc_status pcc_hrcs_stats(pcc_ctx c, const int32_t* d_xyz, const size_t* offs, int frames, int bit_depth,
                          uint64_t* h_nodes, uint64_t* h_nbr) {
  if (!c || !offs || frames < 1 || !h_nodes || !h_nbr) return PCC_ERR_INVALID_ARG;
  return guard(c, [&] {
    if (bit_depth < 1 || bit_depth > MAX_DEPTH) throw Error{PCC_ERR_UNSUPPORTED_DEPTH};
    for (int f = 0; f < frames; ++f) {
      if (offs[f + 1] < offs[f]) throw Error{PCC_ERR_INVALID_ARG};
      if (offs[f + 1] == offs[f]) throw Error{PCC_ERR_EMPTY};
    }
    if (!d_xyz) throw Error{PCC_ERR_INVALID_ARG};
    PCC_CUDA(cudaSetDevice(c->device));
    const int L = bit_depth, fb_max = 64 - 3 * L;
    const int chunk = frames_per_chunk(frames, fb_max);
    std::vector<uint64_t> res(size_t(chunk) * (L + 1));
    std::vector<size_t> sub;
    for (int f0 = 0; f0 < frames; f0 += chunk) {
      const int B = std::min(chunk, frames - f0);
      sub.assign(offs + f0, offs + f0 + B + 1);
      for (auto& v : sub) v -= offs[f0];
      OctreeOut o;
      build_octree(c, d_xyz + 3 * offs[f0], sub.data(), B, L, o);
      unsigned long long* d_sum = buf<unsigned long long>(c, "hrcs_sum", size_t(B) * (L + 1));
      for (int d = 0; d <= L; ++d)
        hrcs_counts(c, static_cast<uint64_t*>(c->bufs.at("key").p) + o.nb[d], o.N[d], d, B, d_sum + size_t(d) * B);
      PCC_CUDA(cudaMemcpyAsync(res.data(), d_sum, size_t(B) * (L + 1) * 8, cudaMemcpyDeviceToHost, c->stream));
      PCC_CUDA(cudaStreamSynchronize(c->stream));
      for (int f = 0; f < B; ++f)
        for (int d = 0; d <= L; ++d) {
          h_nodes[size_t(f0 + f) * (L + 1) + d] = o.foff[size_t(d) * (B + 1) + f + 1] - o.foff[size_t(d) * (B + 1) + f];
          h_nbr[size_t(f0 + f) * (L + 1) + d] = res[size_t(d) * B + f];
        }
    }
  });
}

// Splits a batch so that the frame id fits above the 3L Morton bits of a u64 key.
pcc_status pcc_encode_batch(pcc_ctx c, pcc_model m, const int32_t* d_xyz, const size_t* offs, int frames, int bit_depth,
                            uint8_t* d_out, size_t out_cap, size_t* out_offs) {
  return guard(c, [&] {
    if (!c || !m || !offs || !out_offs || frames < 1) throw Error{PCC_ERR_INVALID_ARG};
    check_depth(m, bit_depth);
    const int fb_max = 64 - 3 * bit_depth;
    const int chunk = frames_per_chunk(frames, fb_max);
    size_t base_out = 0;
    std::vector<size_t> sub_offs, sub_out;
    for (int f0 = 0; f0 < frames; f0 += chunk) {
      const int nb = std::min(chunk, frames - f0);
      sub_offs.assign(offs + f0, offs + f0 + nb + 1);
      for (auto& v : sub_offs) v -= offs[f0];
      sub_out.assign(nb + 1, 0);
      const size_t rem = out_cap > base_out ? out_cap - base_out : 0;
      try {
        encode_batch(c, m, d_xyz + 3 * offs[f0], sub_offs.data(), nb, bit_depth, d_out ? d_out + base_out : nullptr, rem,
                     sub_out.data());
      } catch (const Error& e) {
        if (e.st == PCC_ERR_CAPACITY) {
          for (int k = 0; k <= nb; ++k) out_offs[f0 + k] = base_out + sub_out[k];
        }
        throw;
      }
      for (int k = 0; k < nb; ++k) out_offs[f0 + k] = base_out + sub_out[k];
      base_out += sub_out[nb];
      out_offs[f0 + nb] = base_out;
    }
  });
}

pcc_status pcc_encode(pcc_ctx c, pcc_model m, const int32_t* d_xyz, size_t n, int bit_depth, uint8_t* d_out,
                      size_t out_cap, size_t* out_len) {
  if (!out_len) return PCC_ERR_INVALID_ARG;
  size_t offs[2] = {0, n}, oo[2] = {0, 0};
  pcc_status st = pcc_encode_batch(c, m, d_xyz, offs, 1, bit_depth, d_out, out_cap, oo);
  *out_len = oo[1];
  return st;
}

pcc_status pcc_decode_batch(pcc_ctx c, pcc_model m, const uint8_t* d_bs, const size_t* bs_offs, int frames,
                            int32_t* d_xyz_out, size_t cap_points, size_t* out_offs) {
  return guard(c, [&] { decode_batch(c, m, d_bs, bs_offs, frames, d_xyz_out, cap_points, out_offs); });
}

pcc_status pcc_decode(pcc_ctx c, pcc_model m, const uint8_t* d_bs, size_t len, int32_t* d_xyz_out, size_t cap_points,
                      size_t* n_out, int* bit_depth_out) {
  if (!n_out) return PCC_ERR_INVALID_ARG;
  size_t offs[2] = {0, len}, oo[2] = {0, 0};
  pcc_status st = pcc_decode_batch(c, m, d_bs, offs, 1, d_xyz_out, cap_points, oo);
  *n_out = oo[1];
  if (bit_depth_out && c && (st == PCC_OK || st == PCC_ERR_CAPACITY)) {
    uint8_t h[8] = {0};
    if (len >= 8 && cudaMemcpy(h, d_bs, 8, cudaMemcpyDeviceToHost) == cudaSuccess) *bit_depth_out = h[6];
  }
  return st;
}

pcc_status pcc_encode_batch_host(pcc_ctx c, pcc_model m, const int32_t* h_xyz, const size_t* offs, int frames,
                                 int bit_depth, uint8_t* h_out, size_t out_cap, size_t* out_offs) {
  if (!c || !h_xyz || !offs || frames < 1) return PCC_ERR_INVALID_ARG;
  int32_t* d_in = nullptr;
  uint8_t* d_out = nullptr;
  pcc_status st = guard(c, [&] {
    d_in = wsT<int32_t>(c, "e2e_in", offs[frames] * 3);
    PCC_CUDA(cudaMemcpyAsync(d_in, h_xyz, offs[frames] * 12, cudaMemcpyHostToDevice, c->stream));
    d_out = wsT<uint8_t>(c, "e2e_out", out_cap);
  });
  if (st != PCC_OK) return st;
  const uint64_t l0 = 0;
  st = pcc_encode_batch(c, m, d_in, offs, frames, bit_depth, d_out, out_cap, out_offs);
  (void)l0;
  if (st != PCC_OK) return st;
  return guard(c, [&] {
    PCC_CUDA(cudaMemcpyAsync(h_out, d_out, out_offs[frames], cudaMemcpyDeviceToHost, c->stream));
    PCC_CUDA(cudaStreamSynchronize(c->stream));
  });
}

pcc_status pcc_decode_batch_host(pcc_ctx c, pcc_model m, const uint8_t* h_bs, const size_t* bs_offs, int frames,
                                 int32_t* h_xyz_out, size_t cap_points, size_t* out_offs) {
  if (!c || !h_bs || !bs_offs || frames < 1) return PCC_ERR_INVALID_ARG;
  uint8_t* d_bs = nullptr;
  int32_t* d_xyz = nullptr;
  pcc_status st = guard(c, [&] {
    d_bs = wsT<uint8_t>(c, "e2e_bs", bs_offs[frames]);
    PCC_CUDA(cudaMemcpyAsync(d_bs, h_bs, bs_offs[frames], cudaMemcpyHostToDevice, c->stream));
    d_xyz = wsT<int32_t>(c, "e2e_xyz", cap_points * 3);
  });
  if (st != PCC_OK) return st;
  st = pcc_decode_batch(c, m, d_bs, bs_offs, frames, d_xyz, cap_points, out_offs);
  if (st != PCC_OK) return st;
  return guard(c, [&] {
    PCC_CUDA(cudaMemcpyAsync(h_xyz_out, d_xyz, out_offs[frames] * 12, cudaMemcpyDeviceToHost, c->stream));
    PCC_CUDA(cudaStreamSynchronize(c->stream));
  });
}

pcc_status pcc_debug_tensor(pcc_ctx c, const char* name, void* h_dst, size_t cap, size_t* len) {
  if (!c || !name || !len) return PCC_ERR_INVALID_ARG;
  auto it = c->dbg.find(name);
  if (it == c->dbg.end()) return PCC_ERR_INVALID_ARG;
  *len = it->second.size();
  if (h_dst) std::memcpy(h_dst, it->second.data(), std::min(cap, it->second.size()));
  return PCC_OK;
}

pcc_status pcc_debug_gemm_i8(pcc_ctx c, const int8_t* h_a, const int8_t* h_b, int n_cols, int32_t* h_d) {
  if (!c || !h_a || !h_b || !h_d) return PCC_ERR_INVALID_ARG;
  return guard(c, [&] {
    PCC_CUDA(cudaSetDevice(c->device));
    int8_t* dA = wsT<int8_t>(c, "gt_a", 128 * 32);
    int8_t* dB = wsT<int8_t>(c, "gt_b", size_t(n_cols) * 32);
    int32_t* dD = wsT<int32_t>(c, "gt_d", size_t(128) * n_cols);
    PCC_CUDA(cudaMemcpyAsync(dA, h_a, 128 * 32, cudaMemcpyHostToDevice, c->stream));
    PCC_CUDA(cudaMemcpyAsync(dB, h_b, size_t(n_cols) * 32, cudaMemcpyHostToDevice, c->stream));
    gemm_i8_test(c, dA, dB, n_cols, dD);
    PCC_CUDA(cudaMemcpyAsync(h_d, dD, size_t(128) * n_cols * 4, cudaMemcpyDeviceToHost, c->stream));
    PCC_CUDA(cudaStreamSynchronize(c->stream));
    PCC_CUDA(cudaGetLastError());
  });
}

pcc_status pcc_ctx_set_debug(pcc_ctx c, int on) {
  if (!c) return PCC_ERR_INVALID_ARG;
  c->debug = on != 0;
  if (!c->debug) c->dbg.clear();
  return PCC_OK;
}

uint64_t pcc_ctx_launch_count(pcc_ctx c) { return c ? c->launches : 0; }

pcc_status pcc_ctx_set_profile(pcc_ctx c, int on) {
  if (!c) return PCC_ERR_INVALID_ARG;
  return guard(nullptr, [&] {
    prof_collect(c);
    c->prof = on != 0;
    c->tot.clear();
  });
}

pcc_status pcc_ctx_profile_get(pcc_ctx c, const char* category, double* ms, uint64_t* launches, uint64_t* bytes) {
  if (!c) return PCC_ERR_INVALID_ARG;
  return guard(nullptr, [&] {
    prof_collect(c);
    if (!category) {  // total over categories
      double t = 0;
      uint64_t l = 0, b = 0;
      for (auto& kv : c->tot) {
        t += kv.second.ms;
        l += kv.second.launches;
        b += kv.second.bytes;
      }
      if (ms) *ms = t;
      if (launches) *launches = l;
      if (bytes) *bytes = b;
      return;
    }
    auto it = c->tot.find(category);
    if (ms) *ms = it == c->tot.end() ? 0.0 : it->second.ms;
    if (launches) *launches = it == c->tot.end() ? 0 : it->second.launches;
    if (bytes) *bytes = it == c->tot.end() ? 0 : it->second.bytes;
  });
}

const char* pcc_ctx_profile_categories(pcc_ctx c) {
  static thread_local std::string s;
  s.clear();
  if (!c) return "";
  try {
    prof_collect(c);
  } catch (...) {
  }
  for (auto& kv : c->tot) s += kv.first + "\n";
  return s.c_str();
}

const char* pcc_status_string(pcc_status s) {
  switch (s) {
    case PCC_OK: return "OK";
    case PCC_ERR_INVALID_ARG: return "INVALID_ARG";
    case PCC_ERR_EMPTY: return "EMPTY";
    case PCC_ERR_RANGE: return "RANGE";
    case PCC_ERR_UNSUPPORTED_DEPTH: return "UNSUPPORTED_DEPTH";
    case PCC_ERR_CAPACITY: return "CAPACITY";
    case PCC_ERR_BAD_MAGIC: return "BAD_MAGIC";
    case PCC_ERR_VERSION: return "VERSION";
    case PCC_ERR_MODEL_MISMATCH: return "MODEL_MISMATCH";
    case PCC_ERR_TRUNCATED: return "TRUNCATED";
    case PCC_ERR_CORRUPT: return "CORRUPT";
    case PCC_ERR_CUDA: return "CUDA";
    case PCC_ERR_OOM: return "OOM";
  }
  return "?";
}

}  // extern "C"
