// =============================================================================
// pcc_oracle.cpp — CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
//
// This file is the plain, slow, single-threaded reference for the integer-only
// octree coder of "Towards Practical Lossless Neural Compression for LiDAR
// Point Clouds" (arxiv 2603.25260; /root/reference/PAPER.md = "P:<line>").
// It follows the method step by step in the paper's order, with the readings of
// DESIGN.md §"Readings" (mirroring SURVEY.md §8(c) O1–O12 and Q1–Q31) wherever
// the paper is silent.  It shares NO code with the CUDA path
// (paper_2603_25260_b200/csrc): no headers, helpers, tables or constants.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load it.  The product path never calls it.
//
// Conventions: depth d in [0, L]; a depth-d node has d-bit coordinates; X_d is
// the child-occupancy byte of depth-d nodes (the paper's X^{d+1}, reading Q1).
// No floating point is used anywhere in this file.
//
// Parity status per function (DESIGN.md §"Oracle pins"):
//   morton/build_octree/expand ............ pinned (SPEC examples, inverse, brute force)
//   kernel_map ............................ pinned (brute force)
//   conv3_acc / down_acc .................. pinned (dense 3D conv, numpy, tests)
//   rq / prq .............................. pinned (exact rationals)
//   up_prune .............................. pinned (code 255 / code 1 / expand keys)
//   cdf_quantize .......................... pinned (closed forms, softmax bound)
//   rans segment .......................... pinned (round trip, entropy bound)
//   encode / decode ....................... pinned (round trip, zero-model and
//                                           bias-only-head closed-form lengths)
//   layer WIRING of ResBlock/XFP (O7) ..... parity unpinned vs the paper beyond the
//                                           special cases (the structure figure,
//                                           P:604-608, is missing)
// =============================================================================
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

// ---- status codes (values are the C-ABI's, include/pcc.h) --------------------
enum Status {
  OK = 0, INVALID_ARG = 1, EMPTY = 2, RANGE = 3, UNSUPPORTED_DEPTH = 4, CAPACITY = 5,
  BAD_MAGIC = 6, VERSION = 7, MODEL_MISMATCH = 8, TRUNCATED = 9, CORRUPT = 10,
};

struct Fail {
  int status;
};

constexpr int NCODE = 255;  // occupancy classes, "255 classes"

// ---- Morton keys ("sort the input coordinates in Morton order") ------------
// Reading O1/Q25: bit triple b of the key is (x_b, y_b, z_b) with x most significant,
// so the child index of a node is c = 4*bx + 2*by + bz = key & 7.
uint64_t morton(uint32_t x, uint32_t y, uint32_t z, int bits) {
  uint64_t k = 0;
  for (int b = 0; b < bits; ++b) {
    uint64_t t = (uint64_t(((x >> b) & 1u) << 2) | uint64_t(((y >> b) & 1u) << 1) | uint64_t((z >> b) & 1u));
    k |= t << (3 * b);
  }
  return k;
}

void unmorton(uint64_t k, int bits, uint32_t& x, uint32_t& y, uint32_t& z) {
  x = y = z = 0;
  for (int b = 0; b < bits; ++b) {
    uint64_t t = (k >> (3 * b)) & 7u;
    x |= uint32_t((t >> 2) & 1u) << b;
    y |= uint32_t((t >> 1) & 1u) << b;
    z |= uint32_t(t & 1u) << b;
  }
}

// ---- Octree ("Coordinate Sampling", "Occupancy Code Generation") -----
struct Tree {
  int L = 0;
  std::vector<std::vector<uint64_t>> key;  // key[d], d = 0..L, sorted ascending
  std::vector<std::vector<uint8_t>> code;  // code[d], d = 0..L-1
};

// O1: Morton keys, sort, dedup.  O2: "repeatedly divide them by 2, apply floor
// rounding, and remove consecutive duplicates"; X_d[i] has bit c set iff
// child c of node i is occupied (the K2S2 all-ones conv of P:658, bit-equivalent).
Tree build_tree(const int32_t* xyz, size_t n, int L) {
  if (n == 0) throw Fail{EMPTY};
  Tree t;
  t.L = L;
  t.key.resize(L + 1);
  t.code.resize(L);
  std::vector<uint64_t> leaf(n);
  const int64_t lim = int64_t(1) << L;
  for (size_t i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) {
      int64_t v = xyz[3 * i + a];
      if (v < 0 || v >= lim) throw Fail{RANGE};
    }
    leaf[i] = morton(uint32_t(xyz[3 * i]), uint32_t(xyz[3 * i + 1]), uint32_t(xyz[3 * i + 2]), L);
  }
  std::sort(leaf.begin(), leaf.end());
  leaf.erase(std::unique(leaf.begin(), leaf.end()), leaf.end());
  t.key[L] = leaf;
  for (int d = L - 1; d >= 0; --d) {
    const std::vector<uint64_t>& ch = t.key[d + 1];
    std::vector<uint64_t>& par = t.key[d];
    std::vector<uint8_t>& cd = t.code[d];
    for (size_t j = 0; j < ch.size(); ++j) {
      uint64_t p = ch[j] >> 3;  // floor(coord / 2) on every axis
      if (par.empty() || par.back() != p) {
        par.push_back(p);
        cd.push_back(0);
      }
      cd.back() |= uint8_t(1u << (ch[j] & 7u));
    }
  }
  return t;
}

// Decoder expansion ("adding a pre-defined offset matrix ... masking"):
// children of each parent in order, child c for each set bit c ascending.
std::vector<uint64_t> expand(const std::vector<uint64_t>& keys, const std::vector<uint8_t>& codes) {
  std::vector<uint64_t> out;
  for (size_t i = 0; i < keys.size(); ++i)
    for (int c = 0; c < 8; ++c)
      if ((codes[i] >> c) & 1u) out.push_back((keys[i] << 3) | uint64_t(c));
  return out;
}

// ---- Kernel map ("indexed linear transforms"; reading D04) ------------------
// nbr[i][delta] = row of the node at coord(i) + delta at the same depth, or -1.
// delta index = (dx+1)*9 + (dy+1)*3 + (dz+1).  Plain binary search in the sorted keys.
std::vector<int32_t> kernel_map(const std::vector<uint64_t>& keys, int depth) {
  const size_t n = keys.size();
  std::vector<int32_t> nbr(n * 27, -1);
  const int64_t lim = int64_t(1) << depth;
  for (size_t i = 0; i < n; ++i) {
    uint32_t x, y, z;
    unmorton(keys[i], depth, x, y, z);
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          int64_t X = int64_t(x) + dx, Y = int64_t(y) + dy, Z = int64_t(z) + dz;
          if (X < 0 || Y < 0 || Z < 0 || X >= lim || Y >= lim || Z >= lim) continue;
          uint64_t k = morton(uint32_t(X), uint32_t(Y), uint32_t(Z), depth);
          auto it = std::lower_bound(keys.begin(), keys.end(), k);
          if (it != keys.end() && *it == k)
            nbr[i * 27 + (dx + 1) * 9 + (dy + 1) * 3 + (dz + 1)] = int32_t(it - keys.begin());
        }
  }
  return nbr;
}

// ---- Integer primitives (Eq.13-14; readings O5, Q15-Q18) -------------
// Eq.13: y_int32 = sum (q_x - z_x) q_w + b with z_x = z_w = 0 (reading Q16).
// The oracle accumulates in int64 and asserts the result fits int32 (reading O6).
int32_t to_i32(int64_t acc) {
  if (acc < INT32_MIN || acc > INT32_MAX) throw std::runtime_error("int32 accumulator overflow");
  return int32_t(acc);
}

// Eq.14: q_y = clip(round(y * m / 2^r)), round half up via +2^(r-1) and an arithmetic
// shift (reading Q15), clip to [-128, 127] (Q17).  C++20: >> on negatives is arithmetic.
int8_t rq(int32_t acc, int32_t m, int32_t r) {
  int64_t v = int64_t(acc) * int64_t(m);
  if (r > 0) v = (v + (int64_t(1) << (r - 1))) >> r;
  if (v < -128) v = -128;
  if (v > 127) v = 127;
  return int8_t(v);
}

// PReLU fused into the requant with a single rounding (reading Q18/Q19).
int8_t prq(int32_t acc, int32_t m_pos, int32_t m_neg, int32_t r) {
  return rq(acc, acc >= 0 ? m_pos : m_neg, r);
}

struct RQ {
  int32_t m_pos = 1, m_neg = 1, r = 0;
};

// Sparse conv K3S1 as indexed linear transforms: for every offset delta,
// acc[i] += W_delta * f[nbr(i, delta)]; absent neighbours contribute 0.
// W layout [27][cout][cin]; f layout [n][cin].
std::vector<int64_t> conv3_acc(const std::vector<int32_t>& nbr, size_t n, const int8_t* f, int cin,
                               const int8_t* W, int cout) {
  std::vector<int64_t> acc(n * cout, 0);
  for (size_t i = 0; i < n; ++i)
    for (int dl = 0; dl < 27; ++dl) {
      int32_t j = nbr[i * 27 + dl];
      if (j < 0) continue;
      for (int o = 0; o < cout; ++o) {
        int64_t s = 0;
        for (int c = 0; c < cin; ++c) s += int64_t(f[size_t(j) * cin + c]) * int64_t(W[(size_t(dl) * cout + o) * cin + c]);
        acc[i * cout + o] += s;
      }
    }
  return acc;
}

// ---- Model file (DESIGN.md §"Model file") -----------------------------------------
struct Head {
  std::vector<int8_t> W1, W2;  // [H][C], [255][H]
  std::vector<int32_t> b1, b2;
  RQ rq1, rql;
};
struct Up {
  std::vector<int8_t> W;  // [8C][C+255]: linear over Concat(S, q_one * onehot(X))
  std::vector<int32_t> b;
  RQ rq;
  int32_t q_one = 0;
};
struct Shallow {
  std::vector<int8_t> Wa, Wb;
  std::vector<int32_t> ba, bb;
  RQ rqa, rqb;
  int32_t k_s = 0;
  Up up;
  Head head;
};
struct Down {
  std::vector<int8_t> W;  // [8][C][C]
  std::vector<int32_t> b;
  RQ rq;
};
struct Deep {
  std::vector<int8_t> E;  // [255][C]
  std::vector<Down> downs;
  // XFP on: Wa [27][C][2C], Wb [27][C][C], P [C][2C].  XFP off (MF_XFP_OFF): Wa, Wb
  // [27][C][C] and the identity skip k_s (the shallow ResBlock form on G_D alone).
  std::vector<int8_t> Wa, Wb, P;
  std::vector<int32_t> ba, bb;
  int32_t k_s = 0;
  RQ rqa, rqb;
  std::vector<Up> ups;
  Head head;
};
// Model flags (model-file header word at byte 44; copied into the bitstream's flags byte):
//   MF_XFP_OFF  the "Baseline + GRED" ablation of Table 4: deep levels
//               drop the cross-scale concat, H = ResBlock(G_D).
//   MF_RAW_FREQ the raw prefix X_0..X_{R-1} is coded "based on their symbol frequencies"
//               (reading Q13', NEXT-4) instead of stored as plain bytes.
// n_deep = 0 is the GRED-off "Baseline" of Table 4: every coded level is a
// shallow level (Eq.8-9), directly exposed to HRCS.
constexpr uint32_t MF_XFP_OFF = 1, MF_RAW_FREQ = 2, MF_ALL = 3;

struct Model {
  int C = 0, H = 0, R = 0, n_deep = 0, min_depth = 0, max_depth = 0;
  uint32_t flags = 0;
  uint64_t seed = 0, hash = 0;
  std::vector<uint32_t> lut;
  std::vector<int8_t> E0;
  std::map<int, Shallow> shallow;
  std::vector<Deep> deep;  // j = 1..n_deep at index j-1
};

struct Reader {
  const uint8_t* p;
  size_t n, pos = 0;
  void need(size_t k) {
    if (pos + k > n) throw Fail{INVALID_ARG};
  }
  uint32_t u32() {
    need(4);
    uint32_t v = uint32_t(p[pos]) | uint32_t(p[pos + 1]) << 8 | uint32_t(p[pos + 2]) << 16 | uint32_t(p[pos + 3]) << 24;
    pos += 4;
    return v;
  }
  int32_t i32() { return int32_t(u32()); }
  uint64_t u64() {
    uint64_t lo = u32();
    uint64_t hi = u32();
    return lo | (hi << 32);
  }
  std::vector<int8_t> i8v(size_t k) {
    need(k);
    std::vector<int8_t> v(k);
    std::memcpy(v.data(), p + pos, k);
    pos += k;
    return v;
  }
  std::vector<int32_t> i32v(size_t k) {
    std::vector<int32_t> v(k);
    for (auto& x : v) x = i32();
    return v;
  }
  RQ rq() {
    RQ t;
    t.m_pos = i32();
    t.m_neg = i32();
    t.r = i32();
    return t;
  }
};

uint64_t fnv1a64(const uint8_t* p, size_t n) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001B3ull;
  }
  return h;
}

Model parse_model(const uint8_t* bytes, size_t len) {
  if (len < 64 + 8 || std::memcmp(bytes, "PCCM", 4) != 0) throw Fail{INVALID_ARG};
  Model m;
  m.hash = 0;
  for (int i = 0; i < 8; ++i) m.hash |= uint64_t(bytes[len - 8 + i]) << (8 * i);
  if (fnv1a64(bytes, len - 8) != m.hash) throw Fail{MODEL_MISMATCH};
  Reader r{bytes, len - 8};
  r.pos = 4;
  if (r.u32() != 1) throw Fail{VERSION};
  m.C = int(r.u32());
  m.H = int(r.u32());
  m.R = int(r.u32());
  m.n_deep = int(r.u32());
  m.min_depth = int(r.u32());
  m.max_depth = int(r.u32());
  m.seed = r.u64();
  uint32_t lut_len = r.u32();
  if (lut_len != 1024) throw Fail{INVALID_ARG};
  m.flags = r.u32();
  if (m.flags & ~MF_ALL) throw Fail{INVALID_ARG};
  // R <= 6 keeps the raw prefix (at most sum_{d<R} 8^d = 37449 nodes) inside the
  // container's u16 raw_bytes field; n_deep in 0..4 (0 = GRED off).
  if (m.R < 1 || m.R > 6 || m.n_deep < 0 || m.n_deep > 4 || m.C < 1 || m.H < 1 || m.C > 64 || m.H > 64 ||
      m.min_depth < m.R + 1 + m.n_deep || m.max_depth < m.min_depth || m.max_depth > 21)
    throw Fail{INVALID_ARG};
  r.pos = 64;
  m.lut.resize(1024);
  for (auto& x : m.lut) x = r.u32();
  // The exp table (reading Q20) must be a valid softmax table: LUT[0] in (65281, 2^24]
  // and non-increasing.  Then S = sum e lies in (65281, 255 * 2^24]: normalisation never
  // divides by zero, every cumulative bound stays below 2^16 + 255, and a row's sum fits
  // 32 bits (the width P:351 fixes for the accumulation).
  if (m.lut[0] <= 65281u || m.lut[0] > (1u << 24)) throw Fail{INVALID_ARG};
  for (size_t j = 1; j < m.lut.size(); ++j)
    if (m.lut[j] > m.lut[j - 1]) throw Fail{INVALID_ARG};
  const size_t C = size_t(m.C), H = size_t(m.H);
  auto head = [&]() {
    Head h;
    h.W1 = r.i8v(H * C);
    h.b1 = r.i32v(H);
    h.rq1 = r.rq();
    h.W2 = r.i8v(NCODE * H);
    h.b2 = r.i32v(NCODE);
    h.rql = r.rq();
    return h;
  };
  auto up = [&]() {
    Up u;
    u.W = r.i8v(8 * C * (C + NCODE));
    u.b = r.i32v(8 * C);
    u.rq = r.rq();
    u.q_one = r.i32();
    return u;
  };
  m.E0 = r.i8v(NCODE * C);
  for (int d = m.R; d < m.max_depth - m.n_deep; ++d) {
    Shallow s;
    s.Wa = r.i8v(27 * C * C);
    s.ba = r.i32v(C);
    s.rqa = r.rq();
    s.Wb = r.i8v(27 * C * C);
    s.bb = r.i32v(C);
    s.k_s = r.i32();
    s.rqb = r.rq();
    s.up = up();
    s.head = head();
    m.shallow[d] = std::move(s);
  }
  for (int j = 1; j <= m.n_deep; ++j) {
    Deep dp;
    dp.E = r.i8v(NCODE * C);
    for (int s = 0; s < j - 1; ++s) {
      Down dn;
      dn.W = r.i8v(8 * C * C);
      dn.b = r.i32v(C);
      dn.rq = r.rq();
      dp.downs.push_back(std::move(dn));
    }
    if (m.flags & MF_XFP_OFF) {  // ResBlock(G_D), same layout as a shallow ResBlock
      dp.Wa = r.i8v(27 * C * C);
      dp.ba = r.i32v(C);
      dp.rqa = r.rq();
      dp.Wb = r.i8v(27 * C * C);
      dp.bb = r.i32v(C);
      dp.k_s = r.i32();
      dp.rqb = r.rq();
    } else {
      dp.Wa = r.i8v(27 * C * 2 * C);
      dp.ba = r.i32v(C);
      dp.rqa = r.rq();
      dp.Wb = r.i8v(27 * C * C);
      dp.P = r.i8v(C * 2 * C);
      dp.bb = r.i32v(C);
      dp.rqb = r.rq();
    }
    for (int s = 0; s < j; ++s) dp.ups.push_back(up());
    dp.head = head();
    m.deep.push_back(std::move(dp));
  }
  if (r.pos != r.n) throw Fail{INVALID_ARG};
  return m;
}

// ---- Dumps of every intermediate tensor (for per-tensor GPU parity) -------------
struct Dump {
  std::map<std::string, std::vector<uint8_t>> t;
  std::string names;
  template <class T>
  void put(const std::string& name, const std::vector<T>& v) {
    std::vector<uint8_t> b(v.size() * sizeof(T));
    if (!b.empty()) std::memcpy(b.data(), v.data(), b.size());
    t[name] = std::move(b);
  }
};

template <class T>
void dump(Dump* D, const std::string& name, const std::vector<T>& v) {
  if (D) D->put(name, v);
}

// ---- Network layers (Eq.4-11; readings O7, Q2-Q9, Q14) ------------------------
using Feat = std::vector<int8_t>;  // [n][C] row-major, rows in Morton order

// Eq.5/8 ResBlock, reading Q7: h = prq(conv3(F)+b_a); S = rq(conv3(h)+k_s*F+b_b).
Feat resblock_shallow(const Shallow& s, const Feat& F, const std::vector<int32_t>& nbr, size_t n, int C,
                      Dump* D, int d) {
  std::vector<int64_t> a = conv3_acc(nbr, n, F.data(), C, s.Wa.data(), C);
  Feat h(n * C);
  for (size_t i = 0; i < n; ++i)
    for (int o = 0; o < C; ++o)
      h[i * C + o] = prq(to_i32(a[i * C + o] + s.ba[o]), s.rqa.m_pos, s.rqa.m_neg, s.rqa.r);
  dump(D, "ha/" + std::to_string(d), h);
  std::vector<int64_t> b = conv3_acc(nbr, n, h.data(), C, s.Wb.data(), C);
  Feat S(n * C);
  for (size_t i = 0; i < n; ++i)
    for (int o = 0; o < C; ++o) {
      int64_t acc = b[i * C + o] + int64_t(s.k_s) * F[i * C + o] + s.bb[o];
      S[i * C + o] = prq(to_i32(acc), s.rqb.m_pos, s.rqb.m_neg, s.rqb.r);
    }
  dump(D, "S/" + std::to_string(d), S);
  return S;
}

// Eq.6/9/11: F^{k+1} = Pruning(Upsampling(Concat(S, X^k)), X^k).  Upsampling is "a
// linear transformation followed by a PReLU activation, performing an 8x channel
// expansion" over the concatenation [S | q_one*onehot(X)] (reading Q6);
// Pruning "discards features of unoccupied child nodes"; block c -> child c (Q8).
Feat up_prune(const Up& u, const Feat& S, const std::vector<uint8_t>& X, int C) {
  const size_t n = X.size();
  const int Cin = C + NCODE, Cout = 8 * C;
  Feat out;
  std::vector<int8_t> x(Cin);
  std::vector<int8_t> U(Cout);
  for (size_t p = 0; p < n; ++p) {
    for (int i = 0; i < C; ++i) x[i] = S[p * C + i];
    for (int v = 0; v < NCODE; ++v) x[C + v] = (X[p] == v + 1) ? int8_t(u.q_one) : int8_t(0);
    for (int o = 0; o < Cout; ++o) {
      int64_t acc = u.b[o];
      for (int i = 0; i < Cin; ++i) acc += int64_t(x[i]) * int64_t(u.W[size_t(o) * Cin + i]);
      U[o] = prq(to_i32(acc), u.rq.m_pos, u.rq.m_neg, u.rq.r);
    }
    for (int c = 0; c < 8; ++c)
      if ((X[p] >> c) & 1u)
        for (int i = 0; i < C; ++i) out.push_back(U[c * C + i]);
  }
  return out;
}

// Eq.4 Downsampling step (reading Q4): K2S2 sparse conv, one weight matrix per
// child index c: g_{j-1}[p] = prq(sum_{children ch of p} W_c * g_j[ch] + b).
// down_acc is the raw int64 accumulator (no bias, no requant); down_step (the codec)
// and the test entry point oracle_down_acc both call it.  W layout [8][C_out][C_in].
std::vector<int64_t> down_acc(const int8_t* W, const Feat& g, const std::vector<uint64_t>& child_keys,
                              const std::vector<uint64_t>& parent_keys, int C) {
  std::vector<int64_t> acc(parent_keys.size() * C, 0);
  for (size_t ch = 0; ch < child_keys.size(); ++ch) {
    uint64_t pk = child_keys[ch] >> 3;
    size_t p = size_t(std::lower_bound(parent_keys.begin(), parent_keys.end(), pk) - parent_keys.begin());
    if (p >= parent_keys.size() || parent_keys[p] != pk) throw Fail{INVALID_ARG};
    int c = int(child_keys[ch] & 7u);
    for (int o = 0; o < C; ++o) {
      int64_t s = 0;
      for (int i = 0; i < C; ++i) s += int64_t(g[ch * C + i]) * int64_t(W[(size_t(c) * C + o) * C + i]);
      acc[p * C + o] += s;
    }
  }
  return acc;
}

Feat down_step(const Down& dn, const Feat& g, const std::vector<uint64_t>& child_keys,
               const std::vector<uint64_t>& parent_keys, int C) {
  std::vector<int64_t> acc = down_acc(dn.W.data(), g, child_keys, parent_keys, C);
  Feat out(parent_keys.size() * C);
  for (size_t p = 0; p < parent_keys.size(); ++p)
    for (int o = 0; o < C; ++o) out[p * C + o] = prq(to_i32(acc[p * C + o] + dn.b[o]), dn.rq.m_pos, dn.rq.m_neg, dn.rq.r);
  return out;
}

// Eq.7 Predictor, reading Q9: a = prq(W1 F + b1) (C->H); z = W2 a + b2 (H->255).
std::vector<int32_t> head_logits(const Head& h, const Feat& F, size_t n, int C, int H, Dump* D, int d) {
  Feat a(n * H);
  for (size_t i = 0; i < n; ++i)
    for (int o = 0; o < H; ++o) {
      int64_t acc = h.b1[o];
      for (int c = 0; c < C; ++c) acc += int64_t(F[i * C + c]) * int64_t(h.W1[size_t(o) * C + c]);
      a[i * H + o] = prq(to_i32(acc), h.rq1.m_pos, h.rq1.m_neg, h.rq1.r);
    }
  dump(D, "a/" + std::to_string(d), a);
  std::vector<int32_t> z(n * NCODE);
  for (size_t i = 0; i < n; ++i)
    for (int o = 0; o < NCODE; ++o) {
      int64_t acc = h.b2[o];
      for (int c = 0; c < H; ++c) acc += int64_t(a[i * H + c]) * int64_t(h.W2[size_t(o) * H + c]);
      z[i * NCODE + o] = to_i32(acc);
    }
  dump(D, "z/" + std::to_string(d), z);
  return z;
}

// ---- Integer softmax -> Q16 pmf (Eq.15; readings O8, Q20-Q22) ---------
// l_i = clamp(round(z_i * m_l / 2^r_l), -2^24, 2^24)  (Q8 logits, 1/256 nat)
// delta_i = max_k l_k - l_i >= 0  ("numerically stable form", "non-positive domain")
// e_i = delta_i < 4096 ? LUT[delta_i >> 2] : 0   (LUT[j] = round(2^24 exp(-j/64)))
// S = sum e_i ("accumulation ... 32-bit integer arithmetic");
// normalisation (reading Q21, revised): cumulative floors of the prefix sums
//   E_i = sum_{j<i} e_j,  C_i = i + floor(E_i * 65281 / S)  (i = 0..255),
//   p_i = C_{i+1} - C_i,
// so C_0 = 0, C_255 = 255 + 65281 = 65536 exactly, and every p_i >= 1.
void cdf_quantize(const int32_t* z, const RQ& rql, const std::vector<uint32_t>& lut, uint32_t* p) {
  int64_t l[NCODE];
  for (int i = 0; i < NCODE; ++i) {
    int64_t v = int64_t(z[i]) * int64_t(rql.m_pos);
    if (rql.r > 0) v = (v + (int64_t(1) << (rql.r - 1))) >> rql.r;
    if (v < -(int64_t(1) << 24)) v = -(int64_t(1) << 24);
    if (v > (int64_t(1) << 24)) v = int64_t(1) << 24;
    l[i] = v;
  }
  int64_t mu = l[0];
  for (int i = 1; i < NCODE; ++i)
    if (l[i] > mu) mu = l[i];
  uint64_t e[NCODE], S = 0;
  for (int i = 0; i < NCODE; ++i) {
    int64_t dl = mu - l[i];
    e[i] = dl < 4096 ? uint64_t(lut[size_t(dl >> 2)]) : 0u;
    S += e[i];
  }
  uint64_t E = 0, C = 0;  // E_0 = 0, C_0 = 0
  for (int i = 0; i < NCODE; ++i) {
    E += e[i];
    const uint64_t Cn = uint64_t(i + 1) + (E * 65281u) / S;  // C_{i+1}
    p[i] = uint32_t(Cn - C);
    C = Cn;
  }
}

// ---- rANS (reading O9/O10/Q23/Q24) ---------------------------------------------
// 32-bit state, L = 2^16, 16-bit words, M = 2^16.  Symbol j of a segment of n goes to
// lane j mod K at step j / K with K = clamp(ceil(n/512), 1, 8) (segments of 4096 symbols:
// at most 512 sequential steps per lane, reading Q24').
int lanes_for(size_t n) {
  size_t k = (n + 511) / 512;
  if (k < 1) k = 1;
  if (k > 8) k = 8;
  return int(k);
}

void put_u32(std::vector<uint8_t>& o, uint32_t v) {
  for (int i = 0; i < 4; ++i) o.push_back(uint8_t(v >> (8 * i)));
}
void put_u16(std::vector<uint8_t>& o, uint32_t v) {
  o.push_back(uint8_t(v));
  o.push_back(uint8_t(v >> 8));
}

// Encode one segment: steps in reverse, lanes K-1..0, words pushed on a stack that is
// emitted reversed so the stream is in decoder consumption order.
void rans_encode_segment(const uint32_t* cum, const uint32_t* freq, size_t n, std::vector<uint8_t>& out,
                         int K_force = 0) {
  const int K = K_force > 0 ? K_force : lanes_for(n);
  std::vector<uint32_t> x(static_cast<size_t>(K), 1u << 16);
  std::vector<uint16_t> stack;
  const size_t steps = (n + size_t(K) - 1) / size_t(K);
  for (size_t s = steps; s-- > 0;)
    for (int k = K - 1; k >= 0; --k) {
      size_t j = s * size_t(K) + size_t(k);
      if (j >= n) continue;
      uint32_t f = freq[j], c = cum[j];
      if (uint64_t(x[k]) >= (uint64_t(f) << 16)) {
        stack.push_back(uint16_t(x[k] & 0xFFFFu));
        x[k] >>= 16;
      }
      x[k] = ((x[k] / f) << 16) + (x[k] % f) + c;
    }
  const uint32_t W = uint32_t(stack.size());
  put_u32(out, W);
  for (int k = 0; k < K; ++k) put_u32(out, x[k]);
  for (size_t i = stack.size(); i-- > 0;) put_u16(out, stack[i]);
  if (W & 1u) put_u16(out, 0);
}

uint32_t get_u32(const uint8_t* p) {
  return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}

// Decode one segment; pmf rows p[n][255] are known to the decoder (they depend only on
// previously decoded levels, Eq.2).  Returns bytes consumed.
size_t rans_decode_segment(const uint8_t* in, size_t avail, const uint32_t* p, size_t n, uint8_t* sym) {
  const int K = lanes_for(n);
  if (avail < 4 + 4 * size_t(K)) throw Fail{TRUNCATED};
  const uint32_t W = get_u32(in);
  const size_t bytes = 4 + 4 * size_t(K) + 4 * ((size_t(W) + 1) / 2);
  if (W > n || bytes > avail) throw Fail{W > n ? CORRUPT : TRUNCATED};
  std::vector<uint32_t> x(static_cast<size_t>(K));
  for (int k = 0; k < K; ++k) {
    x[k] = get_u32(in + 4 + 4 * k);
    if (x[k] < (1u << 16)) throw Fail{CORRUPT};
  }
  const uint8_t* w = in + 4 + 4 * K;
  size_t pos = 0;
  const size_t steps = (n + size_t(K) - 1) / size_t(K);
  for (size_t s = 0; s < steps; ++s)
    for (int k = 0; k < K; ++k) {
      size_t j = s * size_t(K) + size_t(k);
      if (j >= n) continue;
      const uint32_t* pj = p + j * NCODE;
      uint32_t slot = x[k] & 0xFFFFu, c = 0;
      int i = 0;
      while (c + pj[i] <= slot) {  // CDF^-1(slot): first i with cum_i <= slot < cum_i + p_i
        c += pj[i];
        ++i;
      }
      sym[j] = uint8_t(i + 1);
      x[k] = pj[i] * (x[k] >> 16) + slot - c;
      if (x[k] < (1u << 16)) {
        if (pos >= W) throw Fail{CORRUPT};
        x[k] = (x[k] << 16) | (uint32_t(w[2 * pos]) | uint32_t(w[2 * pos + 1]) << 8);
        ++pos;
      }
    }
  if (pos != W) throw Fail{CORRUPT};
  for (int k = 0; k < K; ++k)
    if (x[k] != (1u << 16)) throw Fail{CORRUPT};
  return bytes;
}

// ---- Raw prefix coder (NEXT-4; "For the geometry remaining at the maximum
// downsampling level, we directly encode the coordinates based on their symbol
// frequencies"; reading Q13') -------------------------------------------
// The symbols are the raw levels' occupancy bytes X_0..X_{R-1} in level order (the
// depth-R coordinates, losslessly).  Adaptive frequency model (SPEC S:583-584's
// AdaptiveFreqModel): counts n_v = 1 for all 255 symbols, total T; after each symbol
// n_v += RAW_INC, and when T exceeds RAW_LIMIT every count is halved rounding up.
// Symbol probabilities enter the O9 rANS coder as Q16 cumulative bounds by the same
// cumulative-floor normalisation as reading Q21: C_i = i + floor(K_i * 65281 / T),
// K_i = sum_{u<i} n_u (C_255 = 65536, every p >= 1).  One rANS lane (K = 1): the raw
// region is u32 W | u32 x | W u16 words | pad to 4 bytes.
constexpr uint32_t RAW_INC = 32, RAW_LIMIT = 1u << 15;

struct FreqModel {
  uint32_t n[NCODE];
  uint32_t T = NCODE;
  FreqModel() {
    for (auto& v : n) v = 1;
  }
  uint32_t bound(int i) const {  // C_i, i = 0..255
    uint64_t K = 0;
    for (int u = 0; u < i; ++u) K += n[u];
    return uint32_t(uint64_t(i) + K * 65281u / T);
  }
  void update(int i) {
    n[i] += RAW_INC;
    T += RAW_INC;
    if (T > RAW_LIMIT) {
      T = 0;
      for (auto& v : n) {
        v = (v + 1) / 2;
        T += v;
      }
    }
  }
};

std::vector<uint8_t> raw_encode(const std::vector<uint8_t>& sym) {
  FreqModel fm;
  std::vector<uint32_t> cum(sym.size()), freq(sym.size());
  for (size_t j = 0; j < sym.size(); ++j) {
    const int i = sym[j] - 1;
    cum[j] = fm.bound(i);
    freq[j] = fm.bound(i + 1) - cum[j];
    fm.update(i);
  }
  std::vector<uint8_t> out;
  rans_encode_segment(cum.data(), freq.data(), sym.size(), out, 1);
  return out;
}

// ---- Level-wise context model (Eq.2-11; readings O3, O7, Q1-Q3) -------------------
// State carried across coded levels: the shallow chain's current feature map and F_D.
struct Coder {
  const Model& m;
  int L, R, D;
  Dump* Dp;
  Feat F_prev;  // features on depth d-1 nodes (shallow chain)
  Feat F_D;     // shallow chain output at the dense depth D (Eq.10's F^k, k = t)
  Coder(const Model& mm, int L_, Dump* d) : m(mm), L(L_), R(mm.R), D(L_ - 1 - mm.n_deep), Dp(d) {}

  // pmf rows p[N_d][255] for coded level d given key[0..d], code[0..d-1].
  std::vector<uint32_t> level_pmf(const std::vector<std::vector<uint64_t>>& key,
                                  const std::vector<std::vector<uint8_t>>& code, int d) {
    const int C = m.C;
    const std::string sd = std::to_string(d);
    Feat Fd;
    if (d <= D) {
      // Shallow-level propagation (Eq.8-9), on depth d-1 nodes.
      const Shallow& s = m.shallow.at(d);
      const size_t n = key[d - 1].size();
      if (d == R) {  // reading Q14: F_{R-1} = E0[X_{R-1}]
        F_prev.assign(n * C, 0);
        for (size_t i = 0; i < n; ++i)
          for (int c = 0; c < C; ++c) F_prev[i * C + c] = m.E0[size_t(code[d - 1][i] - 1) * C + c];
        dump(Dp, "F/" + std::to_string(d - 1), F_prev);
      }
      std::vector<int32_t> nbr = kernel_map(key[d - 1], d - 1);
      dump(Dp, "nbr/" + std::to_string(d - 1), nbr);
      Feat S = resblock_shallow(s, F_prev, nbr, n, C, Dp, d);  // Eq.8
      Fd = up_prune(s.up, S, code[d - 1], C);                    // Eq.9
      dump(Dp, "F/" + sd, Fd);
      F_prev = Fd;
      if (d == D) F_D = Fd;
      return pmf_from_head(s.head, Fd, key[d].size(), d);
    }
    // Deep-level propagation with re-densification (Eq.4, Eq.10-11).
    const int j = d - D;
    const Deep& dp = m.deep[size_t(j - 1)];
    // Eq.4: G^k = Downsampling(X^{l-1}): embed X_{d-1} on depth d-1 nodes (reading Q5),
    // then one K2S2 conv + PReLU per depth step down to D (reading Q4).
    Feat g(key[d - 1].size() * C);
    for (size_t i = 0; i < key[d - 1].size(); ++i)
      for (int c = 0; c < C; ++c) g[i * C + c] = dp.E[size_t(code[d - 1][i] - 1) * C + c];
    dump(Dp, "G/" + sd + "/" + std::to_string(d - 1), g);
    for (int s = 0; s < j - 1; ++s) {
      int kd = d - 1 - s;  // g on depth kd -> depth kd-1
      g = down_step(dp.downs[size_t(s)], g, key[kd], key[kd - 1], C);
      dump(Dp, "G/" + sd + "/" + std::to_string(kd - 1), g);
    }
    const size_t n = key[D].size();
    if (m.flags & MF_XFP_OFF) {
      // "Baseline + GRED" (Table 4: "removing cross-scale feature propagation"):
      // no Concat with F^k; H^k = ResBlock(G^k) in the Eq.8 form (reading Q7).
      Shallow rb;
      rb.Wa = dp.Wa; rb.ba = dp.ba; rb.rqa = dp.rqa;
      rb.Wb = dp.Wb; rb.bb = dp.bb; rb.rqb = dp.rqb; rb.k_s = dp.k_s;
      std::vector<int32_t> nbr = kernel_map(key[D], D);
      Feat Hk = resblock_shallow(rb, g, nbr, n, C, nullptr, d);
      if (Dp) {  // the same dump names as the XFP block
        std::vector<int64_t> a = conv3_acc(nbr, n, g.data(), C, dp.Wa.data(), C);
        Feat h(n * C);
        for (size_t i = 0; i < n; ++i)
          for (int o = 0; o < C; ++o) h[i * C + o] = prq(to_i32(a[i * C + o] + dp.ba[o]), dp.rqa.m_pos, dp.rqa.m_neg, dp.rqa.r);
        dump(Dp, "hx/" + sd, h);
        dump(Dp, "H/" + sd, Hk);
      }
      Feat cur = Hk;
      for (int k = D; k < d; ++k) {
        cur = up_prune(dp.ups[size_t(k - D)], cur, code[k], C);
        dump(Dp, "Fp/" + sd + "/" + std::to_string(k + 1), cur);
      }
      return pmf_from_head(dp.head, cur, key[d].size(), d);
    }
    // Eq.10: H^k = ResBlock(Concat(F^k, G^k)), k = t = D (reading Q2); conv_a 2C->C,
    // conv_b C->C plus a 1x1 projection of the concat as the skip (reading Q7).
    Feat x(n * 2 * C);
    for (size_t i = 0; i < n; ++i)
      for (int c = 0; c < C; ++c) {
        x[i * 2 * C + c] = F_D[i * C + c];
        x[i * 2 * C + C + c] = g[i * C + c];
      }
    std::vector<int32_t> nbr = kernel_map(key[D], D);
    std::vector<int64_t> a = conv3_acc(nbr, n, x.data(), 2 * C, dp.Wa.data(), C);
    Feat h(n * C);
    for (size_t i = 0; i < n; ++i)
      for (int o = 0; o < C; ++o) h[i * C + o] = prq(to_i32(a[i * C + o] + dp.ba[o]), dp.rqa.m_pos, dp.rqa.m_neg, dp.rqa.r);
    dump(Dp, "hx/" + sd, h);
    std::vector<int64_t> b = conv3_acc(nbr, n, h.data(), C, dp.Wb.data(), C);
    Feat Hk(n * C);
    for (size_t i = 0; i < n; ++i)
      for (int o = 0; o < C; ++o) {
        int64_t acc = b[i * C + o] + dp.bb[o];
        for (int c = 0; c < 2 * C; ++c) acc += int64_t(x[i * 2 * C + c]) * int64_t(dp.P[size_t(o) * 2 * C + c]);
        Hk[i * C + o] = prq(to_i32(acc), dp.rqb.m_pos, dp.rqb.m_neg, dp.rqb.r);
      }
    dump(Dp, "H/" + sd, Hk);
    // Eq.11: F^{k+1} = Pruning(Upsampling(Concat(H^k or F^k, X^k)), X^k), k = t..l-1;
    // H only at k = t (reading Q3).
    Feat cur = Hk;
    for (int k = D; k < d; ++k) {
      cur = up_prune(dp.ups[size_t(k - D)], cur, code[k], C);
      dump(Dp, "Fp/" + sd + "/" + std::to_string(k + 1), cur);
    }
    return pmf_from_head(dp.head, cur, key[d].size(), d);
  }

  std::vector<uint32_t> pmf_from_head(const Head& h, const Feat& F, size_t n, int d) {
    std::vector<int32_t> z = head_logits(h, F, n, m.C, m.H, Dp, d);
    std::vector<uint32_t> p(n * NCODE);
    for (size_t i = 0; i < n; ++i) cdf_quantize(z.data() + i * NCODE, h.rql, m.lut, p.data() + i * NCODE);
    if (Dp) {
      std::vector<uint16_t> p16(p.begin(), p.end());
      Dp->put("p/" + std::to_string(d), p16);
    }
    return p;
  }
};

// ---- Container (reading O11) ------------------------------------------------------
// header (24 B): "PCC1" | u16 version=2 (reading Q24': 4096-symbol segments) | u8 L | u8 R | u8 n_deep | u8 flags=0 |
//                u16 raw_bytes | u32 N_L | u64 model_hash
// u32 level_bytes[L-R]; raw prefix X_0..X_{R-1} (raw_bytes, zero-padded to 4);
// level payloads d = R..L-1 (each a sequence of 4-byte-aligned rANS segments).
constexpr size_t SEG = 4096;

void check_depth(const Model& m, int L) {
  if (L < m.R + 1 + m.n_deep || L < m.min_depth || L > m.max_depth || L > 21) throw Fail{UNSUPPORTED_DEPTH};
}

std::vector<uint8_t> encode(const Model& m, const int32_t* xyz, size_t n, int L, Dump* Dp) {
  check_depth(m, L);
  Tree t = build_tree(xyz, n, L);
  if (Dp) {
    for (int d = 0; d <= L; ++d) Dp->put("key/" + std::to_string(d), t.key[d]);
    for (int d = 0; d < L; ++d) Dp->put("code/" + std::to_string(d), t.code[d]);
  }
  const int R = m.R;
  Coder cd(m, L, Dp);
  std::vector<std::vector<uint8_t>> payload(static_cast<size_t>(L - R));
  for (int d = R; d < L; ++d) {
    std::vector<uint32_t> p = cd.level_pmf(t.key, t.code, d);
    const size_t N = t.key[d].size();
    std::vector<uint32_t> cum(N), freq(N);
    std::vector<uint16_t> cf(2 * N);
    for (size_t i = 0; i < N; ++i) {
      int s = t.code[d][i] - 1;
      uint32_t c = 0;
      for (int k = 0; k < s; ++k) c += p[i * NCODE + k];
      cum[i] = c;
      freq[i] = p[i * NCODE + s];
      cf[2 * i] = uint16_t(c);
      cf[2 * i + 1] = uint16_t(freq[i]);
    }
    dump(Dp, "cf/" + std::to_string(d), cf);
    std::vector<uint8_t>& out = payload[size_t(d - R)];
    for (size_t s0 = 0; s0 < N; s0 += SEG) {
      size_t len = std::min(SEG, N - s0);
      rans_encode_segment(cum.data() + s0, freq.data() + s0, len, out);
    }
    dump(Dp, "seg/" + std::to_string(d), out);
  }
  std::vector<uint8_t> bs;
  bs.insert(bs.end(), {'P', 'C', 'C', '1'});
  put_u16(bs, 2);
  bs.push_back(uint8_t(L));
  bs.push_back(uint8_t(R));
  bs.push_back(uint8_t(m.n_deep));
  bs.push_back(uint8_t(m.flags));
  std::vector<uint8_t> rawsym;
  for (int d = 0; d < R; ++d) rawsym.insert(rawsym.end(), t.code[d].begin(), t.code[d].end());
  // reading Q13: plain bytes; MF_RAW_FREQ: the adaptive symbol-frequency coder
  std::vector<uint8_t> rawreg = (m.flags & MF_RAW_FREQ) ? raw_encode(rawsym) : rawsym;
  if (rawreg.size() > 0xFFFFu) throw Fail{CAPACITY};
  put_u16(bs, uint32_t(rawreg.size()));
  put_u32(bs, uint32_t(t.key[L].size()));
  put_u32(bs, uint32_t(m.hash));
  put_u32(bs, uint32_t(m.hash >> 32));
  for (auto& pl : payload) put_u32(bs, uint32_t(pl.size()));
  bs.insert(bs.end(), rawreg.begin(), rawreg.end());
  while (bs.size() % 4) bs.push_back(0);
  for (auto& pl : payload) bs.insert(bs.end(), pl.begin(), pl.end());
  return bs;
}

std::vector<uint64_t> decode(const Model& m, const uint8_t* bs, size_t len, int& L_out, Dump* Dp) {
  if (len < 24) throw Fail{TRUNCATED};
  if (std::memcmp(bs, "PCC1", 4) != 0) throw Fail{BAD_MAGIC};
  if ((uint32_t(bs[4]) | uint32_t(bs[5]) << 8) != 2u) throw Fail{VERSION};
  const int L = bs[6], R = bs[7], nd = bs[8];
  const size_t raw = uint32_t(bs[10]) | uint32_t(bs[11]) << 8;
  const uint32_t NL = get_u32(bs + 12);
  const uint64_t hash = uint64_t(get_u32(bs + 16)) | uint64_t(get_u32(bs + 20)) << 32;
  if (hash != m.hash || R != m.R || nd != m.n_deep || bs[9] != m.flags) throw Fail{MODEL_MISMATCH};
  check_depth(m, L);
  L_out = L;
  size_t pos = 24;
  if (len < pos + 4 * size_t(L - R)) throw Fail{TRUNCATED};
  std::vector<size_t> lb(static_cast<size_t>(L - R));
  for (int d = R; d < L; ++d) lb[size_t(d - R)] = get_u32(bs + pos + 4 * size_t(d - R));
  pos += 4 * size_t(L - R);
  std::vector<std::vector<uint64_t>> key(static_cast<size_t>(L + 1));
  std::vector<std::vector<uint8_t>> code(static_cast<size_t>(L));
  key[0] = {0};
  if (pos + raw > len) throw Fail{TRUNCATED};
  if (m.flags & MF_RAW_FREQ) {  // adaptive symbol-frequency raw prefix, one rANS lane
    const uint8_t* p = bs + pos;
    if (raw < 8) throw Fail{CORRUPT};
    const uint32_t W = get_u32(p);
    uint32_t x = get_u32(p + 4);
    if (raw != 8 + 4 * ((size_t(W) + 1) / 2) || x < (1u << 16)) throw Fail{CORRUPT};
    const uint8_t* w = p + 8;
    size_t wp = 0;
    FreqModel fm;
    for (int d = 0; d < R; ++d) {
      const size_t N = key[d].size();
      code[d].assign(N, 0);
      for (size_t k = 0; k < N; ++k) {
        const uint32_t slot = x & 0xFFFFu;
        int i = 0;
        while (fm.bound(i + 1) <= slot) ++i;  // CDF^-1(slot)
        const uint32_t c = fm.bound(i), f = fm.bound(i + 1) - c;
        x = f * (x >> 16) + slot - c;
        if (x < (1u << 16)) {
          if (wp >= W) throw Fail{CORRUPT};
          x = (x << 16) | (uint32_t(w[2 * wp]) | uint32_t(w[2 * wp + 1]) << 8);
          ++wp;
        }
        code[d][k] = uint8_t(i + 1);
        fm.update(i);
      }
      key[d + 1] = expand(key[d], code[d]);
      if (key[d + 1].size() > NL) throw Fail{CORRUPT};
    }
    if (wp != W || x != (1u << 16)) throw Fail{CORRUPT};
  } else {
    size_t rp = 0;
    for (int d = 0; d < R; ++d) {  // raw prefix (reading O4/Q13)
      const size_t N = key[d].size();
      if (rp + N > raw) throw Fail{CORRUPT};
      code[d].assign(bs + pos + rp, bs + pos + rp + N);
      for (uint8_t c : code[d])
        if (c == 0) throw Fail{CORRUPT};
      rp += N;
      key[d + 1] = expand(key[d], code[d]);
    }
    if (rp != raw) throw Fail{CORRUPT};
  }
  pos += (raw + 3) / 4 * 4;
  Coder cd(m, L, Dp);
  for (int d = R; d < L; ++d) {
    const size_t N = key[d].size();
    if (N > NL) throw Fail{CORRUPT};  // node counts never exceed the leaf count
    const size_t end = pos + lb[size_t(d - R)];
    if (end > len) throw Fail{TRUNCATED};
    std::vector<uint32_t> p = cd.level_pmf(key, code, d);
    code[d].assign(N, 0);
    for (size_t s0 = 0; s0 < N; s0 += SEG) {
      size_t cnt = std::min(SEG, N - s0);
      pos += rans_decode_segment(bs + pos, end - pos, p.data() + s0 * NCODE, cnt, code[d].data() + s0);
    }
    if (pos != end) throw Fail{CORRUPT};
    key[d + 1] = expand(key[d], code[d]);
  }
  if (key[L].size() != NL) throw Fail{CORRUPT};
  if (Dp)
    for (int d = 0; d <= L; ++d) Dp->put("key/" + std::to_string(d), key[d]);
  return key[L];
}

}  // namespace

// =============================================================================
// C ABI for the Python test harness (oracle/oracle.py).  All functions return a
// status (0 = OK) unless documented otherwise; buffers returned through **out are
// malloc'ed and released with oracle_free().
// =============================================================================
template <class T>
static T* dup_vec(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(std::max<size_t>(1, v.size() * sizeof(T))));
  if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
  return p;
}

extern "C" {

void oracle_free(void* p) { std::free(p); }


#define ORACLE_TRY(...)                 \
  try {                                 \
    __VA_ARGS__;                        \
    return 0;                           \
  } catch (const Fail& f) {             \
    return f.status;                    \
  } catch (const std::exception&) {     \
    return 100;                         \
  }

int oracle_model_load(const uint8_t* bytes, size_t len, void** out) {
  ORACLE_TRY(*out = new Model(parse_model(bytes, len)))
}
void oracle_model_free(void* m) { delete static_cast<Model*>(m); }
uint64_t oracle_model_hash(void* m) { return static_cast<Model*>(m)->hash; }

void* oracle_dump_new() { return new Dump(); }
void oracle_dump_free(void* d) { delete static_cast<Dump*>(d); }
size_t oracle_dump_get(void* d, const char* name, const uint8_t** ptr) {
  Dump* D = static_cast<Dump*>(d);
  auto it = D->t.find(name);
  if (it == D->t.end()) {
    *ptr = nullptr;
    return 0;
  }
  *ptr = it->second.data();
  return it->second.size();
}
int oracle_dump_has(void* d, const char* name) {
  return static_cast<Dump*>(d)->t.count(name) ? 1 : 0;
}
const char* oracle_dump_names(void* d) {
  Dump* D = static_cast<Dump*>(d);
  D->names.clear();
  for (auto& kv : D->t) D->names += kv.first + "\n";
  return D->names.c_str();
}

// Octree: keys (u64) and codes per depth, concatenated depth 0..L; counts[L+1].
int oracle_build_octree(const int32_t* xyz, size_t n, int L, uint64_t** keys, uint8_t** codes, uint32_t* counts) {
  ORACLE_TRY({
    if (L < 1 || L > 21) throw Fail{UNSUPPORTED_DEPTH};
    Tree t = build_tree(xyz, n, L);
    std::vector<uint64_t> k;
    std::vector<uint8_t> c;
    for (int d = 0; d <= L; ++d) {
      counts[d] = uint32_t(t.key[d].size());
      k.insert(k.end(), t.key[d].begin(), t.key[d].end());
      if (d < L) c.insert(c.end(), t.code[d].begin(), t.code[d].end());
    }
    *keys = dup_vec(k);
    *codes = dup_vec(c);
  })
}

int oracle_expand(const uint64_t* keys, const uint8_t* codes, size_t n, uint64_t** out, size_t* n_out) {
  ORACLE_TRY({
    std::vector<uint64_t> k(keys, keys + n);
    std::vector<uint8_t> c(codes, codes + n);
    std::vector<uint64_t> e = expand(k, c);
    *n_out = e.size();
    *out = dup_vec(e);
  })
}

uint64_t oracle_morton(uint32_t x, uint32_t y, uint32_t z, int bits) { return morton(x, y, z, bits); }

int oracle_kernel_map(const uint64_t* keys, size_t n, int depth, int32_t* nbr) {
  ORACLE_TRY({
    std::vector<int32_t> v = kernel_map(std::vector<uint64_t>(keys, keys + n), depth);
    std::memcpy(nbr, v.data(), v.size() * sizeof(int32_t));
  })
}

// Raw int64 accumulators (no bias, no requant) of the K3S1 conv on sparse features.
int oracle_conv3_acc(const uint64_t* keys, size_t n, int depth, const int8_t* f, int cin, const int8_t* W,
                     int cout, int64_t* acc) {
  ORACLE_TRY({
    std::vector<int32_t> nbr = kernel_map(std::vector<uint64_t>(keys, keys + n), depth);
    std::vector<int64_t> a = conv3_acc(nbr, n, f, cin, W, cout);
    std::memcpy(acc, a.data(), a.size() * sizeof(int64_t));
  })
}

// Raw accumulators of the codec's own K2S2 down step (down_acc, called by down_step).
int oracle_down_acc(const uint64_t* child_keys, size_t nc, const uint64_t* parent_keys, size_t np,
                    const int8_t* g, int C, const int8_t* W, int64_t* acc) {
  ORACLE_TRY({
    std::vector<uint64_t> ck(child_keys, child_keys + nc), pk(parent_keys, parent_keys + np);
    Feat gv(g, g + nc * size_t(C));
    std::vector<int64_t> a = down_acc(W, gv, ck, pk, C);
    std::memcpy(acc, a.data(), a.size() * sizeof(int64_t));
  })
}

// The codec's own Eq.7 predictor (head_logits) on explicit weights: a [n][H] int8 and
// z [n][255] int32.
int oracle_head_logits(const int8_t* F, size_t n, int C, int H, const int8_t* W1, const int32_t* b1, int32_t mp,
                       int32_t mn, int32_t r, const int8_t* W2, const int32_t* b2, int8_t* a_out, int32_t* z_out) {
  ORACLE_TRY({
    Head h;
    h.W1.assign(W1, W1 + size_t(H) * C);
    h.b1.assign(b1, b1 + H);
    h.rq1 = RQ{mp, mn, r};
    h.W2.assign(W2, W2 + size_t(NCODE) * H);
    h.b2.assign(b2, b2 + NCODE);
    Feat f(F, F + n * size_t(C));
    Dump D;
    std::vector<int32_t> z = head_logits(h, f, n, C, H, &D, 0);
    std::memcpy(a_out, D.t["a/0"].data(), n * size_t(H));
    std::memcpy(z_out, z.data(), z.size() * sizeof(int32_t));
  })
}

int32_t oracle_rq(int32_t acc, int32_t m, int32_t r) { return rq(acc, m, r); }
int32_t oracle_prq(int32_t acc, int32_t mp, int32_t mn, int32_t r) { return prq(acc, mp, mn, r); }

// Upsampling+Pruning with an explicit layer (W [8C][C+255], b, rq, q_one).
int oracle_up_prune(const int8_t* S, const uint8_t* X, size_t n, int C, const int8_t* W, const int32_t* b,
                    int32_t mp, int32_t mn, int32_t r, int32_t q_one, int8_t** out, size_t* rows) {
  ORACLE_TRY({
    Up u;
    u.W.assign(W, W + size_t(8 * C) * size_t(C + NCODE));
    u.b.assign(b, b + 8 * C);
    u.rq = RQ{mp, mn, r};
    u.q_one = q_one;
    Feat s(S, S + n * size_t(C));
    std::vector<uint8_t> x(X, X + n);
    Feat o = up_prune(u, s, x, C);
    *rows = o.size() / size_t(C);
    *out = dup_vec(o);
  })
}

// Q16 pmf rows from int32 logits z[n][255].
int oracle_cdf(const int32_t* z, size_t n, int32_t m_l, int32_t r_l, const uint32_t* lut, uint32_t* p) {
  ORACLE_TRY({
    std::vector<uint32_t> L(lut, lut + 1024);
    RQ t{m_l, m_l, r_l};
    for (size_t i = 0; i < n; ++i) cdf_quantize(z + i * NCODE, t, L, p + i * NCODE);
  })
}

// One rANS segment from (cum, freq) pairs; decode back with pmf rows.
int oracle_rans_encode(const uint32_t* cum, const uint32_t* freq, size_t n, uint8_t** out, size_t* len) {
  ORACLE_TRY({
    std::vector<uint8_t> o;
    rans_encode_segment(cum, freq, n, o);
    *len = o.size();
    *out = dup_vec(o);
  })
}
int oracle_rans_decode(const uint8_t* in, size_t avail, const uint32_t* p, size_t n, uint8_t* sym, size_t* used) {
  ORACLE_TRY(*used = rans_decode_segment(in, avail, p, n, sym))
}

int oracle_encode(void* model, const int32_t* xyz, size_t n, int L, void* dump, uint8_t** out, size_t* len) {
  ORACLE_TRY({
    std::vector<uint8_t> bs = encode(*static_cast<Model*>(model), xyz, n, L, static_cast<Dump*>(dump));
    *len = bs.size();
    *out = dup_vec(bs);
  })
}

int oracle_decode(void* model, const uint8_t* bs, size_t len, void* dump, int32_t** xyz, size_t* n_out, int* L_out) {
  ORACLE_TRY({
    int L = 0;
    std::vector<uint64_t> k = decode(*static_cast<Model*>(model), bs, len, L, static_cast<Dump*>(dump));
    std::vector<int32_t> p(k.size() * 3);
    for (size_t i = 0; i < k.size(); ++i) {
      uint32_t x, y, z;
      unmorton(k[i], L, x, y, z);
      p[3 * i] = int32_t(x);
      p[3 * i + 1] = int32_t(y);
      p[3 * i + 2] = int32_t(z);
    }
    *n_out = k.size();
    *L_out = L;
    *xyz = dup_vec(p);
  })
}

}  // extern "C"
