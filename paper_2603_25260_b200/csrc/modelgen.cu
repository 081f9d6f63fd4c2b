// modelgen.cu — seeded random-init integer model of the paper's architecture (host code).
//
// No trained checkpoint exists offline (BASELINE.json north_star: "seeded random-init
// integer weights"), so the library can create one: int8 weights uniform in [-63, 63],
// int8 occupancy embeddings in [-100, 100], int32 biases, and requant triples (m, r) set
// from each layer's nominal fan-in so activations keep a std of about 40 (the recipe of
// DESIGN.md §4 "Model generator"; P:300-335 fix the int8 / int32 / fixed-point formats).
// The exp LUT of reading Q20 (LUT[j] = floor(2^24 e^{-j/64} + 1/2), "precomputed
// lookup table") is evaluated here once and stored in the file.  The output is a model
// file with its FNV-1a-64 trailer, loadable by pcc_model_load and by the
// oracle.  This is not the Python generator's byte stream (a different PRNG): parity
// always compares the GPU and the oracle on the SAME saved file.
#include <cmath>
#include <cstring>
#include <vector>

#include "pcc_internal.cuh"

namespace {

struct Rng {  // splitmix64
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  int64_t uniform(int64_t lo, int64_t hi) { return lo + int64_t(next() % uint64_t(hi - lo + 1)); }
};

struct Out {
  std::vector<uint8_t> b;
  void u32(uint32_t v) {
    for (int i = 0; i < 4; ++i) b.push_back(uint8_t(v >> (8 * i)));
  }
  void i32(int32_t v) { u32(uint32_t(v)); }
  void u64(uint64_t v) {
    u32(uint32_t(v));
    u32(uint32_t(v >> 32));
  }
};

constexpr double ACT_STD = 40.0, W_MAX = 63.0;
constexpr int NC = 255;

struct Gen {
  Rng rng;
  Out o;
  int C, H;
  double sa = ACT_STD, sw = W_MAX / std::sqrt(3.0);

  void w(size_t n) {
    for (size_t i = 0; i < n; ++i) o.b.push_back(uint8_t(int8_t(rng.uniform(-63, 63))));
  }
  void emb(size_t n) {
    for (size_t i = 0; i < n; ++i) o.b.push_back(uint8_t(int8_t(rng.uniform(-100, 100))));
  }
  void bias(size_t n, double acc_std) {
    const int64_t lim = int64_t(acc_std / 4.0);
    for (size_t i = 0; i < n; ++i) o.i32(int32_t(rng.uniform(-lim, lim)));
  }
  // requant triple for an accumulator of nominal std acc_std -> target std
  void rq(double acc_std, bool prelu, double target = ACT_STD, int r = 24) {
    const double scale = target / std::max(acc_std, 1e-9);
    int64_t m = std::llround(scale * std::ldexp(1.0, r));
    while (m >= (int64_t(1) << 31)) {
      --r;
      m = std::llround(scale * std::ldexp(1.0, r));
    }
    m = std::max<int64_t>(m, 1);
    const int64_t mn = prelu ? std::max<int64_t>(1, std::llround(double(m) / 4.0)) : m;
    o.i32(int32_t(m));
    o.i32(int32_t(mn));
    o.i32(r);
  }
  void head() {
    const double s1 = sa * sw * std::sqrt(double(C)), sz = sa * sw * std::sqrt(double(H));
    w(size_t(H) * C);
    bias(H, s1);
    rq(s1, true);
    w(size_t(NC) * H);
    bias(NC, sz);
    rq(sz, false, 1.5 * 256.0, 20);  // Q8 logits (reading Q20), about 1.5 nat std
  }
  void up() {
    const int q_one = 127;
    const double s = std::sqrt(C * (sa * sw) * (sa * sw) + (q_one * sw) * (q_one * sw));
    w(size_t(8) * C * (C + NC));
    bias(size_t(8) * C, s);
    rq(s, true);
    o.i32(q_one);
  }
  void resblock_cc() {  // conv_a C->C, conv_b C->C + k_s identity skip (Eq.8, reading Q7)
    const double sc = sa * sw * std::sqrt(7.0 * C);
    w(size_t(27) * C * C);
    bias(C, sc);
    rq(sc, true);
    w(size_t(27) * C * C);
    bias(C, sc);
    o.i32(int32_t(std::llround(sc / sa)));
    rq(std::sqrt(2.0) * sc, false);
  }
};

}  // namespace

namespace pcc {

bool model_config_valid(const pcc_model_config& c) {
  return (c.channels == 8 || c.channels == 16 || c.channels == 32) && c.head_hidden == c.channels &&
         c.raw_levels >= 1 && c.raw_levels <= 6 && c.deep_levels >= 0 && c.deep_levels <= 4 &&
         c.min_depth >= c.raw_levels + 1 + c.deep_levels && c.max_depth >= c.min_depth && c.max_depth <= MAX_DEPTH &&
         (c.flags & ~uint32_t(MF_ALL)) == 0;
}

std::vector<uint8_t> random_model_file(const pcc_model_config& cfg) {
  Gen g{Rng{cfg.seed}, Out{}, cfg.channels, cfg.head_hidden};
  const int C = g.C, R = cfg.raw_levels, nd = cfg.deep_levels;
  Out& o = g.o;
  o.b.insert(o.b.end(), {'P', 'C', 'C', 'M'});
  for (uint32_t v : {1u, uint32_t(C), uint32_t(g.H), uint32_t(R), uint32_t(nd), uint32_t(cfg.min_depth),
                     uint32_t(cfg.max_depth)})
    o.u32(v);
  o.u64(cfg.seed);
  o.u32(1024);
  o.u32(cfg.flags);
  o.b.resize(64, 0);
  for (int j = 0; j < 1024; ++j) o.u32(uint32_t(std::floor(std::ldexp(std::exp(-j / 64.0), 24) + 0.5)));
  g.emb(size_t(NC) * C);  // E0 (reading Q14)
  for (int d = R; d < cfg.max_depth - nd; ++d) {  // shallow levels (own weights per depth, Q11)
    g.resblock_cc();
    g.up();
    g.head();
  }
  for (int j = 1; j <= nd; ++j) {  // deep levels j = d - D
    g.emb(size_t(NC) * C);
    for (int s = 0; s < j - 1; ++s) {  // K2S2 down steps (Eq.4)
      const double sd = g.sa * g.sw * std::sqrt(3.0 * C);
      g.w(size_t(8) * C * C);
      g.bias(C, sd);
      g.rq(sd, true);
    }
    if (cfg.flags & MF_XFP_OFF) {
      g.resblock_cc();  // H = ResBlock(G_D) (P:528 ablation)
    } else {            // Eq.10: ResBlock(Concat(F_D, G_D)) with a 1x1 projection skip
      const double sa2 = g.sa * g.sw * std::sqrt(14.0 * C), sb = g.sa * g.sw * std::sqrt(7.0 * C),
                   sp = g.sa * g.sw * std::sqrt(2.0 * C);
      g.w(size_t(27) * C * 2 * C);
      g.bias(C, sa2);
      g.rq(sa2, true);
      g.w(size_t(27) * C * C);
      g.w(size_t(C) * 2 * C);
      g.bias(C, sb);
      g.rq(std::hypot(sb, sp), false);
    }
    for (int s = 0; s < j; ++s) g.up();
    g.head();
  }
  uint64_t h = 0xCBF29CE484222325ull;
  for (uint8_t b : o.b) {
    h ^= b;
    h *= 0x100000001B3ull;
  }
  o.u64(h);
  return o.b;
}

}  // namespace pcc
