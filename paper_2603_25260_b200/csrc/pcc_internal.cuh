// pcc_internal.cuh — shared declarations of the CUDA path (sm_100a).
// Nothing here is shared with oracle/: the two implementations are independent.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <map>
#include <string>
#include <vector>

#include "../../include/pcc.h"

namespace pcc {

constexpr int NCODE = 255;     // occupancy classes
constexpr int SEG_SYMS = 4096;  // rANS segment length (reading Q24': <= 512 steps per lane, K <= 8)
constexpr int MAX_LANES = 8;
constexpr int MAX_DEPTH = 21;   // 63-bit Morton key cap

// Device error flags (atomicOr'ed by kernels, read at sync points).
enum : uint32_t {
  EF_RANGE = 1u << 0,
  EF_CORRUPT = 1u << 1,
};

struct RQ {  // fixed-point requant, Eq.14; m_neg != m_pos = fused PReLU (reading Q18)
  int32_t mp, mn, r;
  // precomputed by rq_prepare (rq.cuh): the one-multiply exact forms
  int32_t fast;       // |x| form valid (Mp, Mn, Ap, An)
  uint32_t Mp, Mn, Ap, An;
  int32_t fast_s;     // signed form valid (Sp, Sn)
  int32_t Sp, Sn;
};

struct DConv {       // K3S1 conv: W [27][cout][cin], b [cout]
  const int8_t* W;
  const int32_t* b;
  RQ rq;
};
struct DUp {         // Upsampling over Concat(S, onehot X): W_S [8C][C], E [255][8C] (= q_one*W_X), b [8C]
  const int8_t* W;
  const int32_t* E;
  const int32_t* b;
  RQ rq;
  // WXt [255][8C] int8 = W_X transposed (row v = the weights of one-hot column v) and the
  // one-hot value q_one, for the tensor-core kernel: E[v][o] = q_one * WXt[v][o]
  const int8_t* WXt;
  int32_t q_one;
};
struct DHead {       // Predictor: W1 [H][C], b1, rq1; W2 [256][H] (row 255 = 0), b2 [256]; logit rq
  const int8_t* W1;
  const int32_t* b1;
  RQ rq1;
  const int8_t* W2;
  const int32_t* b2;
  RQ rql;
  // Saturation thresholds of the logit requant (exact, computed at load): z > zsat_hi
  // gives +2^24, z < zsat_lo gives -2^24, otherwise the result fits in 32 bits.
  int32_t zsat_lo, zsat_hi;
  // false when max_i(|b2_i| + 128 sum_h |W2_ih|) is inside both thresholds
  bool can_saturate;
  // head4_tc.cu: the biases as a second K = 32 MMA slab, b = 127 sum_{j<31} d_j + d_31
  // (B1d [32][32], rows >= H zero; B2d [256][32], row 255 zero); valid iff bias_fold
  const int8_t* B1d;
  const int8_t* B2d;
  bool bias_fold;
};
struct DShallow {
  DConv a, b;
  int32_t k_s;
  DUp up;
  DHead head;
};
struct DDown {       // K2S2: W [8][C][C], b [C]
  const int8_t* W;
  const int32_t* b;
  RQ rq;
};
struct DDeep {
  const int8_t* E;   // [255][C]
  DDown down[3];
  DConv a;           // [27][C][2C]  (XFP off: [27][C][C])
  DConv b;           // [27][C][C]
  const int8_t* P;   // [C][2C]      (XFP off: null, identity skip k_s * G_D instead)
  int32_t k_s;
  DUp up[4];
  DHead head;
};

}  // namespace pcc

// Model flags (DESIGN.md §4 "Model file", header word at byte 44; stamped into the
// bitstream's flags byte): the Table 4 "Baseline + GRED" ablation without cross-scale
// propagation and the P:601 symbol-frequency raw-prefix coder.  n_deep = 0 is the
// GRED-off "Baseline".
enum : uint32_t { MF_XFP_OFF = 1u, MF_RAW_FREQ = 2u, MF_ALL = 3u };

struct pcc_model_s {
  int device = 0;
  int C = 0, H = 0, R = 0, n_deep = 0, min_depth = 0, max_depth = 0;
  uint32_t flags = 0;
  std::vector<uint8_t> file;  // the model file image (pcc_model_save)
  uint64_t hash = 0;
  void* dmem = nullptr;
  const uint32_t* lut = nullptr;
  const int8_t* E0 = nullptr;
  std::vector<pcc::DShallow> shallow;  // index d - R
  std::vector<pcc::DDeep> deep;        // index j - 1
};

struct pcc_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  struct Buf {
    void* p = nullptr;
    size_t cap = 0;
  };
  std::map<std::string, Buf> bufs;
  void* pinned = nullptr;
  size_t pinned_cap = 0;
  void* pinned1 = nullptr;   // second pinned staging buffer (the decoder's segment-list ring)
  size_t pinned1_cap = 0;
  bool debug = false;
  std::map<std::string, std::vector<uint8_t>> dbg;
  uint64_t launches = 0;
  // per-category CUDA-event timing of launches (pcc_ctx_set_profile)
  bool prof = false;
  struct Rec {
    std::string cat;
    cudaEvent_t a, b;
    uint64_t bytes;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  struct Tot {
    double ms = 0;
    uint64_t launches = 0, bytes = 0;
  };
  std::map<std::string, Tot> tot;
};

namespace pcc {

struct Error {
  pcc_status st;
};

#define PCC_CUDA(x)                                      \
  do {                                                   \
    cudaError_t e_ = (x);                                \
    if (e_ != cudaSuccess) throw ::pcc::Error{e_ == cudaErrorMemoryAllocation ? PCC_ERR_OOM : PCC_ERR_CUDA}; \
  } while (0)

// One-time, per-device, thread-safe cudaFuncSetAttribute(MaxDynamicSharedMemorySize) at
// a launch site: the attribute is set on the current device before its bit is published,
// so a thread that sees the bit also sees the attribute; a race only sets it twice.
#define PCC_SMEM_ATTR(kern, bytes)                                                           \
  do {                                                                                       \
    static std::atomic<uint64_t> attr_mask_{0};                                              \
    int dev_ = 0;                                                                            \
    PCC_CUDA(cudaGetDevice(&dev_));                                                          \
    const uint64_t bit_ = 1ull << (dev_ & 63);                                               \
    if (!(attr_mask_.load(std::memory_order_acquire) & bit_)) {                              \
      PCC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes))); \
      attr_mask_.fetch_or(bit_, std::memory_order_release);                                  \
    }                                                                                        \
  } while (0)

// Workspace arena: named buffers, grown on demand, never shrunk.
void* ws(pcc_ctx c, const char* name, size_t bytes);
template <class T>
T* wsT(pcc_ctx c, const char* name, size_t count) {
  return static_cast<T*>(ws(c, name, count * sizeof(T) + 16));
}
void* pinned(pcc_ctx c, size_t bytes);
void* pinned_ring(pcc_ctx c, size_t bytes);  // a separate buffer, not shared with pinned()
void launched(pcc_ctx c, int n = 1);

// Scoped event pair around one launch of category `cat` (only when profiling is on).
// `bytes` = algorithmic (compulsory) bytes the launch moves, for roofline accounting.
struct Prof {
  pcc_ctx c;
  const char* cat;
  uint64_t bytes;
  cudaEvent_t a = nullptr, b = nullptr;
  Prof(pcc_ctx c_, const char* cat_, uint64_t bytes_);
  ~Prof();
};
void prof_collect(pcc_ctx c);
void dbg_copy(pcc_ctx c, const std::string& name, const void* dptr, size_t bytes);

// ---- scan.cu ----
// Exclusive scan of n u32 values; out[n] receives the total.  in may equal out.
void scan_u32(pcc_ctx c, const uint32_t* in, uint32_t* out, size_t n);

// ---- octree.cu ----
struct OctreeOut {            // concatenated across depths; node arrays indexed nb[d] + local
  std::vector<uint32_t> N;    // N[d], d = 0..L (totals over frames)
  std::vector<uint64_t> nb;   // base offset of depth d in the concatenated arrays
  std::vector<uint32_t> foff; // host copy: foff[d*(B+1) + f] local index of frame f's first node at depth d
};
// Encoder: Morton keys + radix sort + all levels.  Fills ctx buffers
// "key" (u64), "code" (u8), "cs" (u32 child start, local), "par" (u32 parent, local),
// "foff" (u32 [(L+1)*(B+1)]).
void build_octree(pcc_ctx c, const int32_t* d_xyz, const size_t* offs, int B, int L, OctreeOut& o);
// Decoder: expand depth d -> d+1 from decoded codes (arrays as above).  Returns N_{d+1}.
// err (device flags, may be null): read back with the child count in the level's single sync.
uint32_t expand_level(pcc_ctx c, int d, int B, OctreeOut& o, uint32_t max_nodes, const uint32_t* err = nullptr);
// Morton-decode depth-L keys of all frames into xyz (frame bits dropped).
void keys_to_xyz(pcc_ctx c, const uint64_t* keys, size_t n, int L, int32_t* xyz);
// HRCS: d_sum[f] = sum over frame f's depth-d nodes of occupied 26-neighbours.
void hrcs_counts(pcc_ctx c, const uint64_t* keys, uint32_t N, int depth, int B, unsigned long long* d_sum);

// ---- kmap.cu ----
// nbr[N][27] for the N nodes of one depth (keys include frame bits); absent -> N.
void kernel_map(pcc_ctx c, const uint64_t* keys, uint32_t N, int depth, int32_t* nbr);
// the same map derived from the parent depth's map (pnbr [Np][27], absent = Np), the parent
// codes Xp and child starts csp (local to depth d) and the nodes' parents par (local)
void kernel_map_derive(pcc_ctx c, const uint64_t* keys, const uint32_t* par, uint32_t N, const int32_t* pnbr,
                       uint32_t Np, const uint8_t* Xp, const uint32_t* csp, int32_t* nbr);

// ---- nn.cu ----
void embed(pcc_ctx c, const int8_t* E, const uint8_t* X, uint32_t n, int C, int8_t* out);
// out = act(conv3([in0 | in1]) + skip + b) with the zero row written at index n.
//   skip_mode 0: none; 1: k_s * skip0[i]; 2: P [cout][2C] * [skip0 | skip1][i]
void conv3(pcc_ctx c, const int8_t* in0, const int8_t* in1, int C, uint32_t n, const int32_t* nbr,
           const DConv& L, int skip_mode, const int8_t* skip0, const int8_t* skip1, int32_t k_s, const int8_t* P,
           int8_t* out);
void down(pcc_ctx c, const int8_t* g, const uint8_t* Xp, const uint32_t* cs_p, uint32_t np, int C, const DDown& L,
          int8_t* out);
void up_prune(pcc_ctx c, const int8_t* S, const uint8_t* Xp, const uint32_t* par_c, const uint64_t* key_c,
              uint32_t nc, int C, const DUp& L, int8_t* out);
// mode 0: encoder -> cf[n] (cum | freq<<16) for true symbols X; mode 1: decoder -> cdf rows u16[n][256]
void head_cdf(pcc_ctx c, const int8_t* F, uint32_t n, int C, int H, const DHead& L, const uint32_t* lut, int mode,
              const uint8_t* X, uint32_t* cf, uint16_t* cdf, int8_t* a_dbg);

// ---- head_tc.cu (tcgen05 kind::i8 predictor + softmax; same contract as head_cdf) ----
void head_cdf_tc(pcc_ctx c, const int8_t* F, uint32_t n, int C, int H, const DHead& L, const uint32_t* lut, int mode,
                 const uint8_t* X, uint32_t* cf, uint16_t* cdf, int8_t* a_dbg);
void gemm_i8_test(pcc_ctx c, const int8_t* dA, const int8_t* dB, int N, int32_t* dD);
// ---- head1_tc.cu (same contract; one thread per node, no row barriers: the default) ----
void head_cdf_tc1(pcc_ctx c, const int8_t* F, uint32_t n, int C, int H, const DHead& L, const uint32_t* lut, int mode,
                  const uint8_t* X, uint32_t* cf, uint16_t* cdf, int8_t* a_dbg);
// ---- head3_tc.cu (same contract; one thread per node, N = 128 half accumulators, ng = 3 or 4
// tile groups per SM) ----
void head_cdf_tc4(pcc_ctx c, const int8_t* F, uint32_t n, int C, int H, const DHead& L, const uint32_t* lut, int mode,
                  const uint8_t* X, uint32_t* cf, uint16_t* cdf, int8_t* a_dbg);
void head_cdf_tc3(pcc_ctx c, const int8_t* F, uint32_t n, int C, int H, const DHead& L, const uint32_t* lut, int mode,
                  const uint8_t* X, uint32_t* cf, uint16_t* cdf, int8_t* a_dbg, int ng);
// ---- head2_tc.cu (same contract; two threads per node, 16 warps per SM) ----
void head_cdf_tc2(pcc_ctx c, const int8_t* F, uint32_t n, int C, int H, const DHead& L, const uint32_t* lut, int mode,
                  const uint8_t* X, uint32_t* cf, uint16_t* cdf, int8_t* a_dbg);

// ---- up_tc.cu (parents x W_S on tcgen05, pruned epilogue; C = 32) ----
// S: parent rows (np), Xp / cs_p: parent codes / child starts, nc: child rows (out has nc+1)
void up_prune_tc(pcc_ctx c, const int8_t* S, const uint8_t* Xp, const uint32_t* par_c, const uint64_t* key_c,
                 uint32_t nc, const DUp& L, int8_t* out);

// ---- down_tc.cu (K2S2 downsampling as a block-diagonal tcgen05 product; C = 32) ----
void down_tc(pcc_ctx c, const int8_t* g, const uint8_t* Xp, const uint32_t* cs_p, uint32_t np, const DDown& L,
             int8_t* out,
             const uint8_t* Xc = nullptr);

// ---- conv_tc.cu (gather -> tcgen05 kind::i8 per kernel offset; C = 32) ----
void conv3_tc(pcc_ctx c, const int8_t* in0, const int8_t* in1, uint32_t n, const int32_t* nbr, const DConv& L,
              int skip_mode, const int8_t* s0, const int8_t* s1, int32_t k_s, const int8_t* P, int8_t* out);

// ---- rans.cu ----
struct EncSeg {      // one rANS segment of the encoder
  uint32_t node;     // first symbol (index into the concatenated cf / code arrays)
  uint32_t n;        // symbols
};
void rans_encode(pcc_ctx c, const EncSeg* d_segs, int nseg, const uint32_t* cf, uint16_t* words, uint32_t* seg_W,
                 uint32_t* seg_state,
                 size_t nsym = 0);
struct DecSeg {
  uint64_t byte;     // offset of the segment's level payload in the bitstream buffer
  uint32_t chunk;    // segment index within the level payload
  uint32_t node;     // first symbol (local index within the depth)
  uint32_t n;        // symbols
  uint32_t level_bytes;
  uint32_t last;     // 1 if this is the level's last segment (must end the payload)
};
// Decoder row per node (DESIGN.md §5 "decoder rows", reading Q21): u32 S = sum_i e_i,
// u32 inv32 = floor(65281 * 2^32 / S), i32 mu = max_i l_i (the Q8 logit maximum), u32
// E_{16k} for k = 1..15 (prefix mass before symbol 16k) at word 2 + k, 8 zero bytes, then
// the H hidden activations a (int8, Eq.7's C -> H layer) at byte DROW_A = 80, zero padded
// to 32 bytes: 112 bytes (a 16-byte multiple for TMA, a 16-byte aligned).  The rANS decoder recomputes the 16 logits of the one block
// its coarse test selects (z_i = b2_i + a . W2_i, exact int32), their exponentials e_i =
// LUT[(mu - l_i) >> 2] and C_i = i + floor(E_i * 65281 / S) where its search needs them.
constexpr int DROW_BYTES = 112, DROW_A = 80, DROW_U16 = DROW_BYTES / 2;
void rans_decode(pcc_ctx c, const DecSeg* d_segs, int nseg, const uint8_t* bs, const uint16_t* rows, int H,
                 const DHead& head, const uint32_t* lut, uint8_t* X, uint32_t* err, int max_lanes, size_t nsym, size_t nstates);

// ---- modelgen.cu ----
bool model_config_valid(const pcc_model_config& c);
std::vector<uint8_t> random_model_file(const pcc_model_config& c);

// ---- rawcoder.cu (raw prefix X_0..X_{R-1}: plain bytes, or the P:601 frequency coder) ----
uint32_t raw_max_symbols(int R);  // sum_{d<R} 8^d
// sz[f] = raw region bytes of frame f; freq: region written at region + f * cap
void raw_encode(pcc_ctx c, bool freq, const uint8_t* code, const uint64_t* d_nb, const uint32_t* d_foff, int B, int R,
                uint8_t* region, uint32_t cap, uint32_t* sz);
// decodes the frequency-coded regions: symbols at sym + f * raw_max_symbols(R), node
// counts per depth cnt[f * (R + 1) + d] (0 at d = R and EF_CORRUPT on a bad region)
void raw_decode(pcc_ctx c, const uint8_t* bs, const uint64_t* raw_off, const uint32_t* raw_len, int B, int R,
                const uint32_t* d_NL, uint8_t* sym, uint32_t* cnt, uint32_t* err);

// ---- pack (runtime.cu) ----
struct PackItem {    // encoder output item: frame header+raw prefix (kind 0) or one segment (kind 1)
  uint32_t kind;
  uint32_t frame;
  uint32_t seg;      // kind 1: encoder segment index
  uint32_t level;    // kind 1: coded depth d
  uint32_t bytes;    // kind 0: header + padded raw prefix bytes
  uint32_t nitems;   // kind 0: items of this frame (header + its segments)
};

}  // namespace pcc
