/*
 * pcc.h — C ABI of the B200-native integer-only octree LiDAR coder.
 *
 * Hot path of "Towards Practical Lossless Neural Compression for LiDAR Point
 * Clouds" (arxiv 2603.25260; PAPER.md = P:<line>).  Per octree level the coder
 * builds the Morton-ordered voxel set and its occupancy bytes, runs
 * the GRED / XFP context network in integer-only arithmetic (Eq.4-14),
 * turns the predictor's 255 logits into an exact Q16 distribution with a LUT
 * softmax (Eq.15) and rANS-codes the occupancy bytes (
 * the coder itself is our reading Q23).  Decoding is level-serial
 * (Eq.2) and parallel within a level.
 *
 * Conventions (all functions):
 *  - Every compute call requires an sm_100 device; there is no CPU fallback.
 *    Without one, calls return PCC_ERR_CUDA.
 *  - Buffers named d_* are DEVICE pointers owned by the caller (e.g. torch tensors'
 *    data_ptr()); h_* and plain arrays are HOST pointers owned by the caller.  The
 *    library never frees caller memory.  Handles (pcc_model, pcc_ctx) are owned by
 *    the library and released with *_destroy.
 *  - Work is ordered on the ctx's CUDA stream.  Calls return after their output
 *    lengths are known (each call synchronises the ctx stream at least once).
 *  - On error no partial output is promised.  On PCC_ERR_CAPACITY the *_len /
 *    *n_out arguments receive the required size.
 *  - Coordinates are int32 [n][3] (x, y, z), row-major, each in [0, 2^bit_depth).
 *    Duplicates are allowed.  Decoded output is the set of unique voxels in Morton
 *    order (reading Q27), so decode(encode(x)) == sorted_unique(x).
 */
#ifndef PCC_H_
#define PCC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PCC_OK = 0,
  PCC_ERR_INVALID_ARG = 1,      /* null pointer, bad frame offsets, malformed model file */
  PCC_ERR_EMPTY = 2,            /* a frame with zero points (SPEC S:669 EmptyCloud) */
  PCC_ERR_RANGE = 3,            /* a coordinate outside [0, 2^bit_depth) */
  PCC_ERR_UNSUPPORTED_DEPTH = 4,/* bit_depth outside [max(R+5, min_depth), min(max_depth, 21)] */
  PCC_ERR_CAPACITY = 5,         /* output buffer too small; required size returned */
  PCC_ERR_BAD_MAGIC = 6,        /* bitstream does not start with "PCC1" */
  PCC_ERR_VERSION = 7,          /* unsupported bitstream version */
  PCC_ERR_MODEL_MISMATCH = 8,   /* bitstream model hash / R / n_deep differ */
  PCC_ERR_TRUNCATED = 9,        /* bitstream shorter than its header says */
  PCC_ERR_CORRUPT = 10,         /* inconsistent payload (word counts, states, N_L) */
  PCC_ERR_CUDA = 11,            /* no sm_100 device or a CUDA runtime failure */
  PCC_ERR_OOM = 12              /* device allocation failed */
} pcc_status;

/* Immutable after creation; holds the device-resident int8 weights, int32
 * biases, requant triples and the exp LUT.  Safe to share between contexts on
 * the same device. */
typedef struct pcc_model_s* pcc_model;
/* Per (device, stream) workspace arena; grows on demand, never shrinks; not
 * thread-safe.  Reuse one ctx across calls to avoid steady-state allocation. */
typedef struct pcc_ctx_s* pcc_ctx;

/* Model flags (model-file header word at byte 44, stamped into every bitstream):
 *  PCC_MODEL_XFP_OFF  Table 4's "Baseline + GRED" ablation: deep levels
 *                     code from H = ResBlock(G_D) without the cross-scale concat of Eq.10.
 *  PCC_MODEL_RAW_FREQ the raw prefix X_0..X_{R-1} is coded "based on their symbol
 *                     frequencies" (adaptive counts + one rANS lane, DESIGN.md
 *                     reading Q13') instead of stored as plain bytes (reading Q13).
 * deep_levels = 0 is Table 4's GRED-off "Baseline": every level shallow. */
#define PCC_MODEL_XFP_OFF 1u
#define PCC_MODEL_RAW_FREQ 2u

/* Architecture of a model.  channels C in {8, 16, 32}; head_hidden H = C
 * (reading Q9); raw_levels R in [1, 6] (reading Q12); deep_levels n_deep in [0, 4] (4 = the
 * paper's t = L - 4; 3 = the t = L - 3 ablation; 0 = GRED off); the model
 * codes bit depths L in [min_depth, max_depth] with R + 1 + n_deep <= min_depth and
 * max_depth <= 21 (63-bit Morton keys); seed of the random initialisation; flags above. */
typedef struct {
  int channels, head_hidden, raw_levels, deep_levels, min_depth, max_depth;
  uint64_t seed;
  uint32_t flags;
} pcc_model_config;

/* Model file = DESIGN.md §4 "Model file" (little-endian, FNV-1a-64 trailer).
 * Parses and validates it (hash -> MODEL_MISMATCH; layout, exp table outside
 * (65281, 2^24] or increasing, unsupported shape -> INVALID_ARG) and uploads it to
 * `device`.  The caller keeps ownership of `bytes`. */
pcc_status pcc_model_load(const void* bytes, size_t len, int device, pcc_model* out);
/* Seeded random-init integer model of the architecture `cfg` (int8 weights, int32
 * biases, fixed-point requant triples and the exp LUT; no trained checkpoint
 * exists offline), uploaded to `device`.  INVALID_ARG for an unsupported cfg. */
pcc_status pcc_model_create_random(const pcc_model_config* cfg, int device, pcc_model* out);
/* The same model FILE as pcc_model_create_random builds, written to host memory without
 * touching a GPU (buf may be NULL to query *len).  CAPACITY if cap < *len. */
pcc_status pcc_model_random_file(const pcc_model_config* cfg, void* buf, size_t cap, size_t* len);
/* Serialise a loaded / created model to its model file (host buf, cap bytes).  *len =
 * file size; CAPACITY (with *len set) if cap is too small; buf may be NULL to query. */
pcc_status pcc_model_save(pcc_model m, void* buf, size_t cap, size_t* len);
pcc_status pcc_model_hash(pcc_model m, uint64_t* out);
pcc_status pcc_model_flags(pcc_model m, uint32_t* out);
/* channels C, head hidden H, raw levels R, deep levels n_deep, min/max depth. */
pcc_status pcc_model_info(pcc_model m, int* C, int* H, int* R, int* n_deep, int* min_depth, int* max_depth);
void pcc_model_destroy(pcc_model m);

/* stream: a cudaStream_t cast to void* (NULL = legacy default stream). */
pcc_status pcc_ctx_create(int device, void* stream, pcc_ctx* out);
void pcc_ctx_destroy(pcc_ctx c);

/* Worst-case encoded size of one frame of n points (bytes). */
size_t pcc_encode_bound(size_t n, int bit_depth);

/* Octree of one frame.  d_xyz: device int32 [n][3].  Fills
 * h_level_counts[bit_depth+1] with the node count N_d of each depth d = 0..L
 * (N_L = unique voxels) and, if d_codes != NULL, writes the occupancy bytes
 * X_0 | X_1 | ... | X_{L-1} (depth-major, Morton order) into d_codes
 * (device, capacity codes_cap bytes; CAPACITY if sum_{d<L} N_d > codes_cap). */
pcc_status pcc_build_octree(pcc_ctx c, const int32_t* d_xyz, size_t n, int bit_depth,
                            uint8_t* d_codes, size_t codes_cap, uint32_t* h_level_counts);

/* HRCS statistic (Fig.1c: "(i) the total number of nodes at each level, and
 * (ii) the average number of occupied neighbors within a 3x3x3 neighborhood"; SPEC
 * hrcs_stats S:158-166).  `frames` frames concatenated in d_xyz (device int32 [n][3]);
 * offs is a HOST array of frames+1 point offsets; every frame non-empty (EMPTY),
 * coordinates < 2^bit_depth (RANGE), bit_depth in [1, 21].  Fills the HOST arrays
 * h_nodes[f*(L+1) + d] = N_d of frame f and h_nbr[f*(L+1) + d] = sum over frame f's
 * depth-d nodes of the number of occupied coordinates among the node's 26 neighbours
 * (exact hash membership, frames never see each other); the paper's mean is
 * h_nbr / h_nodes.  Caller owns all buffers; no partial output on error. */
pcc_status pcc_hrcs_stats(pcc_ctx c, const int32_t* d_xyz, const size_t* offs, int frames, int bit_depth,
                          uint64_t* h_nodes, uint64_t* h_nbr);

/* Encode one frame (the paper's encoder, Fig.2 / P:139-151): octree of the Morton-sorted
 * unique voxels, level-wise occupancy prediction "in a layer-wise
 * autoregressive manner" (Eq.2) by the integer-only GRED/XFP network (Eq.4-14),
 * the Eq.15 integer softmax, and entropy coding of the occupancy symbols with the
 * predicted distributions.  d_xyz device int32 [n][3] -> bitstream at d_out
 * (device, out_cap bytes).  *out_len = bytes written (or required, on CAPACITY).  Errors:
 * EMPTY (n = 0), RANGE, UNSUPPORTED_DEPTH, CAPACITY, CUDA, OOM. */
pcc_status pcc_encode(pcc_ctx c, pcc_model m, const int32_t* d_xyz, size_t n, int bit_depth,
                      uint8_t* d_out, size_t out_cap, size_t* out_len);

/* Decode one bitstream (Eq.2: level l's distribution depends only on decoded levels < l,
 * P:177-184, so decoding is level-serial and parallel within a level; the decoder
 * expands each decoded level as P:654-655 describes).  d_bs: device bytes d_bs[len];
 * output d_xyz_out device int32 [cap_points][3]: the unique voxels in Morton order.
 * *n_out = unique voxels, *bit_depth_out = L from the header.  Validation order: magic
 * (BAD_MAGIC), version (VERSION), model hash / R / n_deep / flags (MODEL_MISMATCH)
 * before any entropy decoding; TRUNCATED / CORRUPT never hang; CAPACITY sets *n_out. */
pcc_status pcc_decode(pcc_ctx c, pcc_model m, const uint8_t* d_bs, size_t len,
                      int32_t* d_xyz_out, size_t cap_points, size_t* n_out, int* bit_depth_out);

/* Throughput variants (the frame-level data parallelism of BASELINE.json north_star;
 * frames are independent, P:651-660 builds each frame's octree on its own): `frames`
 * frames concatenated.  offs / bs_offs are HOST
 * arrays of frames+1 prefix offsets (points / bytes).  All frames of a batch
 * share bit_depth.  out_offs (HOST, frames+1) receives the per-frame bitstream
 * (encode, bytes) or voxel (decode, points) prefix offsets into d_out /
 * d_xyz_out.  Each frame's bitstream is identical to pcc_encode of that frame
 * alone; frames start at 4-byte-aligned offsets (zero padding in between). */
pcc_status pcc_encode_batch(pcc_ctx c, pcc_model m, const int32_t* d_xyz, const size_t* offs, int frames,
                            int bit_depth, uint8_t* d_out, size_t out_cap, size_t* out_offs);
pcc_status pcc_decode_batch(pcc_ctx c, pcc_model m, const uint8_t* d_bs, const size_t* bs_offs, int frames,
                            int32_t* d_xyz_out, size_t cap_points, size_t* out_offs);

/* Host-buffer convenience (end-to-end path): copies h_xyz (host int32 [n][3])
 * to the device, encodes the batch, copies the bitstreams back into h_out. */
pcc_status pcc_encode_batch_host(pcc_ctx c, pcc_model m, const int32_t* h_xyz, const size_t* offs, int frames,
                                 int bit_depth, uint8_t* h_out, size_t out_cap, size_t* out_offs);
pcc_status pcc_decode_batch_host(pcc_ctx c, pcc_model m, const uint8_t* h_bs, const size_t* bs_offs, int frames,
                                 int32_t* h_xyz_out, size_t cap_points, size_t* out_offs);

/* Debug / parity: copy a named intermediate tensor of the LAST call on this ctx
 * (single-frame calls only) to host memory.  Names follow the oracle's dumps:
 * "key/d" (u64), "code/d" (u8), "nbr/d" (i32 [N][27], absent = -1), "F/d",
 * "ha/d", "S/d", "G/l/d", "hx/l", "H/l", "Fp/l/d", "a/l" (i8 [N][C or H]),
 * "cf/l" (u16 pairs cum,freq; encode), "cdf/l" (u16 [N][256] cumulative; decode).
 * *len = bytes available; copies min(cap, len).  INVALID_ARG if unknown. */
pcc_status pcc_debug_tensor(pcc_ctx c, const char* name, void* h_dst, size_t cap, size_t* len);
/* Self-test of the tensor-core primitive used by the path (tcgen05.mma kind::i8,
 * int32 accumulation in TMEM): h_d[128][n_cols] = h_a[128][32] * h_b[n_cols][32]^T,
 * all HOST row-major int8/int32 arrays; n_cols in {32, 64, ..., 256}. */
pcc_status pcc_debug_gemm_i8(pcc_ctx c, const int8_t* h_a, const int8_t* h_b, int n_cols, int32_t* h_d);
/* Enable (1) / disable (0) retention of intermediate tensors for
 * pcc_debug_tensor (adds device->host copies; parity tests only). */
pcc_status pcc_ctx_set_debug(pcc_ctx c, int on);
/* Kernel launches issued by the last call on this ctx (own kernels only). */
uint64_t pcc_ctx_launch_count(pcc_ctx c);

/* Profiling: when on, every kernel launch is bracketed by CUDA events on the ctx
 * stream and accumulated per category ("sort", "octree", "kmap", "conv", "down",
 * "up", "head", "rans_enc", "rans_dec", "pack", "expand", ...).  Turning it on or
 * off resets the totals.  profile_get(category = NULL) returns the sum over
 * categories.  bytes = algorithmic (compulsory) bytes the launches move
 * (DESIGN.md §5), for roofline accounting.  Categories: newline-separated list. */
pcc_status pcc_ctx_set_profile(pcc_ctx c, int on);
pcc_status pcc_ctx_profile_get(pcc_ctx c, const char* category, double* ms, uint64_t* launches, uint64_t* bytes);
const char* pcc_ctx_profile_categories(pcc_ctx c);

const char* pcc_status_string(pcc_status s);

#ifdef __cplusplus
}
#endif
#endif /* PCC_H_ */
