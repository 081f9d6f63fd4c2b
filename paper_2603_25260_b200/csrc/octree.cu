// octree.cu — Morton keys, LSD radix sort, per-level occupancy bytes (encoder) and
// level expansion (decoder).  PAPER.md P:651-660: "sort the input coordinates in Morton
// order ... repeatedly divide them by 2, apply floor rounding, and remove consecutive
// duplicates"; occupancy codes = the K2S2 all-ones conv (bit-equivalent OR of child bits);
// decoder "adding a pre-defined offset matrix ... masking" preserves Morton order.
//
// Frames of a batch are sorted together: key = frame << 3L | morton (bits 3L..), so each
// frame stays contiguous and every depth's node list is frame-major, Morton-minor.
#include "pcc_internal.cuh"

namespace pcc {

namespace {

__device__ __forceinline__ uint64_t spread3(uint32_t v) {
  uint64_t x = v & 0x1fffffu;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}
__device__ __forceinline__ uint32_t compact3(uint64_t x) {
  x &= 0x1249249249249249ull;
  x = (x ^ (x >> 2)) & 0x10c30c30c30c30c3ull;
  x = (x ^ (x >> 4)) & 0x100f00f00f00f00full;
  x = (x ^ (x >> 8)) & 0x1f0000ff0000ffull;
  x = (x ^ (x >> 16)) & 0x1f00000000ffffull;
  x = (x ^ (x >> 32)) & 0x1fffffull;
  return uint32_t(x);
}

// ---- a1: Morton keys (x is the MSB of each bit triple, reading O1/Q25) -------------
// a1 front end in one pass (r2): Morton keys, the consecutive-duplicate drop and the
// compaction together.  Grid (tiles, frames), MD_V points per thread at stride MD_T: each
// CTA counts its kept keys (warp ballots + one shared-memory atomic per warp), reserves its
// range of the frame's output with ONE global atomic, and writes the kept keys from
// registers.  The kept keys of a frame land at out[offs[f] ..  offs[f] + kept[f]) in an
// arbitrary order: the radix sort below orders them (a sort is a function of the multiset),
// so the result is deterministic.
constexpr int MD_T = 256, MD_V = 16, MD_TILE = MD_T * MD_V;
__global__ void __launch_bounds__(MD_T) k_morton_dedup(const int32_t* __restrict__ xyz, const uint64_t* __restrict__ offs,
                                                       int B, int L, uint64_t* __restrict__ out,
                                                       uint32_t* __restrict__ kept, uint32_t* __restrict__ err) {
  __shared__ uint32_t s_cnt, s_base;
  const int f = blockIdx.y;
  const uint64_t a = offs[f];
  const uint32_t nf = uint32_t(offs[f + 1] - a);
  const uint32_t c0 = blockIdx.x * MD_TILE;
  if (c0 >= nf) return;  // whole CTA
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int32_t lim = 1 << L;
  const uint64_t fb = B > 1 ? uint64_t(f) << (3 * L) : 0ull;
  uint64_t kv[MD_V];
  uint32_t keepm = 0, woff[MD_V];
  // all MD_V points' coordinates first (independent loads in flight together), then the
  // keys; the previous point of a lane's point is the lower lane's (a shuffle), lane 0
  // loads it
  int32_t px[MD_V], py[MD_V], pz[MD_V], qx[MD_V], qy[MD_V], qz[MD_V];
#pragma unroll
  for (int v = 0; v < MD_V; ++v) {
    const uint32_t i = c0 + uint32_t(v) * MD_T + threadIdx.x;
    px[v] = py[v] = pz[v] = 0;
    qx[v] = qy[v] = qz[v] = -1;
    if (i < nf) {
      const int32_t* p = xyz + 3 * (a + i);
      px[v] = p[0], py[v] = p[1], pz[v] = p[2];
      if (lane == 0 && i > 0) qx[v] = p[-3], qy[v] = p[-2], qz[v] = p[-1];
    }
  }
#pragma unroll
  for (int v = 0; v < MD_V; ++v) {
    const uint32_t i = c0 + uint32_t(v) * MD_T + threadIdx.x;  // frame-local point index
    const int32_t x = px[v], y = py[v], z = pz[v];
    const int32_t ux = __shfl_up_sync(0xffffffffu, x, 1), uy = __shfl_up_sync(0xffffffffu, y, 1),
                  uz = __shfl_up_sync(0xffffffffu, z, 1);
    const int32_t prx = lane ? ux : qx[v], pry = lane ? uy : qy[v], prz = lane ? uz : qz[v];
    bool keep = false;
    kv[v] = 0;
    if (i < nf) {
      if (x < 0 || y < 0 || z < 0 || x >= lim || y >= lim || z >= lim) {
        atomicOr(err, EF_RANGE);
      } else {
        keep = i == 0 || prx != x || pry != y || prz != z;
        kv[v] = fb | spread3(uint32_t(x)) << 2 | spread3(uint32_t(y)) << 1 | spread3(uint32_t(z));
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    uint32_t wb = 0;
    if (lane == 0 && m) wb = atomicAdd(&s_cnt, uint32_t(__popc(m)));
    wb = __shfl_sync(0xffffffffu, wb, 0);
    woff[v] = wb + __popc(m & ((1u << lane) - 1u));
    keepm |= keep ? (1u << v) : 0u;
  }
  __syncthreads();
  if (threadIdx.x == 0) s_base = s_cnt ? atomicAdd(&kept[f], s_cnt) : 0u;
  __syncthreads();
  uint64_t* o = out + a + s_base;
#pragma unroll
  for (int v = 0; v < MD_V; ++v)
    if (keepm >> v & 1u) o[woff[v]] = kv[v];
}

// ---- radix sort (LSD, 8- or 9-bit digits, stable per pass, frame-segmented) ----------
// The input keys are frame-contiguous (frame f = points offs[f]..offs[f+1]) and carry the
// frame id above bit 3L, so only the 3L Morton bits are sorted: every tile lies inside
// one frame, and the per-tile digit counts are laid out frame-major, digit-major,
// tile-minor (hist[256 T0_f + d nt_f + (g - T0_f)] for tile g of frame f, whose tiles
// are T0_f .. T0_f + nt_f), so one exclusive scan of the whole array gives every
// (frame, digit, tile) its output offset and the frames stay where they were.
constexpr int RS_T = 256, RS_V = 16, RS_TILE = RS_T * RS_V, RS_W = RS_T / 32;

struct __align__(16) RsTile {  // tile g -> its frame's key range and histogram geometry
  uint32_t start, count, T0, nt;
};
// once per sort: one thread per tile
__global__ void k_rs_tiles(const uint32_t* __restrict__ tp, const uint64_t* __restrict__ offs, int B, uint32_t ntiles,
                           RsTile* __restrict__ tiles, const uint64_t* __restrict__ in_offs, RsTile* __restrict__ tiles_in) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ntiles) return;
  int lo = 0, hi = B - 1;  // frame: largest f < B with tp[f] <= g
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tp[mid] <= g) lo = mid; else hi = mid - 1;
  }
  RsTile t;
  t.T0 = tp[lo];
  t.nt = tp[lo + 1] - t.T0;
  t.start = uint32_t(offs[lo]) + (g - t.T0) * uint32_t(RS_TILE);
  t.count = min(uint32_t(RS_TILE), uint32_t(offs[lo + 1]) - t.start);
  tiles[g] = t;
  // the first pass reads frame f's keys where k_morton_dedup left them (from in_offs[f])
  t.start = uint32_t(in_offs[lo]) + (g - t.T0) * uint32_t(RS_TILE);
  tiles_in[g] = t;
}

template <int DB>
__global__ void __launch_bounds__(RS_T) k_rs_hist(const uint64_t* __restrict__ keys, int shift,
                                                  const RsTile* __restrict__ tiles, uint32_t* __restrict__ hist) {
  constexpr int ND = 1 << DB;
  constexpr uint32_t MASK = ND - 1;
  __shared__ uint32_t h[ND];
  for (int i = threadIdx.x; i < ND; i += RS_T) h[i] = 0;
  const RsTile t = tiles[blockIdx.x];
  __syncthreads();
#pragma unroll 4
  for (int k = 0; k < RS_V; ++k) {
    const uint32_t i = uint32_t(k) * RS_T + threadIdx.x;
    const uint32_t d = i < t.count ? uint32_t(keys[t.start + i] >> shift) & MASK : uint32_t(ND);
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (d < uint32_t(ND) && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[d], __popc(peers));
  }
  __syncthreads();
  const size_t hb = size_t(ND) * t.T0 + (blockIdx.x - t.T0);
  for (int d = threadIdx.x; d < ND; d += RS_T) hist[hb + size_t(d) * t.nt] = h[d];
}

template <int DB>
__global__ void __launch_bounds__(RS_T) k_rs_scatter(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                                     int shift, const RsTile* __restrict__ tiles,
                                                     const uint32_t* __restrict__ hscan) {
  constexpr int ND = 1 << DB, DPT = ND / RS_T;  // digits per thread in the per-digit phases
  constexpr uint32_t MASK = ND - 1;
  __shared__ uint16_t wc[RS_W][ND + 1];  // per-warp digit counts, then offsets (< RS_TILE)
  __shared__ uint32_t tstart[ND];
  __shared__ uint32_t gbase[ND];
  __shared__ uint32_t wtot[RS_W];
  __shared__ uint64_t stage[RS_TILE];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < RS_W * (ND + 1); i += RS_T) (&wc[0][0])[i] = 0;
  const RsTile t = tiles[blockIdx.x];
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  uint64_t kv[RS_V];
  uint32_t rk[RS_V];
  const uint32_t wbase = uint32_t(w) * (RS_TILE / RS_W);
#pragma unroll
  for (int v = 0; v < RS_V; ++v) {
    const uint32_t i = wbase + uint32_t(v) * 32 + lane;
    const uint64_t k = i < t.count ? in[t.start + i] : 0ull;
    const uint32_t d = i < t.count ? uint32_t(k >> shift) & MASK : uint32_t(ND);
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t base = wc[w][d];
    __syncwarp();
    if (lane == __ffs(peers) - 1) wc[w][d] = uint16_t(base + __popc(peers));
    __syncwarp();
    kv[v] = k;
    rk[v] = (d << 16) | (base + __popc(peers & lt));  // rank < 4096 fits 16 bits
  }
  __syncthreads();
  // per digit: exclusive prefix over warps and the tile count; this thread owns digits
  // DPT * tid .. DPT * tid + DPT - 1 (consecutive, so the block scan is in digit order)
  uint32_t cnt[DPT], s = 0;
#pragma unroll
  for (int j = 0; j < DPT; ++j) {
    const int d = DPT * threadIdx.x + j;
    uint32_t run = 0;
    for (int ww = 0; ww < RS_W; ++ww) {
      const uint32_t c = wc[ww][d];
      wc[ww][d] = uint16_t(run);
      run += c;
    }
    cnt[j] = run;
    s += run;
  }
  uint32_t inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += x;
  }
  if (lane == 31) wtot[w] = inc;
  __syncthreads();
  uint32_t pre = inc - s;
  for (int ww = 0; ww < w; ++ww) pre += wtot[ww];
  const size_t hb = size_t(ND) * t.T0 + (blockIdx.x - t.T0);
#pragma unroll
  for (int j = 0; j < DPT; ++j) {
    const int d = DPT * threadIdx.x + j;
    tstart[d] = pre;
    pre += cnt[j];
    gbase[d] = hscan[hb + size_t(d) * t.nt];
  }
  __syncthreads();
#pragma unroll
  for (int v = 0; v < RS_V; ++v) {
    const uint32_t d = rk[v] >> 16;
    if (d < uint32_t(ND)) stage[tstart[d] + wc[w][d] + (rk[v] & 0xffffu)] = kv[v];
  }
  __syncthreads();
  for (uint32_t p = threadIdx.x; p < t.count; p += RS_T) {
    const uint64_t k = stage[p];
    const uint32_t d = uint32_t(k >> shift) & MASK;
    out[gbase[d] + p - tstart[d]] = k;
  }
}

// ---- a2: all levels at once from the sorted leaf keys --------------------------------
// lvl(i) = first depth at which sorted key i starts a new node (its key differs from key
// i-1 above bit 3(L-d)); duplicates get L+1.  N_d = #{i : lvl(i) <= d}.
__device__ __forceinline__ int leaf_lvl(const uint64_t* keys, size_t i, int L) {
  if (i == 0) return 0;
  uint64_t x = keys[i] ^ keys[i - 1];
  if (x == 0) return L + 1;
  int hb = 63 - __clzll((long long)x);
  int l = L - hb / 3;
  return l < 0 ? 0 : l;
}

constexpr int LV_T = 256, LV_R = 4, LV_TILE = LV_T * LV_R, LV_W = LV_T / 32;

__global__ void __launch_bounds__(LV_T) k_lvl_count(const uint64_t* __restrict__ keys, size_t n, int L,
                                                    uint32_t* __restrict__ cnt, uint32_t nblk) {
  __shared__ uint32_t h[MAX_DEPTH + 2];
  if (threadIdx.x < MAX_DEPTH + 2) h[threadIdx.x] = 0;
  __syncthreads();
  for (int r = 0; r < LV_R; ++r) {
    size_t i = size_t(blockIdx.x) * LV_TILE + size_t(r) * LV_T + threadIdx.x;
    if (i < n) atomicAdd(&h[leaf_lvl(keys, i, L)], 1u);
  }
  __syncthreads();
  if (threadIdx.x <= L) {
    uint32_t s = 0;
    for (int l = 0; l <= int(threadIdx.x); ++l) s += h[l];
    cnt[size_t(threadIdx.x) * nblk + blockIdx.x] = s;
  }
}

// Node index of leaf i at depth d = #{j < i : lvl(j) <= d}.  Per block: all four rounds'
// keys are loaded up front; phase A counts, per (round, warp, depth), the leaves that
// start a node (one ballot per depth from the warp's minimum level); phase B turns the
// counts into exclusive bases (one thread per depth); phase C recomputes the ranks and
// writes each new node (key, child start = own index one depth down, parent = own index
// one depth up (minus one when the node is the parent's continuation), occupancy bit into
// the parent's code).
__global__ void __launch_bounds__(LV_T) k_lvl_scatter(const uint64_t* __restrict__ keys, size_t n, int L, int B,
                                                      const uint32_t* __restrict__ off, uint32_t nblk,
                                                      uint64_t* __restrict__ key_all, uint8_t* __restrict__ code_all,
                                                      uint32_t* __restrict__ cs_all, uint32_t* __restrict__ par_all,
                                                      uint32_t* __restrict__ foff) {
  __shared__ uint32_t wb[LV_R][LV_W][MAX_DEPTH + 2];  // counts, then exclusive local bases
  __shared__ uint32_t nbs[MAX_DEPTH + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  uint64_t key[LV_R];
  int lvl[LV_R];
#pragma unroll
  for (int r = 0; r < LV_R; ++r) {
    const size_t i = size_t(blockIdx.x) * LV_TILE + size_t(r) * LV_T + threadIdx.x;
    key[r] = i < n ? keys[i] : 0ull;
    const uint64_t pk = (i < n && i > 0) ? keys[i - 1] : 0ull;
    int l = L + 1;
    if (i < n) {
      if (i == 0) l = 0;
      else {
        const uint64_t x = key[r] ^ pk;
        if (x != 0) {
          const int hb = 63 - __clzll((long long)x);
          l = L - hb / 3;
          l = l < 0 ? 0 : l;
        }
      }
    }
    lvl[r] = l;
  }
  // phase A
#pragma unroll
  for (int r = 0; r < LV_R; ++r) {
    const int dm = __reduce_min_sync(0xffffffffu, lvl[r]);
    for (int d = 0; d <= L; ++d) {
      const uint32_t cnt = d < dm ? 0u : uint32_t(__popc(__ballot_sync(0xffffffffu, lvl[r] <= d)));
      if (lane == 0) wb[r][w][d] = cnt;
    }
  }
  if (threadIdx.x <= L) nbs[threadIdx.x] = off[size_t(threadIdx.x) * nblk];
  __syncthreads();
  // phase B
  if (threadIdx.x <= L) {
    const int d = threadIdx.x;
    uint32_t sacc = off[size_t(d) * nblk + blockIdx.x] - off[size_t(d) * nblk];
    for (int r = 0; r < LV_R; ++r)
      for (int ww = 0; ww < LV_W; ++ww) {
        const uint32_t cc = wb[r][ww][d];
        wb[r][ww][d] = sacc;
        sacc += cc;
      }
  }
  __syncthreads();
  // phase C
#pragma unroll
  for (int r = 0; r < LV_R; ++r) {
    const int lv = lvl[r];
    const int dm = __reduce_min_sync(0xffffffffu, lv);
    if (dm > L) continue;  // warp of duplicates only
    auto ex = [&](int d) -> uint32_t { return wb[r][w][d] + uint32_t(__popc(__ballot_sync(0xffffffffu, lv <= d) & lt)); };
    const uint64_t k = key[r];
    const int f = (B > 1) ? int(k >> (3 * L)) : 0;
    uint32_t e_prev = dm >= 1 ? ex(dm - 1) : 0u, e_cur = ex(dm);
    for (int d = dm; d <= L; ++d) {
      const uint32_t e_next = d < L ? ex(d + 1) : 0u;
      if (lv <= d) {
        const size_t g = size_t(nbs[d]) + e_cur;
        key_all[g] = k >> (3 * (L - d));
        if (d < L) cs_all[g] = e_next;
        if (d >= 1) {
          const uint32_t p = e_prev - (lv == d ? 1u : 0u);
          par_all[g] = p;
          const size_t gp = size_t(nbs[d - 1]) + p;
          const uint32_t bit = 1u << uint32_t((k >> (3 * (L - d))) & 7u);
          atomicOr(reinterpret_cast<unsigned*>(code_all + (gp & ~size_t(3))), bit << (8 * (gp & 3)));
        }
        if (lv == 0) foff[size_t(d) * (B + 1) + f] = e_cur;
      }
      e_prev = e_cur;
      e_cur = e_next;
    }
  }
}

// counts[d] = N_d, foff[d][B] = N_d
__global__ void k_lvl_totals(const uint32_t* __restrict__ off, uint32_t nblk, int L, int B, uint32_t* __restrict__ counts,
                             uint32_t* __restrict__ foff) {
  int d = threadIdx.x;
  if (d > L) return;
  uint32_t lo = off[size_t(d) * nblk], hi = off[size_t(d + 1) * nblk];
  counts[d] = hi - lo;
  foff[size_t(d) * (B + 1) + B] = hi - lo;
}

// ---- a2': decoder expansion -------------------------------------------------------
__global__ void k_popc(const uint8_t* __restrict__ X, uint32_t n, uint32_t* __restrict__ out) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __popc(uint32_t(X[i]));
}

// cap: room left in the node arrays (a corrupt stream can decode more children than any
// valid one; those are dropped and flagged instead of written out of bounds).  A warp
// expands 32 consecutive parents: their children are one contiguous run of the next
// depth, written lane-strided (coalesced 8- and 4-byte stores); child e of the run belongs
// to the lane whose exclusive child prefix is the largest <= e (binary search over the
// lanes by shuffles), and is that lane's (e - prefix)-th set occupancy bit (__fns).
__global__ void k_expand(const uint64_t* __restrict__ key_d, const uint8_t* __restrict__ X, const uint32_t* __restrict__ cs,
                         uint32_t n, uint64_t* __restrict__ key_c, uint32_t* __restrict__ par_c, uint64_t cap,
                         uint32_t* __restrict__ err) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const uint32_t p0 = p - uint32_t(lane);
  if (p0 >= n) return;  // whole warp
  const bool ok = p < n;
  const uint32_t x = ok ? uint32_t(X[p]) : 0u;
  const uint64_t k = ok ? key_d[p] << 3 : 0ull;
  const uint32_t j0 = cs[p0];
  uint32_t incl = __popc(x);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const uint32_t excl = incl - __popc(x);
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  for (uint32_t e0 = 0; e0 < total; e0 += 32) {
    const uint32_t e = e0 + uint32_t(lane);
    int lo = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const uint32_t ex = __shfl_sync(0xffffffffu, excl, lo + step);
      if (ex <= e) lo += step;
    }
    const uint32_t xo = __shfl_sync(0xffffffffu, x, lo);
    const uint32_t eo = __shfl_sync(0xffffffffu, excl, lo);
    const uint64_t ko = __shfl_sync(0xffffffffu, k, lo);
    if (e < total) {
      const uint32_t c = __fns(xo, 0, int(e - eo) + 1);  // the (e - eo)-th set bit (from 0)
      const uint64_t j = uint64_t(j0) + e;
      if (j < cap) {
        key_c[j] = ko | uint64_t(c);
        par_c[j] = p0 + uint32_t(lo);
      } else if (err) {
        atomicOr(err, EF_CORRUPT);
      }
    }
  }
}

__global__ void k_foff_next(const uint32_t* __restrict__ cs, const uint32_t* __restrict__ foff_d, int B,
                            uint32_t* __restrict__ foff_n) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f <= B) foff_n[f] = cs[foff_d[f]];
}

__global__ void k_keys_to_xyz(const uint64_t* __restrict__ keys, size_t n, int L, int32_t* __restrict__ xyz) {
  size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t m = keys[i] & ((L >= 21) ? ~0ull >> 1 : ((1ull << (3 * L)) - 1ull));
  xyz[3 * i] = int32_t(compact3(m >> 2));
  xyz[3 * i + 1] = int32_t(compact3(m >> 1));
  xyz[3 * i + 2] = int32_t(compact3(m));
}

inline unsigned cdiv(size_t a, size_t b) { return unsigned((a + b - 1) / b); }

}  // namespace

void build_octree(pcc_ctx c, const int32_t* d_xyz, const size_t* offs, int B, int L, OctreeOut& o) {
  const size_t n_in = offs[B];
  cudaStream_t s = c->stream;
  // device copy of frame offsets
  uint64_t* d_offs = wsT<uint64_t>(c, "oct_offs", B + 1);
  // pinned staging, one block (no reallocation while a copy from it is pending): input offs
  // (u64), kept counts (u32), kept offsets (u64), the sort's per-frame first tiles (u32)
  const size_t B1 = size_t(B) + 1, B2 = (B1 + 2) & ~size_t(1);  // hk[B] = the error flags
  uint64_t* h_in = static_cast<uint64_t*>(pinned(c, B1 * 8 + B2 * 4 + B1 * 8 + B1 * 4));
  uint32_t* hk = reinterpret_cast<uint32_t*>(h_in + B1);
  uint64_t* h = reinterpret_cast<uint64_t*>(hk + B2);
  for (int f = 0; f <= B; ++f) h_in[f] = offs[f];
  PCC_CUDA(cudaMemcpyAsync(d_offs, h_in, B1 * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
  uint32_t* err = wsT<uint32_t>(c, "err", 4);
  PCC_CUDA(cudaMemsetAsync(err, 0, 4 * sizeof(uint32_t), s));

  uint64_t* ka = wsT<uint64_t>(c, "sort_a", n_in);
  uint64_t* kb = wsT<uint64_t>(c, "sort_b", n_in);
  uint32_t* kept = wsT<uint32_t>(c, "dd_kept", B);
  uint64_t* d_noffs = wsT<uint64_t>(c, "dd_offs", B + 1);
  PCC_CUDA(cudaMemsetAsync(kept, 0, B * sizeof(uint32_t), s));
  {
    // Morton keys + consecutive-duplicate drop + compaction in one pass: LiDAR frames arrive
    // in scan order, where neighbouring returns of one beam often share a voxel (cfg2: 131k
    // points -> 61k kept, 56k unique)
    Prof p(c, "morton", n_in * 12 + n_in * 8);
    size_t maxf = 0;
    for (int f = 0; f < B; ++f) maxf = std::max<size_t>(maxf, offs[f + 1] - offs[f]);
    k_morton_dedup<<<dim3(cdiv(std::max<size_t>(maxf, 1), MD_TILE), B), MD_T, 0, s>>>(d_xyz, d_offs, B, L, ka, kept,
                                                                                     err);
    launched(c);
  }
  PCC_CUDA(cudaMemcpyAsync(hk, kept, B * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  PCC_CUDA(cudaMemcpyAsync(hk + B, err, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  PCC_CUDA(cudaStreamSynchronize(s));
  if (hk[B] & EF_RANGE) throw Error{PCC_ERR_RANGE};  // out-of-range points are not kept
  // kept offsets (contiguous, what the sort writes) on the host and the device
  h[0] = 0;
  for (int f = 0; f < B; ++f) h[f + 1] = h[f] + hk[f];
  const size_t n = h[B];
  PCC_CUDA(cudaMemcpyAsync(d_noffs, h, (B + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
  const uint64_t* d_in_offs = d_offs;
  d_offs = d_noffs;

  // frame-aligned tiles: tp[f] = first tile of frame f (host copy of the kept offsets)
  uint32_t* htp = reinterpret_cast<uint32_t*>(h + (B + 1));  // inside the pinned block above
  htp[0] = 0;
  for (int f = 0; f < B; ++f) htp[f + 1] = htp[f] + cdiv(h[f + 1] - h[f], RS_TILE);
  const uint32_t ntiles = htp[B];
  uint32_t* d_tp = wsT<uint32_t>(c, "rs_tp", B + 1);
  PCC_CUDA(cudaMemcpyAsync(d_tp, htp, (B + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
  RsTile* tiles = wsT<RsTile>(c, "rs_tiles", ntiles);
  RsTile* tiles_in = wsT<RsTile>(c, "rs_tiles_in", ntiles);
  {
    Prof p(c, "sort", 0);
    k_rs_tiles<<<cdiv(ntiles, 256), 256, 0, s>>>(d_tp, d_offs, B, ntiles, tiles, d_in_offs, tiles_in);
    launched(c);
  }
  // 3L Morton bits in 8- or 9-bit digits, whichever needs fewer passes
  const int bits = 3 * L;
  static const int db_forced = [] {
    const char* e = getenv("PCC_SORT_DB");  // development override (8 or 9)
    return e ? atoi(e) : 0;
  }();
  const int DB = db_forced == 8 || db_forced == 9 ? db_forced : ((bits + 8) / 9 < (bits + 7) / 8 ? 9 : 8);
  uint32_t* hist = wsT<uint32_t>(c, "rs_hist", (size_t(1) << DB) * ntiles + 1);
  for (int sh = 0; sh < bits; sh += DB) {
    {
      Prof p(c, "sort", n * 8);
      const RsTile* tl = sh == 0 ? tiles_in : tiles;
      if (DB == 9) k_rs_hist<9><<<ntiles, RS_T, 0, s>>>(ka, sh, tl, hist);
      else k_rs_hist<8><<<ntiles, RS_T, 0, s>>>(ka, sh, tl, hist);
      launched(c);
    }
    scan_u32(c, hist, hist, (size_t(1) << DB) * ntiles);
    {
      Prof p(c, "sort", n * 16);
      const RsTile* tl = sh == 0 ? tiles_in : tiles;
      if (DB == 9) k_rs_scatter<9><<<ntiles, RS_T, 0, s>>>(ka, kb, sh, tl, hist);
      else k_rs_scatter<8><<<ntiles, RS_T, 0, s>>>(ka, kb, sh, tl, hist);
      launched(c);
    }
    std::swap(ka, kb);
  }
  const uint64_t* sorted = ka;

  const uint32_t nblk = cdiv(n, LV_TILE);
  uint32_t* cnt = wsT<uint32_t>(c, "lv_cnt", size_t(L + 1) * nblk + 1);
  {
    Prof p(c, "octree", n * 8);
    k_lvl_count<<<nblk, LV_T, 0, s>>>(sorted, n, L, cnt, nblk);
    launched(c);
  }
  scan_u32(c, cnt, cnt, size_t(L + 1) * nblk);
  // sizes: total nodes over all depths <= (L+1) n
  uint32_t* small = wsT<uint32_t>(c, "lv_small", (L + 1) + size_t(L + 1) * (B + 1));
  uint32_t* d_counts = small;
  uint32_t* d_foff = wsT<uint32_t>(c, "foff", size_t(L + 2) * (B + 1));
  {
    Prof p(c, "octree", 0);
    k_lvl_totals<<<1, 32, 0, s>>>(cnt, nblk, L, B, d_counts, d_foff);
  }
  launched(c);
  // read totals to size the node arrays (sync #1)
  uint32_t* hc = static_cast<uint32_t*>(pinned(c, (L + 2) * sizeof(uint32_t)));
  PCC_CUDA(cudaMemcpyAsync(hc, d_counts, (L + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  PCC_CUDA(cudaMemcpyAsync(hc + L + 1, err, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  PCC_CUDA(cudaStreamSynchronize(s));
  if (hc[L + 1] & EF_RANGE) throw Error{PCC_ERR_RANGE};
  o.N.assign(hc, hc + L + 1);
  o.nb.assign(L + 2, 0);
  for (int d = 0; d <= L; ++d) o.nb[d + 1] = o.nb[d] + o.N[d];
  const size_t tot = o.nb[L + 1];
  uint64_t* key_all = wsT<uint64_t>(c, "key", tot);
  uint8_t* code_all = wsT<uint8_t>(c, "code", tot + 8);
  uint32_t* cs_all = wsT<uint32_t>(c, "cs", tot);
  uint32_t* par_all = wsT<uint32_t>(c, "par", tot);
  PCC_CUDA(cudaMemsetAsync(code_all, 0, tot + 8, s));
  {
    Prof p(c, "octree", n * 8 + tot * (8 + 1 + 4 + 4));
    k_lvl_scatter<<<nblk, LV_T, 0, s>>>(sorted, n, L, B, cnt, nblk, key_all, code_all, cs_all, par_all, d_foff);
    launched(c);
  }
  // host copy of frame offsets (for rANS segment layout)
  uint32_t* hf = static_cast<uint32_t*>(pinned(c, size_t(L + 1) * (B + 1) * sizeof(uint32_t)));
  PCC_CUDA(cudaMemcpyAsync(hf, d_foff, size_t(L + 1) * (B + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  PCC_CUDA(cudaStreamSynchronize(s));
  o.foff.assign(hf, hf + size_t(L + 1) * (B + 1));
}

uint32_t expand_level(pcc_ctx c, int d, int B, OctreeOut& o, uint32_t max_nodes, const uint32_t* err) {
  cudaStream_t s = c->stream;
  const uint32_t n = o.N[d];
  uint64_t* key_all = static_cast<uint64_t*>(c->bufs.at("key").p);
  uint8_t* code_all = static_cast<uint8_t*>(c->bufs.at("code").p);
  uint32_t* cs_all = static_cast<uint32_t*>(c->bufs.at("cs").p);
  uint32_t* par_all = static_cast<uint32_t*>(c->bufs.at("par").p);
  uint32_t* d_foff = static_cast<uint32_t*>(c->bufs.at("foff").p);
  uint32_t* cs = cs_all + o.nb[d];
  uint32_t* tmp = wsT<uint32_t>(c, "exp_tmp", size_t(n) + 1);
  {
    Prof p(c, "expand", size_t(n) * 5);
    k_popc<<<cdiv(n, 256), 256, 0, s>>>(code_all + o.nb[d], n, tmp);
    launched(c);
  }
  scan_u32(c, tmp, tmp, n);
  PCC_CUDA(cudaMemcpyAsync(cs, tmp, (size_t(n) + 1) * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  // children are written without knowing their count on the host: the node arrays' room
  // bounds the writes (k_expand flags anything beyond it)
  const uint64_t room_keys = c->bufs.at("key").cap / sizeof(uint64_t);
  const uint64_t room_par = c->bufs.at("par").cap / sizeof(uint32_t);
  const uint64_t room = std::min(room_keys, room_par);
  const uint64_t cap = room > o.nb[d + 1] ? room - o.nb[d + 1] : 0;
  uint32_t* eflag = const_cast<uint32_t*>(err);
  {
    Prof pe(c, "expand", size_t(n) * 13);
    k_expand<<<cdiv(n, 256), 256, 0, s>>>(key_all + o.nb[d], code_all + o.nb[d], cs, n, key_all + o.nb[d + 1],
                                          par_all + o.nb[d + 1], cap, eflag);
    launched(c);
  }
  {
    Prof pf(c, "expand", 0);
    k_foff_next<<<cdiv(B + 1, 256), 256, 0, s>>>(cs, d_foff + size_t(d) * (B + 1), B, d_foff + size_t(d + 1) * (B + 1));
    launched(c);
  }
  // ONE readback per level: the child count, the error flags (this level's rANS decode and
  // the expansion), and the per-frame child offsets
  uint32_t* hb = static_cast<uint32_t*>(pinned(c, (B + 3) * sizeof(uint32_t)));
  PCC_CUDA(cudaMemcpyAsync(hb, tmp + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  if (err) PCC_CUDA(cudaMemcpyAsync(hb + 1, err, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  PCC_CUDA(cudaMemcpyAsync(hb + 2, d_foff + size_t(d + 1) * (B + 1), (B + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  PCC_CUDA(cudaStreamSynchronize(s));
  const uint32_t nn = hb[0];
  if ((err && hb[1]) || nn > max_nodes || nn > cap) throw Error{PCC_ERR_CORRUPT};
  o.N.resize(d + 2);
  o.N[d + 1] = nn;
  o.nb.resize(d + 3);
  o.nb[d + 2] = o.nb[d + 1] + nn;
  o.foff.resize(size_t(d + 2) * (B + 1));
  for (int f = 0; f <= B; ++f) o.foff[size_t(d + 1) * (B + 1) + f] = hb[2 + f];
  return nn;
}

void keys_to_xyz(pcc_ctx c, const uint64_t* keys, size_t n, int L, int32_t* xyz) {
  if (!n) return;
  Prof p(c, "expand", n * 20);
  k_keys_to_xyz<<<cdiv(n, 256), 256, 0, c->stream>>>(keys, n, L, xyz);
  launched(c);
}

}  // namespace pcc
