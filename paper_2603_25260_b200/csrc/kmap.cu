// kmap.cu — sparse-conv kernel map via a GPU open-addressing hash table (sparse
// convolution "decomposed into multiple indexed linear transforms"; the kernel map is the
// index list of each transform).  Keys carry the frame id above bit 3d, so neighbours
// never cross frames.  nbr[i][delta] = row of coord(i)+delta, or N (the zero row).
#include <string>

#include "pcc_internal.cuh"

namespace pcc {

namespace {

constexpr uint64_t EMPTY = ~0ull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
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

__global__ void k_hash_insert(const uint64_t* __restrict__ keys, uint32_t n, unsigned long long* __restrict__ tk,
                              uint32_t* __restrict__ tv, uint64_t mask) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = keys[i];
  uint64_t h = mix64(k) & mask;
  while (true) {
    unsigned long long prev = atomicCAS(&tk[h], (unsigned long long)EMPTY, (unsigned long long)k);
    if (prev == EMPTY || prev == k) {
      tv[h] = i;
      return;
    }
    h = (h + 1) & mask;
  }
}

__global__ void k_kmap(const uint64_t* __restrict__ keys, uint32_t n, int depth, const unsigned long long* __restrict__ tk,
                       const uint32_t* __restrict__ tv, uint64_t mask, int32_t* __restrict__ nbr) {
  const size_t t = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= size_t(n) * 27) return;
  const uint32_t i = uint32_t(t / 27), dl = uint32_t(t % 27);
  const uint64_t k = keys[i];
  const int sh = 3 * depth;
  const uint64_t mbits = sh >= 64 ? ~0ull : ((1ull << sh) - 1ull);
  const uint64_t fr = sh >= 64 ? 0ull : (k >> sh) << sh;
  const uint64_t m = k & mbits;
  const int dx = int(dl / 9) - 1, dy = int((dl / 3) % 3) - 1, dz = int(dl % 3) - 1;
  const int64_t lim = int64_t(1) << depth;
  const int64_t X = int64_t(compact3(m >> 2)) + dx, Y = int64_t(compact3(m >> 1)) + dy, Z = int64_t(compact3(m)) + dz;
  int32_t r = int32_t(n);
  if (X >= 0 && Y >= 0 && Z >= 0 && X < lim && Y < lim && Z < lim) {
    const uint64_t q = fr | spread3(uint32_t(X)) << 2 | spread3(uint32_t(Y)) << 1 | spread3(uint32_t(Z));
    uint64_t h = mix64(q) & mask;
    while (true) {
      const unsigned long long s = tk[h];
      if (s == q) {
        r = int32_t(tv[h]);
        break;
      }
      if (s == EMPTY) break;
      h = (h + 1) & mask;
    }
  }
  nbr[t] = r;
}

// Kernel map of depth d derived from the parent level's (no hashing): the neighbour of
// node i at offset delta is a child of the parent's neighbour.  Per axis, with the node's
// child bit b and offset o in {-1, 0, 1}: t = b + o, parent offset floor(t / 2), child bit
// t & 1.  The child exists iff its bit is set in the parent neighbour's code X, and its
// row is cs[p'] + popc(X & ((1 << c') - 1)) (children in ascending child index, Q8).
// Frames never mix: a parent's neighbours are in its own frame.
__global__ void k_kmap_derive(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ par, uint32_t n,
                              const int32_t* __restrict__ pnbr, uint32_t np, const uint8_t* __restrict__ Xp,
                              const uint32_t* __restrict__ csp, int32_t* __restrict__ nbr) {
  const size_t t = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= size_t(n) * 27) return;
  const uint32_t i = uint32_t(t / 27), dl = uint32_t(t % 27);
  const uint32_t c = uint32_t(keys[i] & 7u);
  const int ox = int(dl / 9) - 1, oy = int((dl / 3) % 3) - 1, oz = int(dl % 3) - 1;
  const int tx = int(c >> 2) + ox, ty = int((c >> 1) & 1u) + oy, tz = int(c & 1u) + oz;  // in -1..2
  const int px = (tx + 2) / 2 - 1, py = (ty + 2) / 2 - 1, pz = (tz + 2) / 2 - 1;        // floor(t / 2)
  const uint32_t cc = uint32_t(((tx & 1) << 2) | ((ty & 1) << 1) | (tz & 1));
  const int32_t q = pnbr[size_t(par[i]) * 27 + uint32_t((px + 1) * 9 + (py + 1) * 3 + (pz + 1))];
  int32_t r = int32_t(n);
  if (q != int32_t(np)) {
    const uint32_t x = Xp[q];
    if ((x >> cc) & 1u) r = int32_t(csp[q] + __popc(x & ((1u << cc) - 1u)));
  }
  nbr[t] = r;
}

// The same derivation with one thread per node: a node's 27 neighbours come from only 8
// parent neighbours (per axis, offsets -1/0/+1 of a child with bit b fall into parent
// offsets b-1 and b), so the node loads those 8 parent entries, their codes and child
// starts once (24 loads instead of 81), builds its 27 entries in shared memory and the
// block stores 128 rows coalesced.
__global__ void __launch_bounds__(128) k_kmap_derive8(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ par,
                                                      uint32_t n, const int32_t* __restrict__ pnbr, uint32_t np,
                                                      const uint8_t* __restrict__ Xp, const uint32_t* __restrict__ csp,
                                                      int32_t* __restrict__ nbr) {
  __shared__ int32_t so[128 * 27];
  const uint32_t i0 = blockIdx.x * 128u;
  const uint32_t i = i0 + threadIdx.x;
  if (i < n) {
    const uint32_t c = uint32_t(keys[i] & 7u);
    const int bx = int(c >> 2), by = int((c >> 1) & 1u), bz = int(c & 1u);
    const int32_t* pn = pnbr + size_t(par[i]) * 27;
    int32_t q[8];
    uint32_t qx[8], qc[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) {  // parent neighbour (bx - 1 + sx, by - 1 + sy, bz - 1 + sz)
      const int sx = s >> 2, sy = (s >> 1) & 1, sz = s & 1;
      q[s] = pn[(bx + sx) * 9 + (by + sy) * 3 + (bz + sz)];
    }
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const bool ok = q[s] != int32_t(np);
      qx[s] = ok ? uint32_t(Xp[q[s]]) : 0u;
      qc[s] = ok ? csp[q[s]] : 0u;
    }
#pragma unroll
    for (int dl = 0; dl < 27; ++dl) {
      const int ox = dl / 9 - 1, oy = (dl / 3) % 3 - 1, oz = dl % 3 - 1;
      const int tx = bx + ox, ty = by + oy, tz = bz + oz;  // in -1..2
      // parent offset floor(t / 2) = b - 1 + side, side = (t + 2) / 2 - b
      const int s = (((tx + 2) / 2 - bx) << 2) | (((ty + 2) / 2 - by) << 1) | ((tz + 2) / 2 - bz);
      const uint32_t cc = uint32_t(((tx & 1) << 2) | ((ty & 1) << 1) | (tz & 1));
      uint32_t x = 0, cs0 = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (u == s) {
          x = qx[u];
          cs0 = qc[u];
        }
      so[threadIdx.x * 27 + dl] = ((x >> cc) & 1u) ? int32_t(cs0 + __popc(x & ((1u << cc) - 1u))) : int32_t(n);
    }
  }
  __syncthreads();
  const uint32_t rows = min(128u, n - i0);
  int32_t* dst = nbr + size_t(i0) * 27;
  for (uint32_t k = threadIdx.x; k < rows * 27; k += 128) dst[k] = so[k];
}

// HRCS statistic (Fig.1c; SPEC hrcs_stats S:158-166): per node, the number of
// occupied coordinates among its 26 neighbours at the same depth (exact hash membership).
// Per-frame sums: the frame id sits above bit 3d of the key, and lanes of a warp holding
// the same frame add their counts with one redux + one 64-bit atomic.
__global__ void k_hrcs(const uint64_t* __restrict__ keys, uint32_t n, int depth, const unsigned long long* __restrict__ tk,
                       uint64_t mask, uint32_t frame0, unsigned long long* __restrict__ sum) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = i < n;
  const uint64_t k = live ? keys[i] : 0ull;
  const int sh = 3 * depth;
  const uint64_t fr = sh >= 64 ? 0ull : (k >> sh) << sh;
  const uint64_t m = k & (sh >= 64 ? ~0ull : ((1ull << sh) - 1ull));
  const int64_t lim = int64_t(1) << depth;
  const int64_t X0 = compact3(m >> 2), Y0 = compact3(m >> 1), Z0 = compact3(m);
  uint32_t cnt = 0;
  if (live)
    for (int dl = 0; dl < 27; ++dl) {
      if (dl == 13) continue;  // the node itself
      const int64_t X = X0 + dl / 9 - 1, Y = Y0 + (dl / 3) % 3 - 1, Z = Z0 + dl % 3 - 1;
      if (X < 0 || Y < 0 || Z < 0 || X >= lim || Y >= lim || Z >= lim) continue;
      const uint64_t q = fr | spread3(uint32_t(X)) << 2 | spread3(uint32_t(Y)) << 1 | spread3(uint32_t(Z));
      uint64_t h = mix64(q) & mask;
      while (true) {
        const unsigned long long s = tk[h];
        if (s == q) { ++cnt; break; }
        if (s == EMPTY) break;
        h = (h + 1) & mask;
      }
    }
  const uint32_t f = live ? uint32_t(sh >= 64 ? 0ull : (k >> sh)) : 0xffffffffu;
  const uint32_t grp = __match_any_sync(0xffffffffu, f);
  const uint32_t tot = __reduce_add_sync(grp, cnt);
  if (live && (threadIdx.x & 31) == uint32_t(__ffs(grp) - 1) && tot)
    atomicAdd(&sum[f - frame0], (unsigned long long)tot);
}

}  // namespace

void kernel_map_derive(pcc_ctx c, const uint64_t* keys, const uint32_t* par, uint32_t N, const int32_t* pnbr,
                       uint32_t Np, const uint8_t* Xp, const uint32_t* csp, int32_t* nbr) {
  if (N == 0) return;
  const size_t t = size_t(N) * 27;
  Prof p(c, "kmap", size_t(N) * (8 + 4 + 27 * 4) + size_t(Np) * (27 * 4 + 5));
  static const bool per_pair = [] {
    const char* e = getenv("PCC_KMAP");
    return e && std::string(e) == "derive27";
  }();
  if (per_pair)
    k_kmap_derive<<<unsigned((t + 255) / 256), 256, 0, c->stream>>>(keys, par, N, pnbr, Np, Xp, csp, nbr);
  else
    k_kmap_derive8<<<unsigned((N + 127) / 128), 128, 0, c->stream>>>(keys, par, N, pnbr, Np, Xp, csp, nbr);
  launched(c);
}

void kernel_map(pcc_ctx c, const uint64_t* keys, uint32_t N, int depth, int32_t* nbr) {
  if (N == 0) return;
  uint64_t cap = 1;
  while (cap < 2ull * N) cap <<= 1;
  unsigned long long* tk = wsT<unsigned long long>(c, "hash_k", cap);
  uint32_t* tv = wsT<uint32_t>(c, "hash_v", cap);
  PCC_CUDA(cudaMemsetAsync(tk, 0xff, cap * sizeof(unsigned long long), c->stream));
  {
    Prof p(c, "kmap", size_t(N) * 8 + cap * 12);
    k_hash_insert<<<(N + 255) / 256, 256, 0, c->stream>>>(keys, N, tk, tv, cap - 1);
  }
  size_t t = size_t(N) * 27;
  {
    Prof p(c, "kmap", size_t(N) * (8 + 27 * 4));
    k_kmap<<<unsigned((t + 255) / 256), 256, 0, c->stream>>>(keys, N, depth, tk, tv, cap - 1, nbr);
  }
  launched(c, 2);
}

void hrcs_counts(pcc_ctx c, const uint64_t* keys, uint32_t N, int depth, int B, unsigned long long* d_sum) {
  PCC_CUDA(cudaMemsetAsync(d_sum, 0, size_t(B) * sizeof(unsigned long long), c->stream));
  if (N == 0) return;
  uint64_t cap = 1;
  while (cap < 2ull * N) cap <<= 1;
  unsigned long long* tk = wsT<unsigned long long>(c, "hash_k", cap);
  uint32_t* tv = wsT<uint32_t>(c, "hash_v", cap);
  PCC_CUDA(cudaMemsetAsync(tk, 0xff, cap * sizeof(unsigned long long), c->stream));
  {
    Prof p(c, "hrcs", size_t(N) * 8 + cap * 12);
    k_hash_insert<<<(N + 255) / 256, 256, 0, c->stream>>>(keys, N, tk, tv, cap - 1);
  }
  {
    Prof p(c, "hrcs", size_t(N) * 8);
    k_hrcs<<<(N + 255) / 256, 256, 0, c->stream>>>(keys, N, depth, tk, cap - 1, 0u, d_sum);
  }
  launched(c, 2);
}

}  // namespace pcc
