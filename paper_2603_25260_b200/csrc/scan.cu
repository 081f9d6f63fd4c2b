// scan.cu — device-wide exclusive scan of u32 (3-phase: tile reduce, scan of tile
// sums (recursive), tile scan + offset).  Used for node/child offsets.
#include "pcc_internal.cuh"

namespace pcc {

namespace {

constexpr int SCAN_T = 256;
constexpr int SCAN_V = 4;
constexpr int SCAN_TILE = SCAN_T * SCAN_V;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

__global__ void k_tile_reduce(const uint32_t* __restrict__ in, size_t n, uint32_t* __restrict__ sums) {
  size_t base = size_t(blockIdx.x) * SCAN_TILE;
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_V; ++k) {
    size_t i = base + size_t(k) * SCAN_T + threadIdx.x;
    if (i < n) s += in[i];
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ uint32_t red[SCAN_T / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < SCAN_T / 32; ++w) t += red[w];
    sums[blockIdx.x] = t;
  }
}

// Scan one tile with an added offset (offs may be null).  Each thread owns SCAN_V
// consecutive elements so the tile is scanned in index order.
__global__ void k_tile_scan(const uint32_t* in, size_t n, uint32_t* out, const uint32_t* __restrict__ offs,
                            uint32_t* total_out) {
  __shared__ uint32_t wsum[SCAN_T / 32 + 1];
  size_t base = size_t(blockIdx.x) * SCAN_TILE + size_t(threadIdx.x) * SCAN_V;
  uint32_t v[SCAN_V];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_V; ++k) {
    v[k] = (base + k < n) ? in[base + k] : 0u;
    s += v[k];
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = warp_incl_scan(s);
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    uint32_t x = lane < SCAN_T / 32 ? wsum[lane] : 0u;
    uint32_t xi = warp_incl_scan(x);
    __syncwarp();
    if (lane < SCAN_T / 32) wsum[lane] = xi - x;
    if (lane == SCAN_T / 32 - 1) wsum[SCAN_T / 32] = xi;
  }
  __syncthreads();
  uint32_t run = (offs ? offs[blockIdx.x] : 0u) + wsum[w] + inc - s;
#pragma unroll
  for (int k = 0; k < SCAN_V; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
  if (total_out && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0)
    *total_out = (offs ? offs[blockIdx.x] : 0u) + wsum[SCAN_T / 32];
}

}  // namespace

void scan_u32(pcc_ctx c, const uint32_t* in, uint32_t* out, size_t n) {
  if (n == 0) {
    PCC_CUDA(cudaMemsetAsync(out, 0, sizeof(uint32_t), c->stream));
    return;
  }
  size_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (tiles == 1) {
    Prof p(c, "scan", n * 8);
    k_tile_scan<<<1, SCAN_T, 0, c->stream>>>(in, n, out, nullptr, out + n);
    launched(c);
    return;
  }
  // per-depth-of-recursion scratch
  static const char* names[] = {"scan_l0", "scan_l1", "scan_l2", "scan_l3"};
  static thread_local int depth = 0;
  uint32_t* sums = wsT<uint32_t>(c, names[depth & 3], tiles + 1);
  {
    Prof p(c, "scan", n * 4);
    k_tile_reduce<<<(unsigned)tiles, SCAN_T, 0, c->stream>>>(in, n, sums);
    launched(c);
  }
  ++depth;
  scan_u32(c, sums, sums, tiles);
  --depth;
  Prof p(c, "scan", n * 8);
  k_tile_scan<<<(unsigned)tiles, SCAN_T, 0, c->stream>>>(in, n, out, sums, out + n);
  launched(c);
}

}  // namespace pcc
