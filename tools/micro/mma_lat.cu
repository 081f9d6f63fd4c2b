// Microbenchmark: tcgen05.mma kind::i8 issue/complete latency with the canonical
// no-swizzle K-major layout used by the library (tc.cuh).
#include <cstdio>
#include <cstdint>
#include "../../paper_2603_25260_b200/csrc/tc.cuh"
using namespace pcc;

template <int N>
__global__ void k(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;           // 4 KB
  uint8_t* sB = sm + 4096;    // N*32 B
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + 4096 + N * 32);
  uint32_t* th = reinterpret_cast<uint32_t*>(mbar + 1);
  for (int i = threadIdx.x; i < (4096 + N * 32) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (threadIdx.x < 32) tc::tmem_alloc<256>(th);
  if (threadIdx.x == 0) tc::mbar_init(mbar, 1);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  uint32_t tm = *th;
  uint32_t ph = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x == 0) {
      tc::mma_i8(tm, tc::sdesc(tc::smem_u32(sA)), tc::sdesc(tc::smem_u32(sB)), tc::idesc_i8(128, N), it > 0);
      tc::commit(mbar);
    }
    tc::mbar_wait(mbar, ph);
    ph ^= 1;
  }
  long long t1 = clock64();
  // back-to-back issue, single commit
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it)
      tc::mma_i8(tm, tc::sdesc(tc::smem_u32(sA)), tc::sdesc(tc::smem_u32(sB)), tc::idesc_i8(128, N), 1);
    tc::commit(mbar);
  }
  tc::mbar_wait(mbar, ph);
  long long t2 = clock64();
  // fence + barrier cost
  for (int it = 0; it < iters; ++it) {
    tc::fence_async_smem();
    __syncthreads();
  }
  long long t3 = clock64();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<256>(tm);
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; }
}

int main() {
  long long* d; cudaMalloc(&d, 64);
  long long h[3];
  int iters = 1000;
  cudaFuncSetAttribute(k<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  cudaFuncSetAttribute(k<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  k<32><<<1, 128, 16384>>>(iters, d);
  cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  printf("N=32 : commit-wait per MMA %.1f cyc, back-to-back %.1f cyc/MMA, fence+bar %.1f cyc  (%s)\n", h[0] / double(iters), h[1] / double(iters), h[2] / double(iters), cudaGetErrorString(cudaGetLastError()));
  k<256><<<1, 128, 16384>>>(iters, d);
  cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  printf("N=256: commit-wait per MMA %.1f cyc, back-to-back %.1f cyc/MMA, fence+bar %.1f cyc  (%s)\n", h[0] / double(iters), h[1] / double(iters), h[2] / double(iters), cudaGetErrorString(cudaGetLastError()));
  return 0;
}
