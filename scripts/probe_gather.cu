// Diagnostic (not product code): random 256-byte row gather vs table
// footprint, to tell DRAM-bandwidth limits from address-translation limits.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_gather probe_gather.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31);
}
__global__ void k_ids(int* ids, int n, long rows, uint64_t seed) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ids[i] = (int)(mix(seed ^ i) % (uint64_t)rows);
}
// 16 lanes per destination row; each destination sums DEG source rows
template <int DEG>
__global__ void __launch_bounds__(256) k_gsum(const uint4* __restrict__ t, const int* __restrict__ ids,
                                              int n_dst, uint4* __restrict__ out) {
  int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 4, l = threadIdx.x & 15;
  if (g >= n_dst) return;
  uint4 x[DEG];
  int id[DEG];
#pragma unroll
  for (int u = 0; u < DEG; ++u) id[u] = ids[g * DEG + u];
#pragma unroll
  for (int u = 0; u < DEG; ++u) x[u] = __ldg(t + (int64_t)id[u] * 16 + l);
  uint4 a = x[0];
#pragma unroll
  for (int u = 1; u < DEG; ++u) { a.x ^= x[u].x; a.y += x[u].y; a.z ^= x[u].z; a.w += x[u].w; }
  out[(int64_t)g * 16 + l] = a;
}
__global__ void k_flush(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = make_uint4(i, 0, 0, 0);
}

int main(int argc, char** argv) {
  const int n_dst = argc > 1 ? atoi(argv[1]) : 10500, DEG = 10, n = n_dst * DEG;
  double gbs[] = {28};
  uint4* flush; size_t fl = (size_t)512 << 20; cudaMalloc(&flush, fl);
  int* ids; cudaMalloc(&ids, n * 4);
  uint4* out; cudaMalloc(&out, (size_t)n_dst * 256);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (double gb : gbs) {
    long rows = (long)(gb * (1l << 30) / 256);
    uint4* t;
    if (cudaMalloc(&t, (size_t)rows * 256) != cudaSuccess) { printf("alloc fail %.2f\n", gb); break; }
    cudaMemset(t, 1, (size_t)rows * 256);
    for (int sorted = 0; sorted < 2; ++sorted) {
      std::vector<float> ts;
      for (int it = 0; it < 25; ++it) {
        k_ids<<<(n + 255) / 256, 256>>>(ids, n, rows, it * 7919ull + 1);
        if (sorted) {
          std::vector<int> h(n); cudaMemcpy(h.data(), ids, n * 4, cudaMemcpyDeviceToHost);
          std::sort(h.begin(), h.end()); cudaMemcpy(ids, h.data(), n * 4, cudaMemcpyHostToDevice);
        }
        k_flush<<<148 * 8, 256>>>(flush, fl / 16);
        cudaEventRecord(e0);
        k_gsum<DEG><<<(n_dst * 16 + 255) / 256, 256>>>(t, ids, n_dst, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (it >= 5) ts.push_back(ms * 1000);
      }
      std::sort(ts.begin(), ts.end());
      float us = ts[ts.size() / 2];
      double bytes = (double)n * 256 + n_dst * 256.0 + n * 4.0;
      printf("%6.2f GB %s %7.2f us %8.1f GB/s\n", gb, sorted ? "sorted" : "random", us, bytes / us / 1e3);
    }
    cudaFree(t);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
