// Shared device helpers for libhopgnn (sm_100a).
//
// splitmix64 hashing restates gnnsim rng.py:21-42 / _kernels_nb.py:13-18 so
// every keyed decision (neighbour draws, features, labels, permutations,
// weight init) is bit-identical to the reference.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/hopgnn.h"

namespace hg {

constexpr uint64_t kInc = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kM1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kM2 = 0x94D049BB133111EBull;
constexpr uint64_t kHi32 = 0xFFFFFFFF00000000ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  uint64_t z = x + kInc;
  z = (z ^ (z >> 30)) * kM1;
  z = (z ^ (z >> 27)) * kM2;
  return z ^ (z >> 31);
}

// chain(a, b) == mix64(mix64(0 ^ a) ^ b); extend an already-folded state.
__host__ __device__ __forceinline__ uint64_t extend(uint64_t state, uint64_t w) {
  return mix64(state ^ w);
}

// float32 feature value of (row key, column), _kernels_nb.py:109-118.
__host__ __device__ __forceinline__ float feature_value(uint64_t row_key, uint32_t col) {
  uint64_t h = mix64(row_key ^ (uint64_t)col);
  double u = (double)(h >> 40) * (1.0 / 16777216.0);
  return (float)(u - 0.5);
}

// 53-bit uniform on [0,1), rng.py:69-71.
__host__ __device__ __forceinline__ double unit_f64(uint64_t h) {
  return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Device-side error flag: kernels that detect an invariant violation write a
// code here; the C-ABI wrapper checks it when the caller syncs.
__device__ __forceinline__ void raise_flag(int* flag, int code) {
  if (flag) atomicCAS(flag, 0, code);
}

template <typename T>
__device__ __forceinline__ int lower_bound(const T* a, int n, T x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Block-wide exclusive scan of one int per thread (blockDim multiple of 32,
// <= 1024).  `scratch` needs 33 ints.  Returns the exclusive prefix; *total
// receives the block sum.
__device__ __forceinline__ int block_exclusive_scan(int v, int* scratch, int* total) {
  const int lane = lane_id(), w = warp_id(), nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = lane < nw ? scratch[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) scratch[lane] = s;
    if (lane == nw - 1) scratch[32] = s;
  }
  __syncthreads();
  int base = w ? scratch[w - 1] : 0;
  int tot = scratch[32];
  __syncthreads();
  if (total) *total = tot;
  return base + x - v;
}

// Launch accounting + optional CUDA-event timing of selected kernel sites
// (bench.py reads them through hg_prof_read / hg_launch_count).
enum ProfSite { PROF_BUILD = 0, PROF_AGG1 = 1, PROF_GEMM1 = 2, PROF_DW1 = 3, PROF_STEP = 4,
                PROF_AGG2 = 5, PROF_SGD = 6, PROF_PG_MARK = 7, PROF_PG_COPY = 8,
                PROF_PG_CLEAR = 9, PROF_NSITES = 12 };
void count_launch(int n = 1);
void prof_begin(int site, cudaStream_t s);
void prof_end(int site, cudaStream_t s);

// Programmatic dependent launch (PDL).  The training chain is ~13 small
// kernels whose launch + CTA setup would otherwise sit between every pair:
// each chain kernel is launched with programmatic stream serialization (also
// recorded as programmatic edges under graph capture), signals its dependent
// at entry (pdl_trigger: the next grid may be scheduled once every CTA of
// this one is resident) and calls pdl_wait() -- which returns when the
// predecessor grid has completed and its writes are visible -- before it
// reads anything a predecessor wrote.  Both are no-ops without the launch
// attribute.  HG_PDL=0 disables the attribute (A/B switch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace hg

#define HG_CUDA_TRY(expr)                                              \
  do {                                                                 \
    cudaError_t _e = (expr);                                           \
    if (_e != cudaSuccess) return hg_fail_cuda(_e, #expr, __FILE__, __LINE__); \
  } while (0)

int hg_fail_cuda(cudaError_t e, const char* what, const char* file, int line);
int hg_fail(int code, const char* fmt, ...);
