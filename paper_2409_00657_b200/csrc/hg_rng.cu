// Counter-RNG products: feature rows, feature tables, epoch permutation,
// Glorot weights.  All bit-identical to the reference generators:
//   feature_rows  _kernels_nb.py:109-118 (f32 = (mix64(mix64(s^v)^j)>>40)*2^-24-0.5)
//   permutation   engine.py:273-275 / rng.py:74-81 (stable argsort of keyed hashes)
//   glorot        model.py:87-90
#include <cuda_bf16.h>

#include <cub/device/device_radix_sort.cuh>

#include "hg_common.cuh"

namespace hg {

__global__ void k_feature_rows(const int64_t* __restrict__ ids, int64_t n, int dim,
                               uint64_t state, float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = n * dim;
  if (i >= total) return;
  const int64_t row = i / dim;
  const int col = (int)(i - row * dim);
  out[i] = feature_value(mix64(state ^ (uint64_t)ids[row]), col);
}

// One warp per row; 8-column chunks so each lane writes 16 B (bf16) / 32 B (f32).
template <typename T>
__global__ void k_feature_table(const int64_t* __restrict__ ids, int64_t first, int64_t count,
                                int dim, int ld, uint64_t state, T* __restrict__ out) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= count) return;
  const int64_t v = ids ? ids[row] : first + row;
  const uint64_t rk = mix64(state ^ (uint64_t)v);
  T* dst = out + row * (int64_t)ld;
  for (int col = (threadIdx.x & 31); col < ld; col += 32) {
    const float v = col < dim ? feature_value(rk, col) : 0.0f;
    if constexpr (sizeof(T) == 4) dst[col] = v;
    else dst[col] = __float2bfloat16_rn(v);
  }
}

__global__ void k_perm_keys(int64_t n, uint64_t state, uint64_t* keys, int64_t* idx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = mix64(state ^ (uint64_t)i);
  idx[i] = i;
}

template <typename T>
__global__ void k_glorot(int rows, int cols, uint64_t state, T* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)rows * cols;
  if (i >= total) return;
  const double a = sqrt(6.0 / (double)(rows + cols));
  const double u = unit_f64(mix64(state ^ (uint64_t)i));
  out[i] = (T)((u * 2.0 - 1.0) * a);
}

}  // namespace hg

using namespace hg;

extern "C" int hg_feature_rows(const int64_t* ids, int64_t n, int32_t dim, uint64_t state,
                               float* out, void* stream) {
  if (dim < 1) return hg_fail(HG_ERANGE, "dim must be >= 1");
  const int64_t total = n * dim;
  if (total == 0) return HG_OK;
  k_feature_rows<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(ids, n, dim,
                                                                                   state, out);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_feature_table(const int64_t* ids, int64_t first, int64_t count, int32_t dim,
                                int32_t ld, uint64_t state, int32_t dtype, void* out,
                                void* stream) {
  if (dim < 1 || ld < dim) return hg_fail(HG_ERANGE, "need 1 <= dim <= ld");
  if (count == 0) return HG_OK;
  const unsigned grid = (unsigned)((count + 7) / 8);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == 0)
    k_feature_table<float><<<grid, 256, 0, s>>>(ids, first, count, dim, ld, state, (float*)out);
  else if (dtype == 1)
    k_feature_table<__nv_bfloat16><<<grid, 256, 0, s>>>(ids, first, count, dim, ld, state,
                                                       (__nv_bfloat16*)out);
  else
    return hg_fail(HG_ECONFIG, "dtype must be 0 (f32) or 1 (bf16)");
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_epoch_permutation(int64_t n, uint64_t state, int64_t* perm_out, void* ws,
                                    size_t* ws_bytes, void* stream) {
  // ws layout: keys_in[n] u64 | keys_out[n] u64 | idx_in[n] i64 | cub temp
  size_t cub_bytes = 0;
  HG_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (uint64_t*)nullptr,
                                              (uint64_t*)nullptr, (int64_t*)nullptr,
                                              (int64_t*)nullptr, n));
  const size_t need = 3 * (size_t)n * 8 + cub_bytes + 256;
  if (ws == nullptr) { *ws_bytes = need; return HG_OK; }
  if (*ws_bytes < need) return hg_fail(HG_ECAPACITY, "epoch permutation workspace too small");
  if (n == 0) return HG_OK;
  char* p = (char*)ws;
  uint64_t* kin = (uint64_t*)p;
  uint64_t* kout = kin + n;
  int64_t* iin = (int64_t*)(kout + n);
  void* tmp = (void*)(((uintptr_t)(iin + n) + 255) & ~(uintptr_t)255);
  cudaStream_t s = (cudaStream_t)stream;
  k_perm_keys<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, state, kin, iin);
  HG_CUDA_TRY(cudaGetLastError());
  // LSD radix sort is stable: equal keys keep index order == np.argsort(kind="stable")
  HG_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, cub_bytes, kin, kout, iin, perm_out, n, 0, 64, s));
  return HG_OK;
}

__global__ void k_iter_stage(const int64_t* __restrict__ perm, const uint64_t* __restrict__ states,
                             int64_t iters, int64_t* it_dev, int batch, int n_batches, int ahead,
                             int advance, int64_t* __restrict__ roots_out,
                             uint64_t* __restrict__ key_out) {
  const int64_t it0 = *it_dev + ahead;
  // iterations it0 .. it0 + n_batches - 1 (those inside the epoch); their roots
  // are contiguous in the permutation
  const int64_t nb = min((int64_t)n_batches, iters - it0);
  if (nb > 0) {
    if (roots_out)
      for (int64_t i = threadIdx.x; i < nb * batch; i += blockDim.x)
        roots_out[i] = perm[it0 * batch + i];
    if (threadIdx.x < nb) key_out[threadIdx.x] = states[it0 + threadIdx.x];
  }
  __syncthreads();  // every thread has read *it_dev before it moves
  if (threadIdx.x == 0 && advance) *it_dev += advance;
}

extern "C" int hg_iter_stage(const int64_t* perm, const uint64_t* states, int64_t iters,
                             int64_t* it_dev, int32_t batch, int32_t ahead, int32_t advance,
                             int64_t* roots_out, uint64_t* key_out, void* stream) {
  return hg_iter_stage_group(perm, states, iters, it_dev, batch, 1, ahead, advance, roots_out,
                             key_out, stream);
}

extern "C" int hg_iter_stage_group(const int64_t* perm, const uint64_t* states, int64_t iters,
                                   int64_t* it_dev, int32_t batch, int32_t n_batches,
                                   int32_t ahead, int32_t advance, int64_t* roots_out,
                                   uint64_t* key_out, void* stream) {
  if (batch < 0) return hg_fail(HG_ERANGE, "bad batch");
  if (n_batches < 1 || n_batches > 1024) return hg_fail(HG_ERANGE, "bad batch count");
  count_launch();
  k_iter_stage<<<1, 1024, 0, (cudaStream_t)stream>>>(perm, states, iters, it_dev, batch, n_batches,
                                                      ahead, advance, roots_out, key_out);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

__global__ void k_iter_stage_ranged(const int64_t* __restrict__ roots,
                                    const int64_t* __restrict__ ranges,
                                    const uint64_t* __restrict__ states, int64_t iters,
                                    int64_t* it_dev, int cap, int ahead, int advance,
                                    int64_t* __restrict__ roots_out, int32_t* n_out,
                                    uint64_t* __restrict__ key_out) {
  const int64_t it = *it_dev + ahead;
  if (it < iters) {
    const int64_t lo = ranges[2 * it];
    const int n = (int)min((int64_t)cap, ranges[2 * it + 1] - lo);
    for (int i = threadIdx.x; i < n; i += blockDim.x) roots_out[i] = roots[lo + i];
    if (threadIdx.x == 0) {
      *n_out = n;
      key_out[0] = states[it];
    }
  } else if (threadIdx.x == 0) {
    *n_out = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0 && advance) *it_dev += advance;
}

extern "C" int hg_iter_stage_ranged(const int64_t* roots, const int64_t* ranges,
                                    const uint64_t* states, int64_t iters, int64_t* it_dev,
                                    int32_t cap, int32_t ahead, int32_t advance,
                                    int64_t* roots_out, int32_t* n_out, uint64_t* key_out,
                                    void* stream) {
  if (cap < 0) return hg_fail(HG_ERANGE, "bad capacity");
  count_launch();
  k_iter_stage_ranged<<<1, 1024, 0, (cudaStream_t)stream>>>(roots, ranges, states, iters, it_dev,
                                                             cap, ahead, advance, roots_out,
                                                             n_out, key_out);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

// Throughput ceiling of the sampler's hash (the "integer-ALU roofline" of
// k_mg_build): every thread runs `per_thread` dependent-free
// mix64 evaluations (4 independent chains) and folds them into a sink.
__global__ void k_mix64_peak(int64_t per_thread, uint64_t* sink) {
  uint64_t a = threadIdx.x, b = blockIdx.x, c = a ^ 0x1234, d = b ^ 0x9876;
  for (int64_t i = 0; i < per_thread; i += 4) {
    a = mix64(a ^ (uint64_t)i);
    b = mix64(b ^ (uint64_t)i);
    c = mix64(c ^ (uint64_t)i);
    d = mix64(d ^ (uint64_t)i);
  }
  if ((a ^ b ^ c ^ d) == 0x5eed) sink[0] = a;  // keeps the chains live
}

extern "C" int hg_bench_mix64(int32_t blocks, int64_t per_thread, uint64_t* sink, void* stream) {
  count_launch();
  k_mix64_peak<<<blocks, 256, 0, (cudaStream_t)stream>>>(per_thread, sink);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_glorot(int32_t rows, int32_t cols, uint64_t state, int32_t dtype, void* out,
                         void* stream) {
  const int64_t total = (int64_t)rows * cols;
  if (total <= 0) return HG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned grid = (unsigned)((total + 255) / 256);
  if (dtype == 0) k_glorot<double><<<grid, 256, 0, s>>>(rows, cols, state, (double*)out);
  else k_glorot<float><<<grid, 256, 0, s>>>(rows, cols, state, (float*)out);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}
