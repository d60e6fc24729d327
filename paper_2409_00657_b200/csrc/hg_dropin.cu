// The rest of the reference operator layer (gnnsim.kernels, kernels.py:31-34)
// on the GPU: pick_k_smallest (the layer-wise sampler's shared draw) and
// sbm_edges (the SBM generator's pair pass).  Both bit-identical to
// _kernels_nb.py / _kernels_np.py:
//   pick_k_smallest  _kernels_nb.py:92-106: key_i = (mix64(state ^ ids[i]) & HI32) | i,
//                    the k smallest keys, returned in index order;
//   sbm_edges        _kernels_nb.py:22-52: every pair u < v once, hash
//                    h = mix64(mix64(state ^ u) ^ v), same-block pairs accepted by
//                    (mode_in, thr_in), others by (mode_out, thr_out); mode 0 never,
//                    1 iff h < thr, 2 always; (u, v) in lexicographic order.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "hg_common.cuh"

namespace hg {

__global__ void k_pick_keys(const int64_t* __restrict__ ids, int64_t n, uint64_t state,
                            uint64_t* __restrict__ keys, uint8_t* __restrict__ flags) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = (mix64(state ^ (uint64_t)ids[i]) & kHi32) | (uint64_t)i;
  flags[i] = 0;
}

__global__ void k_pick_mark(const uint64_t* __restrict__ sorted, int64_t k, uint8_t* flags) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) flags[sorted[i] & 0xFFFFFFFFull] = 1;
}

__device__ __forceinline__ bool sbm_accept(uint64_t h, bool same, int mode_in, uint64_t thr_in,
                                           int mode_out, uint64_t thr_out) {
  const int mode = same ? mode_in : mode_out;
  const uint64_t thr = same ? thr_in : thr_out;
  return mode == 2 || (mode == 1 && h < thr);
}

// count pass: one CTA per u (grid-stride), accepted v > u
__global__ void __launch_bounds__(256)
k_sbm_count(const int64_t* __restrict__ block_of, int64_t n, int mode_in, uint64_t thr_in,
            int mode_out, uint64_t thr_out, uint64_t state, int64_t* __restrict__ counts) {
  __shared__ int64_t red[8];
  for (int64_t u = blockIdx.x; u < n; u += gridDim.x) {
    const uint64_t hu = mix64(state ^ (uint64_t)u);
    const int64_t bu = block_of[u];
    int64_t c = 0;
    for (int64_t v = u + 1 + threadIdx.x; v < n; v += blockDim.x)
      c += sbm_accept(mix64(hu ^ (uint64_t)v), block_of[v] == bu, mode_in, thr_in, mode_out,
                      thr_out);
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane_id() == 0) red[warp_id()] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      counts[u] = t;
    }
    __syncthreads();
  }
}

// fill pass: one CTA per u, v in ascending order (ordered compaction per chunk)
__global__ void __launch_bounds__(256)
k_sbm_fill(const int64_t* __restrict__ block_of, int64_t n, int mode_in, uint64_t thr_in,
           int mode_out, uint64_t thr_out, uint64_t state, const int64_t* __restrict__ pos,
           int64_t* __restrict__ us, int64_t* __restrict__ vs) {
  __shared__ int scan[40];
  for (int64_t u = blockIdx.x; u < n; u += gridDim.x) {
    const uint64_t hu = mix64(state ^ (uint64_t)u);
    const int64_t bu = block_of[u];
    int64_t base = pos[u];
    for (int64_t v0 = u + 1; v0 < n; v0 += blockDim.x) {
      const int64_t v = v0 + threadIdx.x;
      const int ok = v < n && sbm_accept(mix64(hu ^ (uint64_t)v), block_of[v] == bu, mode_in,
                                         thr_in, mode_out, thr_out);
      int total;
      const int at = block_exclusive_scan(ok, scan, &total);
      if (ok) {
        us[base + at] = u;
        vs[base + at] = v;
      }
      base += total;
    }
  }
}

}  // namespace hg

using namespace hg;

extern "C" int hg_pick_k_smallest(const int64_t* ids, int64_t n, int64_t k, uint64_t state,
                                  int64_t* out, void* stream) {
  if (k < 0) return hg_fail(HG_ERANGE, "k must be >= 0");
  if (n >= (1ll << 32)) return hg_fail(HG_ERANGE, "pick_k_smallest: n must be < 2^32");
  cudaStream_t s = (cudaStream_t)stream;
  if (k >= n) {
    if (n) HG_CUDA_TRY(cudaMemcpyAsync(out, ids, n * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    return HG_OK;
  }
  if (k == 0) return HG_OK;
  uint64_t *keys = nullptr, *sorted = nullptr;
  uint8_t* flags = nullptr;
  int64_t* n_sel = nullptr;
  void* tmp = nullptr;
  size_t sort_bytes = 0, sel_bytes = 0;
  HG_CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, keys, sorted, n, 0, 64, s));
  HG_CUDA_TRY(cub::DeviceSelect::Flagged(nullptr, sel_bytes, ids, flags, out, n_sel, n, s));
  const size_t tmp_bytes = sort_bytes > sel_bytes ? sort_bytes : sel_bytes;
  HG_CUDA_TRY(cudaMallocAsync((void**)&keys, 2 * n * sizeof(uint64_t) + n + 16 + tmp_bytes, s));
  sorted = keys + n;
  n_sel = (int64_t*)(sorted + n);
  flags = (uint8_t*)(n_sel + 2);
  tmp = flags + ((n + 15) / 16) * 16;
  const unsigned g = (unsigned)((n + 255) / 256);
  k_pick_keys<<<g, 256, 0, s>>>(ids, n, state, keys, flags);
  HG_CUDA_TRY(cudaGetLastError());
  size_t b = sort_bytes;
  HG_CUDA_TRY(cub::DeviceRadixSort::SortKeys(tmp, b, keys, sorted, n, 0, 64, s));
  k_pick_mark<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(sorted, k, flags);
  HG_CUDA_TRY(cudaGetLastError());
  b = sel_bytes;
  HG_CUDA_TRY(cub::DeviceSelect::Flagged(tmp, b, ids, flags, out, n_sel, n, s));
  HG_CUDA_TRY(cudaFreeAsync(keys, s));
  return HG_OK;
}

extern "C" int hg_sbm_edges(const int64_t* block_of, int64_t n, int32_t mode_in, uint64_t thr_in,
                            int32_t mode_out, uint64_t thr_out, uint64_t state, int64_t* us,
                            int64_t* vs, int64_t cap, int64_t* count_host, void* stream) {
  if (n < 0) return hg_fail(HG_ERANGE, "n must be >= 0");
  if (mode_in < 0 || mode_in > 2 || mode_out < 0 || mode_out > 2)
    return hg_fail(HG_ERANGE, "modes must be 0, 1 or 2");
  cudaStream_t s = (cudaStream_t)stream;
  *count_host = 0;
  if (n < 2) return HG_OK;
  int64_t* counts = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  HG_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, counts, n, s));
  HG_CUDA_TRY(cudaMallocAsync((void**)&counts, 2 * (n + 1) * sizeof(int64_t) + tmp_bytes, s));
  int64_t* pos = counts + (n + 1);
  tmp = pos + (n + 1);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)(n < (int64_t)nsm * 16 ? n : (int64_t)nsm * 16);
  k_sbm_count<<<grid, 256, 0, s>>>(block_of, n, mode_in, thr_in, mode_out, thr_out, state, counts);
  HG_CUDA_TRY(cudaGetLastError());
  HG_CUDA_TRY(cudaMemsetAsync(counts + n, 0, sizeof(int64_t), s));
  size_t b = tmp_bytes;
  HG_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, b, counts, pos, n + 1, s));
  int64_t total = 0;
  HG_CUDA_TRY(cudaMemcpyAsync(&total, pos + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  HG_CUDA_TRY(cudaStreamSynchronize(s));
  *count_host = total;
  int rc = HG_OK;
  if (us && vs) {
    if (total > cap) {
      rc = hg_fail(HG_ECAPACITY, "sbm_edges: %lld edges > capacity %lld", (long long)total,
                   (long long)cap);
    } else {
      k_sbm_fill<<<grid, 256, 0, s>>>(block_of, n, mode_in, thr_in, mode_out, thr_out, state, pos,
                                      us, vs);
      HG_CUDA_TRY(cudaGetLastError());
    }
  }
  HG_CUDA_TRY(cudaFreeAsync(counts, s));
  return rc;
}
