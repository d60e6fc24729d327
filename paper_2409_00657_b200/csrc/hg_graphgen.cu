// Row-local planted-partition power-law graph generator (device side).
//
// Twin of oracle/graphgen.py; the spec and the integer tables are described
// there.  Four passes so a 1.6B-entry papers100M-shaped CSR is built on the
// GPU in seconds: raw row lengths -> (scan) -> slot draws -> per-row sort +
// unique + self-loop drop -> (scan) -> compaction into canonical CSR
// (graph.py:25-48 invariants: sorted, unique, no self-loops).
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "hg_common.cuh"

namespace hg {

__device__ __forceinline__ int floor_log2_p1(uint64_t r) {  // floor(log2(r+1))
  return 63 - __clzll((long long)(r + 1));
}

__device__ __forceinline__ int block_of(const hg_graph_tables& t, int64_t v) {
  return (int)((v * (int64_t)t.n_blocks) / t.n);
}

__global__ void k_raw_degrees(const hg_graph_tables t, int64_t* raw_deg) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= t.n) return;
  const int b = block_of(t, v);
  const uint64_t nbk = (uint64_t)(t.block_start[b + 1] - t.block_start[b]);
  const uint64_t i = (uint64_t)(v - t.block_start[b]);
  const uint64_t rank = (t.a[b] * i + t.c[b]) % nbk;
  int e = floor_log2_p1(rank);
  if (e > t.n_levels - 1) e = t.n_levels - 1;
  const uint64_t u = mix64((uint64_t)v ^ t.deg_key) >> 32;
  raw_deg[v] = t.deg_lo[e] + (int64_t)((u * (uint64_t)t.deg_span[e]) >> 32);
}

__device__ __forceinline__ int32_t draw_target(const hg_graph_tables& t, int64_t v, int own,
                                               uint64_t rk, uint64_t slot) {
  const uint64_t hA = mix64(rk ^ (2 * slot));
  const uint64_t hB = mix64(rk ^ (2 * slot + 1));
  int tb = own;
  const bool inb = t.in_always || (uint32_t)(hB >> 32) < t.thr_in;
  if (!inb && t.n_blocks > 1)
    tb = (int)((own + 1 + (int64_t)((hB & 0xFFFFFFFFull) % (uint64_t)(t.n_blocks - 1))) %
               t.n_blocks);
  const uint64_t u = hA >> 32;
  int e = 0;
  while (e < t.n_levels - 1 && t.cum[e] <= u) ++e;
  const uint64_t off = ((hA & 0xFFFFFFFFull) * (uint64_t)t.lvl_size[e]) >> 32;
  const uint64_t r = ((1ull << e) - 1) + off;
  const uint64_t nbk = (uint64_t)(t.block_start[tb + 1] - t.block_start[tb]);
  const uint64_t diff = (r + nbk - (t.c[tb] % nbk)) % nbk;
  const uint64_t i = (diff * t.a_inv[tb]) % nbk;
  return (int32_t)(t.block_start[tb] + (int64_t)i);
}

// thread per slot; the row is found by binary search over raw_off[v0..v1]
__global__ void k_fill(const hg_graph_tables t, int64_t v0, int64_t v1,
                       const int64_t* __restrict__ raw_off, int32_t* __restrict__ raw_targets) {
  const int64_t base = raw_off[v0];
  const int64_t total = raw_off[v1] - base;
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= total) return;
  const int64_t g = base + s;
  int64_t lo = v0, hi = v1;  // largest v with raw_off[v] <= g
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (raw_off[mid] <= g) lo = mid; else hi = mid;
  }
  const int64_t v = lo;
  const uint64_t rk = mix64(t.key ^ (uint64_t)v);
  raw_targets[s] = draw_target(t, v, block_of(t, v), rk, (uint64_t)(g - raw_off[v]));
}

// warp per row: in-place unique + self-loop drop of a sorted row
__global__ void k_unique_rows(int64_t v0, int64_t v1, const int64_t* __restrict__ raw_off,
                              int32_t* __restrict__ keys, int64_t* __restrict__ row_len) {
  const int64_t v = v0 + (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (v >= v1) return;
  const int lane = threadIdx.x & 31;
  const int64_t base = raw_off[v0];
  int32_t* row = keys + (raw_off[v] - base);
  const int64_t len = raw_off[v + 1] - raw_off[v];
  int64_t out = 0;
  int32_t prev_last = -1;
  for (int64_t c = 0; c < len; c += 32) {
    const int64_t j = c + lane;
    const int32_t x = j < len ? row[j] : -1;
    int32_t left = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) left = prev_last;
    const bool keep = j < len && x != left && x != (int32_t)v;
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) row[out + __popc(m & ((1u << lane) - 1u))] = x;
    out += __popc(m);
    prev_last = __shfl_sync(0xffffffffu, x, 31);
    if (c + 32 > len) {
      // last partial chunk: the last valid element sits at lane (len-1-c)
      prev_last = __shfl_sync(0xffffffffu, x, (int)(len - 1 - c));
    }
    __syncwarp();
  }
  if (lane == 0) row_len[v - v0] = out;
}

__global__ void k_compact_rows(int64_t v0, int64_t v1, const int64_t* __restrict__ raw_off,
                               const int32_t* __restrict__ raw, const int64_t* __restrict__ offsets,
                               int32_t* __restrict__ targets) {
  const int64_t v = v0 + (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (v >= v1) return;
  const int lane = threadIdx.x & 31;
  const int32_t* src = raw + (raw_off[v] - raw_off[v0]);
  int32_t* dst = targets + offsets[v];
  const int64_t len = offsets[v + 1] - offsets[v];
  for (int64_t j = lane; j < len; j += 32) dst[j] = src[j];
}

struct RelOff {
  const int64_t* p;
  int64_t base;
  __host__ __device__ __forceinline__ int64_t operator()(int64_t i) const { return p[i] - base; }
};

}  // namespace hg

using namespace hg;

extern "C" int hg_graph_raw_degrees(const hg_graph_tables* t, int64_t* raw_deg, void* stream) {
  if (t->n <= 0) return HG_OK;
  if (t->n_levels < 1 || t->n_levels > 64 || t->n_blocks < 1 || t->n_blocks > 64)
    return hg_fail(HG_ECONFIG, "bad graph tables");
  k_raw_degrees<<<(unsigned)((t->n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*t, raw_deg);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_graph_fill(const hg_graph_tables* t, int64_t v0, int64_t v1,
                             const int64_t* raw_off, int32_t* raw_targets, void* stream) {
  // slot count comes from device memory; launch a grid over the host-known upper bound
  int64_t lo = 0, hi = 0;
  cudaStream_t s = (cudaStream_t)stream;
  HG_CUDA_TRY(cudaMemcpyAsync(&lo, raw_off + v0, 8, cudaMemcpyDeviceToHost, s));
  HG_CUDA_TRY(cudaMemcpyAsync(&hi, raw_off + v1, 8, cudaMemcpyDeviceToHost, s));
  HG_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t total = hi - lo;
  if (total <= 0) return HG_OK;
  k_fill<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(*t, v0, v1, raw_off, raw_targets);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_graph_canonicalize(int64_t v0, int64_t v1, const int64_t* raw_off,
                                     int32_t* raw_targets, int64_t* row_len, void* ws,
                                     size_t* ws_bytes, void* stream) {
  // raw_targets holds the slots of rows [v0, v1) starting at index 0; the
  // chunk must stay below 2^31 slots (CUB segmented sort uses int counts).
  cudaStream_t s = (cudaStream_t)stream;
  int64_t lo = 0, hi = 0;
  HG_CUDA_TRY(cudaMemcpyAsync(&lo, raw_off + v0, 8, cudaMemcpyDeviceToHost, s));
  HG_CUDA_TRY(cudaMemcpyAsync(&hi, raw_off + v1, 8, cudaMemcpyDeviceToHost, s));
  HG_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t total = hi - lo;
  const int64_t nseg = v1 - v0;
  if (total >= (1ll << 31) || nseg >= (1ll << 31))
    return hg_fail(HG_ECONFIG, "canonicalize chunk too large (%lld slots)", (long long)total);
  auto beg = thrust::make_transform_iterator(thrust::make_counting_iterator<int64_t>(v0),
                                             RelOff{raw_off, lo});
  auto end = thrust::make_transform_iterator(thrust::make_counting_iterator<int64_t>(v0 + 1),
                                             RelOff{raw_off, lo});
  size_t cub_bytes = 0;
  HG_CUDA_TRY(cub::DeviceSegmentedSort::SortKeys(nullptr, cub_bytes, (const int32_t*)nullptr,
                                                 (int32_t*)nullptr, (int)total, (int)nseg, beg,
                                                 end, s));
  const size_t need = (size_t)total * 4 + 256 + cub_bytes;
  if (ws == nullptr) { *ws_bytes = need; return HG_OK; }
  if (*ws_bytes < need) return hg_fail(HG_ECAPACITY, "canonicalize workspace too small");
  if (nseg == 0 || total == 0) {
    if (nseg) HG_CUDA_TRY(cudaMemsetAsync(row_len, 0, nseg * 8, s));
    return HG_OK;
  }
  int32_t* sorted = (int32_t*)ws;
  void* tmp = (void*)(((uintptr_t)(sorted + total) + 255) & ~(uintptr_t)255);
  HG_CUDA_TRY(cub::DeviceSegmentedSort::SortKeys(tmp, cub_bytes, raw_targets, sorted, (int)total,
                                                 (int)nseg, beg, end, s));
  HG_CUDA_TRY(cudaMemcpyAsync(raw_targets, sorted, (size_t)total * 4, cudaMemcpyDeviceToDevice, s));
  k_unique_rows<<<(unsigned)((nseg + 7) / 8), 256, 0, s>>>(v0, v1, raw_off, raw_targets, row_len);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_graph_compact(int64_t v0, int64_t v1, const int64_t* raw_off,
                                const int32_t* raw_targets, const int64_t* offsets,
                                int32_t* targets, void* stream) {
  const int64_t nseg = v1 - v0;
  if (nseg <= 0) return HG_OK;
  k_compact_rows<<<(unsigned)((nseg + 7) / 8), 256, 0, (cudaStream_t)stream>>>(
      v0, v1, raw_off, raw_targets, offsets, targets);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* ws,
                                     size_t* ws_bytes, void* stream) {
  size_t need = 0;
  HG_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, need, in, out, n, (cudaStream_t)stream));
  if (ws == nullptr) { *ws_bytes = need; return HG_OK; }
  if (*ws_bytes < need) return hg_fail(HG_ECAPACITY, "scan workspace too small");
  if (n == 0) return HG_OK;
  HG_CUDA_TRY(cub::DeviceScan::ExclusiveSum(ws, *ws_bytes, in, out, n, (cudaStream_t)stream));
  return HG_OK;
}
