// Peer-memory plumbing for the multi-GPU path (one process per GPU).
//
// Feature shards live in plain cudaMalloc allocations so their CUDA IPC
// handles can be exchanged between the processes of one node; every rank
// maps every peer's shard and the layer-1 gather reads remote rows straight
// out of the owner's HBM over NVLink (k_aggregate, peer addressing).  The
// reference's pre-gather byte accounting (featstore.py:226-279: one message
// per (home -> server) with the DEDUPLICATED remote rows of the iteration)
// is kept without a host sync by k_remote_account: a vertex bitmap marks the
// iteration's remote vertices, first-setters count per home.
#include <cstring>

#include "hg_common.cuh"

namespace hg {

__global__ void k_remote_account(const int32_t* __restrict__ ids, const int32_t* __restrict__ n_dev,
                                 int n_host, const int32_t* __restrict__ home, int rank,
                                 uint32_t* __restrict__ bitmap,
                                 unsigned long long* __restrict__ uniq_per_home,
                                 unsigned long long* __restrict__ total_remote) {
  const int n = n_dev ? *n_dev : n_host;
  unsigned long long mine = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int v = ids[i];
    const int h = home[v];
    if (h == rank) continue;
    ++mine;
    const uint32_t bit = 1u << (v & 31);
    const uint32_t old = atomicOr(bitmap + (v >> 5), bit);
    if (!(old & bit)) atomicAdd(uniq_per_home + h, 1ull);
  }
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(total_remote, mine);
}

__global__ void k_remote_clear(const int32_t* __restrict__ ids, const int32_t* __restrict__ n_dev,
                               int n_host, uint32_t* __restrict__ bitmap) {
  const int n = n_dev ? *n_dev : n_host;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int v = ids[i];
    bitmap[v >> 5] = 0u;  // benign races: every writer stores zero
  }
}

// Device-side pre-gathering over NVLink (featstore.py:226-279 as a kernel
// pair): mark = dedup the iteration's remote vertices (bitmap first-setter),
// append them to a staging list and map vertex -> staging row; copy = pull
// their rows from the owners' HBM with wide, deeply pipelined peer loads.
__global__ void k_stage_mark(const int32_t* __restrict__ ids, const int32_t* __restrict__ n_dev,
                             const int32_t* __restrict__ home, int rank,
                             uint32_t* __restrict__ bitmap, int32_t* __restrict__ stage_list,
                             int32_t* __restrict__ stage_row, int32_t* __restrict__ stage_count,
                             int stage_cap, unsigned long long* __restrict__ uniq_per_home,
                             unsigned long long* __restrict__ total_remote, int* err,
                             const int64_t* __restrict__ it_dev, int row_stride) {
  const int n = *n_dev;
  if (uniq_per_home && it_dev) uniq_per_home += *it_dev * row_stride;
  unsigned long long mine = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int v = ids[i];
    const int h = home[v];
    if (h == rank) continue;
    ++mine;
    const uint32_t bit = 1u << (v & 31);
    const uint32_t old = atomicOr(bitmap + (v >> 5), bit);
    if (!(old & bit)) {
      const int slot = atomicAdd(stage_count, 1);
      if (slot < stage_cap) {
        stage_list[slot] = v;
        stage_row[v] = slot;
      } else {
        raise_flag(err, HG_EINVARIANT);
      }
      if (uniq_per_home) atomicAdd(uniq_per_home + h, 1ull);
    }
  }
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if (total_remote && (threadIdx.x & 31) == 0 && mine) atomicAdd(total_remote, mine);
}

// 16 lanes x 16 B per row (256-byte bf16 rows); 8 rows in flight per warp.
__global__ void __launch_bounds__(256)
k_stage_copy(const int32_t* __restrict__ stage_list, const int32_t* __restrict__ stage_count,
             int stage_cap, const int32_t* __restrict__ home, const int32_t* __restrict__ local_row,
             const uint8_t* const* __restrict__ peers, int row_bytes, uint8_t* __restrict__ staging) {
  const int cnt = min(*stage_count, stage_cap);
  const int vec_per_row = row_bytes / 16;
  const int64_t total = (int64_t)cnt * vec_per_row;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x * 4) {
    uint4 buf[4];
    int64_t idx[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      idx[u] = i + (int64_t)u * gridDim.x * blockDim.x;
      if (idx[u] < total) {
        const int slot = (int)(idx[u] / vec_per_row), c = (int)(idx[u] % vec_per_row);
        const int v = stage_list[slot];
        const uint8_t* src = peers[home[v]] + (int64_t)local_row[v] * row_bytes + c * 16;
        buf[u] = *reinterpret_cast<const uint4*>(src);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (idx[u] < total) {
        const int slot = (int)(idx[u] / vec_per_row), c = (int)(idx[u] % vec_per_row);
        *reinterpret_cast<uint4*>(staging + (int64_t)slot * row_bytes + c * 16) = buf[u];
      }
  }
}

}  // namespace hg

using namespace hg;

extern "C" int hg_pregather_peer_at(const int32_t* ids, const int32_t* n_dev, const int32_t* home,
                                    int32_t rank, const int32_t* local_row, const void* peers,
                                    int32_t row_bytes, uint32_t* bitmap, int32_t* stage_list,
                                    int32_t* stage_row, int32_t* stage_count, int32_t stage_cap,
                                    void* staging, unsigned long long* uniq_per_home,
                                    const int64_t* it_dev, int32_t row_stride,
                                    unsigned long long* total_remote, int* err, void* stream) {
  if (row_bytes % 16) return hg_fail(HG_ECONFIG, "row bytes must be a multiple of 16");
  cudaStream_t s = (cudaStream_t)stream;
  HG_CUDA_TRY(cudaMemsetAsync(stage_count, 0, sizeof(int32_t), s));
  count_launch(3);
  k_stage_mark<<<148 * 2, 256, 0, s>>>(ids, n_dev, home, rank, bitmap, stage_list, stage_row,
                                       stage_count, stage_cap, uniq_per_home, total_remote, err,
                                       it_dev, row_stride);
  k_stage_copy<<<148 * 4, 256, 0, s>>>(stage_list, stage_count, stage_cap, home, local_row,
                                       (const uint8_t* const*)peers, row_bytes, (uint8_t*)staging);
  k_remote_clear<<<148 * 2, 256, 0, s>>>(ids, n_dev, 0, bitmap);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_pregather_peer(const int32_t* ids, const int32_t* n_dev, const int32_t* home,
                                 int32_t rank, const int32_t* local_row, const void* peers,
                                 int32_t row_bytes, uint32_t* bitmap, int32_t* stage_list,
                                 int32_t* stage_row, int32_t* stage_count, int32_t stage_cap,
                                 void* staging, unsigned long long* uniq_per_home,
                                 unsigned long long* total_remote, int* err, void* stream) {
  return hg_pregather_peer_at(ids, n_dev, home, rank, local_row, peers, row_bytes, bitmap,
                              stage_list, stage_row, stage_count, stage_cap, staging,
                              uniq_per_home, nullptr, 0, total_remote, err, stream);
}

extern "C" int hg_alloc(size_t bytes, void** out) {
  *out = nullptr;
  HG_CUDA_TRY(cudaMalloc(out, bytes < 256 ? 256 : bytes));
  return HG_OK;
}

extern "C" int hg_free(void* p) {
  if (p) HG_CUDA_TRY(cudaFree(p));
  return HG_OK;
}

extern "C" int hg_ipc_handle(void* p, void* handle_out /* 64 bytes */) {
  cudaIpcMemHandle_t h;
  HG_CUDA_TRY(cudaIpcGetMemHandle(&h, p));
  memcpy(handle_out, &h, sizeof(h));
  return HG_OK;
}

extern "C" int hg_ipc_open(const void* handle /* 64 bytes */, void** out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  HG_CUDA_TRY(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
  return HG_OK;
}

extern "C" int hg_ipc_close(void* p) {
  if (p) HG_CUDA_TRY(cudaIpcCloseMemHandle(p));
  return HG_OK;
}

extern "C" int hg_remote_account(const int32_t* ids, const int32_t* n_dev, int32_t n_host,
                                 const int32_t* home, int32_t rank, uint32_t* bitmap,
                                 unsigned long long* uniq_per_home,
                                 unsigned long long* total_remote, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  count_launch();
  k_remote_account<<<148 * 2, 256, 0, s>>>(ids, n_dev, n_host, home, rank, bitmap, uniq_per_home,
                                           total_remote);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_remote_clear(const int32_t* ids, const int32_t* n_dev, int32_t n_host,
                               uint32_t* bitmap, void* stream) {
  count_launch();
  k_remote_clear<<<148 * 2, 256, 0, (cudaStream_t)stream>>>(ids, n_dev, n_host, bitmap);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}
