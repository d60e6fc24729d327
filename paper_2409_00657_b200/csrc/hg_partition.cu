// Greedy locality partitioner on the GPU (graph.py:273-327,
// partition_greedy_locality): BFS region growing into parts capped at
// ceil((1 + slack) n / S) vertices; a part seeds at the unassigned vertex of
// highest degree (ties: lowest id) and re-seeds whenever its queue runs dry;
// leftovers (none in practice) round-robin.
//
// The reference's assignment order is sequential by definition (queue order,
// neighbours in CSR order, first come first served, the cap cutting inside a
// row), so one warp runs the whole algorithm: every dequeued vertex's row is
// scanned 32 neighbours per step (ballot + prefix: assignment order = CSR
// order, the cap truncates exactly where the reference stops), and the seed
// cursor advances 32 candidates per step.  Work is O(n + m) warp steps, each
// a short dependent chain of loads: ~0.1 s per 100K vertices, minutes at the
// papers shape (an offline step; the Python reference takes hours there).
#include "hg_common.cuh"

namespace hg {

__global__ void __launch_bounds__(32, 1)
k_partition_greedy(const int64_t* __restrict__ offsets, const int32_t* __restrict__ targets,
                   int64_t n, int n_servers, int64_t cap, const int64_t* __restrict__ seed_order,
                   int32_t* __restrict__ home, int32_t* __restrict__ queue) {
  const int lane = threadIdx.x;
  const unsigned full = 0xffffffffu;
  int64_t cursor = 0, assigned = 0;
  for (int part = 0; part < n_servers; ++part) {
    int64_t size = 0, qh = 0, qt = 0;
    while (size < cap && assigned < n) {
      int64_t src;
      if (qh >= qt) {
        // re-seed: first seed_order entry still unassigned
        int64_t found = -1;
        while (cursor < n) {
          const int64_t c = cursor + lane;
          const bool free_ = c < n && home[seed_order[c]] == -1;
          const unsigned b = __ballot_sync(full, free_);
          if (b) { found = cursor + __ffs(b) - 1; break; }
          cursor += 32;
        }
        if (found < 0) { cursor = n; break; }
        cursor = found;
        src = seed_order[found];
        if (lane == 0) { home[src] = part; queue[0] = (int32_t)src; }
        qh = 1;
        qt = 1;
        ++size;
        ++assigned;
      } else {
        src = queue[qh++];
      }
      __syncwarp();
      const int64_t lo = offsets[src], hi = offsets[src + 1];
      for (int64_t j0 = lo; j0 < hi && size < cap; j0 += 32) {
        const int64_t j = j0 + lane;
        const int nb = j < hi ? targets[j] : -1;
        bool take = nb >= 0 && home[nb] == -1;
        // a non-canonical row may repeat an id inside the chunk: first lane wins
        const unsigned same = __match_any_sync(full, nb);
        take = take && (__ffs(same) - 1 == lane);
        const unsigned b = __ballot_sync(full, take);
        const int before = __popc(b & ((1u << lane) - 1u));
        const int64_t room = cap - size;
        if (take && before < room) {
          home[nb] = part;
          queue[qt + before] = nb;
        }
        const int64_t got = min((int64_t)__popc(b), room);
        qt += got;
        size += got;
        assigned += got;
        __syncwarp();
      }
    }
    if (assigned >= n) break;
  }
}

__global__ void k_partition_leftovers(int32_t* home, int64_t n, int n_servers,
                                      const int64_t* __restrict__ rank) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n && home[v] == -1) home[v] = (int32_t)(rank[v] % n_servers);
}

}  // namespace hg

using namespace hg;

extern "C" int hg_partition_greedy(const int64_t* offsets, const int32_t* targets, int64_t n,
                                   int32_t n_servers, int64_t cap, const int64_t* seed_order,
                                   int32_t* home, int32_t* queue, void* stream) {
  if (n_servers < 1) return hg_fail(HG_ERANGE, "n_servers must be >= 1");
  if (cap < 1) return hg_fail(HG_ERANGE, "part capacity must be >= 1");
  if (n >= (1ll << 31)) return hg_fail(HG_ERANGE, "vertex ids must fit int32");
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) return HG_OK;
  HG_CUDA_TRY(cudaMemsetAsync(home, 0xFF, n * sizeof(int32_t), s));
  k_partition_greedy<<<1, 32, 0, s>>>(offsets, targets, n, n_servers, cap, seed_order, home, queue);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_partition_leftovers(int32_t* home, int64_t n, int32_t n_servers,
                                      const int64_t* rank, void* stream) {
  if (n == 0) return HG_OK;
  k_partition_leftovers<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      home, n, n_servers, rank);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}
