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

#include <algorithm>

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

// The same, charged to row (*it_dev + ahead) of an [iters x row_stride] table
// (fixed arguments for graph capture).
__global__ void k_remote_account_at(const int32_t* __restrict__ ids,
                                    const int32_t* __restrict__ n_dev,
                                    const int32_t* __restrict__ home, int rank,
                                    uint32_t* __restrict__ bitmap,
                                    unsigned long long* __restrict__ table,
                                    const int64_t* __restrict__ it_dev, int ahead, int row_stride,
                                    unsigned long long* __restrict__ total_remote) {
  const int n = *n_dev;
  unsigned long long* uniq_per_home = table + (*it_dev + ahead) * row_stride;
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
  if (total_remote && (threadIdx.x & 31) == 0 && mine) atomicAdd(total_remote, mine);
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
                             const int32_t* __restrict__ home, int rank, int n_homes,
                             uint32_t* __restrict__ bitmap, int32_t* __restrict__ stage_list,
                             int32_t* __restrict__ stage_row, int32_t* __restrict__ stage_count,
                             int stage_cap, unsigned long long* __restrict__ uniq_per_home,
                             unsigned long long* __restrict__ total_remote, int* err,
                             const int64_t* __restrict__ it_dev, int row_stride) {
  const int n = *n_dev;
  if (uniq_per_home && it_dev) uniq_per_home += *it_dev * row_stride;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  unsigned long long mine = 0;
  // warp-uniform trip count: the counters below are warp-aggregated (one
  // atomic per warp instead of one per new remote row on a single address)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    int v = 0, h = rank;
    if (i < n) {
      v = ids[i];
      h = home[v];
    }
    const bool remote = h != rank;
    bool fresh = false;
    if (remote) {
      ++mine;
      const uint32_t bit = 1u << (v & 31);
      fresh = !(atomicOr(bitmap + (v >> 5), bit) & bit);
    }
    const unsigned m = __ballot_sync(0xffffffffu, fresh);
    if (!m) continue;
    int slot0 = 0;
    if (lane == 0) slot0 = atomicAdd(stage_count, __popc(m));
    slot0 = __shfl_sync(0xffffffffu, slot0, 0);
    if (fresh) {
      const int slot = slot0 + __popc(m & lt);
      if (slot < stage_cap) {
        stage_list[slot] = v;
        stage_row[v] = slot;
      } else {
        raise_flag(err, HG_EINVARIANT);
      }
    }
    if (uniq_per_home) {
      for (int q = 0; q < n_homes; ++q) {
        const unsigned mq = __ballot_sync(0xffffffffu, fresh && h == q);
        if (lane == 0 && mq) atomicAdd(uniq_per_home + q, (unsigned long long)__popc(mq));
      }
    }
  }
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if (total_remote && lane == 0 && mine) atomicAdd(total_remote, mine);
}

// Push-path variant of k_stage_mark: dedup by generation stamps instead of a
// bitmap (stamp[v] = tag of the last pre-gather that listed v), so no clearing
// pass is needed afterwards.  tag = the sequence number this call will publish.
__global__ void k_stage_mark_stamp(const int32_t* __restrict__ ids, const int32_t* __restrict__ n_dev,
                                   const int32_t* __restrict__ home, int rank, int n_homes,
                                   int32_t* __restrict__ stamp, const int64_t* __restrict__ seq,
                                   int32_t* __restrict__ stage_list, int32_t* __restrict__ stage_row,
                                   int32_t* __restrict__ stage_count, int stage_cap,
                                   unsigned long long* __restrict__ uniq_per_home,
                                   unsigned long long* __restrict__ total_remote, int* err,
                                   const int64_t* __restrict__ it_dev, int row_stride) {
  const int n = *n_dev;
  int32_t tag = (int32_t)((*seq + 1) & 0x7fffffff);  // unique per call until 2^31 calls
  if (tag == 0) tag = 1;
  if (uniq_per_home && it_dev) uniq_per_home += *it_dev * row_stride;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  unsigned long long mine = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    int v = 0, h = rank;
    if (i < n) {
      v = ids[i];
      h = home[v];
    }
    const bool remote = h != rank;
    bool fresh = false;
    if (remote) {
      ++mine;
      fresh = atomicExch(stamp + v, tag) != tag;
    }
    const unsigned m = __ballot_sync(0xffffffffu, fresh);
    if (!m) continue;
    int slot0 = 0;
    if (lane == 0) slot0 = atomicAdd(stage_count, __popc(m));
    slot0 = __shfl_sync(0xffffffffu, slot0, 0);
    if (fresh) {
      const int slot = slot0 + __popc(m & lt);
      if (slot < stage_cap) {
        stage_list[slot] = v;
        stage_row[v] = slot;
      } else {
        raise_flag(err, HG_EINVARIANT);
      }
    }
    if (uniq_per_home) {
      for (int q = 0; q < n_homes; ++q) {
        const unsigned mq = __ballot_sync(0xffffffffu, fresh && h == q);
        if (lane == 0 && mq) atomicAdd(uniq_per_home + q, (unsigned long long)__popc(mq));
      }
    }
  }
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if (total_remote && lane == 0 && mine) atomicAdd(total_remote, mine);
}

// k_stage_mark_stamp over a whole run-ahead group in ONE launch: blockIdx.y
// selects the segment (iteration); one stamp tag for the call, so a vertex
// several segments want is listed once.
struct StageSegs {
  const int32_t* ids[HG_MAX_GROUP];
  const int32_t* n_dev[HG_MAX_GROUP];
};

__global__ void k_stage_mark_stamp_multi(StageSegs segs, const int32_t* __restrict__ home,
                                         int rank, int32_t* __restrict__ stamp,
                                         const int64_t* __restrict__ seq,
                                         int32_t* __restrict__ stage_list,
                                         int32_t* __restrict__ stage_row,
                                         int32_t* __restrict__ stage_count, int stage_cap,
                                         int* err) {
  const int32_t* ids = segs.ids[blockIdx.y];
  const int n = *segs.n_dev[blockIdx.y];
  int32_t tag = (int32_t)((*seq + 1) & 0x7fffffff);
  if (tag == 0) tag = 1;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    int v = 0, h = rank;
    if (i < n) {
      v = ids[i];
      h = home[v];
    }
    const bool fresh = h != rank && atomicExch(stamp + v, tag) != tag;
    const unsigned m = __ballot_sync(0xffffffffu, fresh);
    if (!m) continue;
    int slot0 = 0;
    if (lane == 0) slot0 = atomicAdd(stage_count, __popc(m));
    slot0 = __shfl_sync(0xffffffffu, slot0, 0);
    if (fresh) {
      const int slot = slot0 + __popc(m & lt);
      if (slot < stage_cap) {
        stage_list[slot] = v;
        stage_row[v] = slot;
      } else {
        raise_flag(err, HG_EINVARIANT);
      }
    }
  }
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

// ---------------------------------------------------------------- push pre-gather
//
// Random row reads from a peer's 10+ GB shard are bound by the requester's
// peer-mapping TLB (measured: 9K random 256-B rows 80 GB/s, 36K rows 29 GB/s;
// sequential 157 GB/s).  The push variant turns them around: each rank
// publishes its deduplicated request list in its mailbox, the OWNER gathers
// the rows from its local shard (local TLB) and writes them into the
// requester's staging rows over NVLink (a small contiguous region).
// Mailbox (one cudaMalloc per rank, IPC-mapped by every peer):
//   flags[S] i64 | done[S] i64 | count i32 | list[cap] i32 | staging[cap x row]
// flags[p] / done[p] = sequence number of p's latest "requests ready" / "my
// rows written" signal; the sequence advances once per pre-gather on every rank.

struct Mailbox {
  int64_t o_flags, o_done, o_count, o_list, o_staging;
};

__device__ __forceinline__ uint8_t* mb_base(const uint64_t* boxes, int p) {
  return reinterpret_cast<uint8_t*>(boxes[p]);
}

// wait until every peer's counter (at box[rank] + off + 8*p, written by p) reaches seq
__device__ bool spin_peers(const uint64_t* boxes, int rank, int S, int64_t off, int64_t seq) {
  volatile int64_t* mine = reinterpret_cast<volatile int64_t*>(mb_base(boxes, rank) + off);
  for (long long it = 0; it < (1ll << 26); ++it) {
    bool all = true;
    for (int p = 0; p < S; ++p)
      if (p != rank && mine[p] < seq) all = false;
    if (all) return true;
    __nanosleep(64);
  }
  return false;
}

__global__ void k_pg_signal(const uint64_t* __restrict__ boxes, int rank, int S, Mailbox m,
                            int64_t* seq, int64_t off) {
  if (threadIdx.x != 0) return;
  const int64_t v = (off == m.o_flags) ? *seq + 1 : *seq;
  if (off == m.o_flags) *seq = v;
  __threadfence_system();
  for (int p = 0; p < S; ++p) {
    if (p == rank) continue;
    volatile int64_t* f = reinterpret_cast<volatile int64_t*>(mb_base(boxes, p) + off);
    f[rank] = v;
  }
  __threadfence_system();
}

__global__ void k_pg_wait(const uint64_t* __restrict__ boxes, int rank, int S, Mailbox m,
                          const int64_t* seq, int64_t off, int* err) {
  if (threadIdx.x == 0 && !spin_peers(boxes, rank, S, off, *seq)) raise_flag(err, HG_EINVARIANT);
}

// owner side: serve every peer's requests homed here.  A warp reads 32 list
// entries of the requester's mailbox in one coalesced NVLink load (the list
// lives in the REQUESTER's memory; one dependent remote read per entry was
// the serve's latency chain), looks their homes up locally, then copies the
// rows homed here two at a time (half a warp per 256-byte row) into the
// requester's staging rows.
__global__ void __launch_bounds__(256)
k_pg_serve(const uint64_t* __restrict__ boxes, int rank, int S, Mailbox m, const int64_t* seq,
           const int32_t* __restrict__ home, const int32_t* __restrict__ local_row,
           const uint8_t* __restrict__ shard, int row_bytes, int stage_cap, int* err) {
  // the requests are ready: k_pg_wait (one CTA) polled the peers' signals, so
  // these CTAs never occupy SM slots while spinning
  const unsigned full = 0xffffffffu;
  const int vec = row_bytes / 16;
  const int lane = threadIdx.x & 31, hl = lane & 15;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int n_w = (gridDim.x * blockDim.x) >> 5;
  for (int p = 0; p < S; ++p) {
    if (p == rank) continue;
    uint8_t* box = mb_base(boxes, p);
    const int n = min(*reinterpret_cast<volatile int32_t*>(box + m.o_count), stage_cap);
    const int32_t* list = reinterpret_cast<const int32_t*>(box + m.o_list);
    uint8_t* staging = box + m.o_staging;
    for (int base = w * 32; base < n; base += n_w * 32) {
      const int i = base + lane;
      const int v = i < n ? list[i] : -1;
      const bool mine = v >= 0 && home[v] == rank;
      const int r = mine ? local_row[v] : 0;
      unsigned todo = __ballot_sync(full, mine);
      while (todo) {  // warp-uniform: two rows per round, one per half-warp
        const int j0 = __ffs(todo) - 1;
        todo &= todo - 1;
        int j1 = -1;
        if (todo) {
          j1 = __ffs(todo) - 1;
          todo &= todo - 1;
        }
        const int j = lane < 16 ? j0 : j1;
        const int rr = __shfl_sync(full, r, j < 0 ? 0 : j);
        if (j >= 0) {
          const uint4* src = reinterpret_cast<const uint4*>(shard + (int64_t)rr * row_bytes);
          uint4* dst = reinterpret_cast<uint4*>(staging + (int64_t)(base + j) * row_bytes);
          for (int c = hl; c < vec; c += 16) dst[c] = src[c];
        }
      }
    }
  }
  __threadfence_system();  // rows land before the "done" signal of the next kernel
}

}  // namespace hg

using namespace hg;

extern "C" int hg_pregather_push(const int32_t* ids, const int32_t* n_dev, const int32_t* home,
                                 int32_t rank, int32_t n_ranks, const int32_t* local_row,
                                 const void* shard, int32_t row_bytes, int32_t* stamp,
                                 int32_t* stage_row, int32_t stage_cap, const void* boxes,
                                 void* own_box, int64_t o_flags, int64_t o_done, int64_t o_count,
                                 int64_t o_list, int64_t o_staging,
                                 unsigned long long* uniq_per_home, const int64_t* it_dev,
                                 int32_t row_stride, unsigned long long* total_remote,
                                 int64_t* seq, int* err, void* stream) {
  if (row_bytes % 16) return hg_fail(HG_ECONFIG, "row bytes must be a multiple of 16");
  cudaStream_t s = (cudaStream_t)stream;
  const Mailbox m{o_flags, o_done, o_count, o_list, o_staging};
  const uint64_t* bx = (const uint64_t*)boxes;
  uint8_t* own = (uint8_t*)own_box;
  int32_t* count = (int32_t*)(own + o_count);
  HG_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(int32_t), s));
  count_launch(6);
  prof_begin(PROF_PG_MARK, s);
  k_stage_mark_stamp<<<148 * 2, 256, 0, s>>>(ids, n_dev, home, rank, n_ranks, stamp, seq,
                                             (int32_t*)(own + o_list), stage_row, count,
                                             stage_cap, uniq_per_home, total_remote, err, it_dev,
                                             row_stride);
  prof_end(PROF_PG_MARK, s);
  prof_begin(PROF_PG_COPY, s);
  k_pg_signal<<<1, 32, 0, s>>>(bx, rank, n_ranks, m, seq, o_flags);          // requests ready
  k_pg_wait<<<1, 32, 0, s>>>(bx, rank, n_ranks, m, seq, o_flags, err);       // peers' requests
  k_pg_serve<<<148 * 2, 256, 0, s>>>(bx, rank, n_ranks, m, seq, home, local_row,
                                     (const uint8_t*)shard, row_bytes, stage_cap, err);
  k_pg_signal<<<1, 32, 0, s>>>(bx, rank, n_ranks, m, seq, o_done);           // my rows written
  k_pg_wait<<<1, 32, 0, s>>>(bx, rank, n_ranks, m, seq, o_done, err);        // all rows here
  prof_end(PROF_PG_COPY, s);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_pregather_push_multi(const int32_t* const* ids, const int32_t* const* n_dev,
                                       int32_t n_seg, const int32_t* home, int32_t rank,
                                       int32_t n_ranks, const int32_t* local_row,
                                       const void* shard, int32_t row_bytes, int32_t* stamp,
                                       int32_t* stage_row, int32_t stage_cap, const void* boxes,
                                       void* own_box, int64_t o_flags, int64_t o_done,
                                       int64_t o_count, int64_t o_list, int64_t o_staging,
                                       int64_t* seq, int* err, void* stream) {
  if (row_bytes % 16) return hg_fail(HG_ECONFIG, "row bytes must be a multiple of 16");
  if (n_seg < 1) return hg_fail(HG_ERANGE, "no segments");
  cudaStream_t s = (cudaStream_t)stream;
  const Mailbox m{o_flags, o_done, o_count, o_list, o_staging};
  const uint64_t* bx = (const uint64_t*)boxes;
  uint8_t* own = (uint8_t*)own_box;
  int32_t* count = (int32_t*)(own + o_count);
  HG_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(int32_t), s));
  count_launch(6);
  prof_begin(PROF_PG_MARK, s);
  // one stamp tag for the whole call: a vertex wanted by several segments is
  // requested once
  if (n_seg > HG_MAX_GROUP) return hg_fail(HG_ERANGE, "at most %d segments", HG_MAX_GROUP);
  StageSegs sg{};
  for (int g = 0; g < n_seg; ++g) {
    sg.ids[g] = ids[g];
    sg.n_dev[g] = n_dev[g];
  }
  k_stage_mark_stamp_multi<<<dim3(148, n_seg), 256, 0, s>>>(sg, home, rank, stamp, seq,
                                                           (int32_t*)(own + o_list), stage_row,
                                                           count, stage_cap, err);
  prof_end(PROF_PG_MARK, s);
  prof_begin(PROF_PG_COPY, s);
  k_pg_signal<<<1, 32, 0, s>>>(bx, rank, n_ranks, m, seq, o_flags);
  k_pg_wait<<<1, 32, 0, s>>>(bx, rank, n_ranks, m, seq, o_flags, err);
  k_pg_serve<<<148 * 2, 256, 0, s>>>(bx, rank, n_ranks, m, seq, home, local_row,
                                     (const uint8_t*)shard, row_bytes, stage_cap, err);
  k_pg_signal<<<1, 32, 0, s>>>(bx, rank, n_ranks, m, seq, o_done);
  k_pg_wait<<<1, 32, 0, s>>>(bx, rank, n_ranks, m, seq, o_done, err);
  prof_end(PROF_PG_COPY, s);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_remote_account_at(const int32_t* ids, const int32_t* n_dev, const int32_t* home,
                                    int32_t rank, uint32_t* bitmap,
                                    unsigned long long* uniq_table, const int64_t* it_dev,
                                    int32_t ahead, int32_t row_stride,
                                    unsigned long long* total_remote, void* stream) {
  count_launch();
  k_remote_account_at<<<148 * 2, 256, 0, (cudaStream_t)stream>>>(
      ids, n_dev, home, rank, bitmap, uniq_table, it_dev, ahead, row_stride, total_remote);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

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
  prof_begin(PROF_PG_MARK, s);
  k_stage_mark<<<148 * 2, 256, 0, s>>>(ids, n_dev, home, rank, row_stride > 0 ? row_stride : 64,
                                       bitmap, stage_list, stage_row, stage_count, stage_cap,
                                       uniq_per_home, total_remote, err, it_dev, row_stride);
  prof_end(PROF_PG_MARK, s);
  prof_begin(PROF_PG_COPY, s);
  k_stage_copy<<<148 * 4, 256, 0, s>>>(stage_list, stage_count, stage_cap, home, local_row,
                                       (const uint8_t* const*)peers, row_bytes, (uint8_t*)staging);
  prof_end(PROF_PG_COPY, s);
  prof_begin(PROF_PG_CLEAR, s);
  k_remote_clear<<<148 * 2, 256, 0, s>>>(ids, n_dev, 0, bitmap);
  prof_end(PROF_PG_CLEAR, s);
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
  const size_t b = bytes < 256 ? 256 : bytes;
  HG_CUDA_TRY(cudaMalloc(out, b));
  HG_CUDA_TRY(cudaMemset(*out, 0, b));  // mailboxes rely on zeroed counters
  return HG_OK;
}

__global__ void k_flag_if_differ(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                                 int64_t n, int* flag, int code) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (a[i] != b[i]) { raise_flag(flag, code); return; }
}

// Device-side replica check of the model hop (model.py:311-314 "replicas
// diverged"): bitwise compare of two f32 buffers, raising HG_EINVARIANT in
// *flag on any difference -- no host synchronisation inside the step.
extern "C" int hg_flag_if_differ(const float* a, const float* b, int64_t n, int* flag,
                                 void* stream) {
  if (n <= 0) return HG_OK;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 4);
  k_flag_if_differ<<<grid, 256, 0, (cudaStream_t)stream>>>((const uint32_t*)a,
                                                            (const uint32_t*)b, n, flag,
                                                            HG_EINVARIANT);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes) HG_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice,
                                         (cudaStream_t)stream));
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

// The reference ledger rows of a whole run-ahead group in two launches
// (blockIdx.y = iteration j of the group, its own bitmap j): per-iteration
// dedup exactly as hg_remote_account_at + hg_remote_clear per iteration.
__global__ void k_remote_account_group(StageSegs segs, const int32_t* __restrict__ home, int rank,
                                       uint32_t* __restrict__ bitmaps, int64_t words,
                                       unsigned long long* __restrict__ table,
                                       const int64_t* __restrict__ it_dev, int row_stride,
                                       unsigned long long* __restrict__ total_remote) {
  const int j = blockIdx.y;
  const int32_t* ids = segs.ids[j];
  const int n = *segs.n_dev[j];
  uint32_t* bitmap = bitmaps + j * words;
  unsigned long long* uniq_per_home = table + (*it_dev + 1 + j) * row_stride;
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
  if (total_remote && (threadIdx.x & 31) == 0 && mine) atomicAdd(total_remote, mine);
}

__global__ void k_remote_clear_group(StageSegs segs, uint32_t* __restrict__ bitmaps,
                                     int64_t words) {
  const int j = blockIdx.y;
  const int32_t* ids = segs.ids[j];
  const int n = *segs.n_dev[j];
  uint32_t* bitmap = bitmaps + j * words;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    bitmap[ids[i] >> 5] = 0u;
}

__global__ void k_resolve_rows_group(StageSegs segs, const int32_t* __restrict__ home, int rank,
                                     const int32_t* __restrict__ local_row,
                                     const int32_t* __restrict__ stage_row, StageSegs outs) {
  const int j = blockIdx.y;
  const int32_t* ids = segs.ids[j];
  const int n = *segs.n_dev[j];
  int32_t* out = const_cast<int32_t*>(outs.ids[j]);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int v = ids[i];
    out[i] = home[v] == rank ? local_row[v] : -1 - stage_row[v];
  }
}

extern "C" int hg_remote_account_group(const int32_t* const* ids, const int32_t* const* n_dev,
                                       int32_t n_seg, const int32_t* home, int32_t rank,
                                       uint32_t* bitmaps, int64_t words,
                                       unsigned long long* uniq_table, const int64_t* it_dev,
                                       int32_t row_stride, unsigned long long* total_remote,
                                       void* stream) {
  if (n_seg < 1 || n_seg > HG_MAX_GROUP) return hg_fail(HG_ERANGE, "bad segment count %d", n_seg);
  StageSegs sg{};
  for (int g = 0; g < n_seg; ++g) {
    sg.ids[g] = ids[g];
    sg.n_dev[g] = n_dev[g];
  }
  cudaStream_t s = (cudaStream_t)stream;
  count_launch(2);
  k_remote_account_group<<<dim3(148, n_seg), 256, 0, s>>>(sg, home, rank, bitmaps, words,
                                                          uniq_table, it_dev, row_stride,
                                                          total_remote);
  HG_CUDA_TRY(cudaGetLastError());
  k_remote_clear_group<<<dim3(148, n_seg), 256, 0, s>>>(sg, bitmaps, words);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_resolve_rows_group(const int32_t* const* ids, const int32_t* const* n_dev,
                                     int32_t n_seg, const int32_t* home, int32_t rank,
                                     const int32_t* local_row, const int32_t* stage_row,
                                     int32_t* const* out, void* stream) {
  if (n_seg < 1 || n_seg > HG_MAX_GROUP) return hg_fail(HG_ERANGE, "bad segment count %d", n_seg);
  StageSegs sg{}, so{};
  for (int g = 0; g < n_seg; ++g) {
    sg.ids[g] = ids[g];
    sg.n_dev[g] = n_dev[g];
    so.ids[g] = out[g];
  }
  count_launch();
  k_resolve_rows_group<<<dim3(148, n_seg), 256, 0, (cudaStream_t)stream>>>(
      sg, home, rank, local_row, stage_row, so);
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

__global__ void k_resolve_rows(const int32_t* __restrict__ ids, const int32_t* __restrict__ n_dev,
                               const int32_t* __restrict__ home, int rank,
                               const int32_t* __restrict__ local_row,
                               const int32_t* __restrict__ stage_row, int32_t* __restrict__ out) {
  const int n = *n_dev;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int v = ids[i];
    out[i] = home[v] == rank ? local_row[v] : -1 - stage_row[v];
  }
}

extern "C" int hg_resolve_rows(const int32_t* ids, const int32_t* n_dev, const int32_t* home,
                               int32_t rank, const int32_t* local_row, const int32_t* stage_row,
                               int32_t* out, void* stream) {
  if (!ids || !n_dev || !home || !local_row || !stage_row || !out)
    return hg_fail(HG_ERANGE, "hg_resolve_rows: null argument");
  count_launch();
  k_resolve_rows<<<148 * 4, 256, 0, (cudaStream_t)stream>>>(ids, n_dev, home, rank, local_row,
                                                            stage_row, out);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

// ---------------------------------------------------------------- P2P all-reduce
namespace hg {
//
// Gradient all-reduce over NVLink peer memory (the synchronous update of
// model.py:299-324 across one-process-per-GPU ranks), replacing the NCCL
// all-reduce on the training stream:
//   push   every rank writes its accumulator into slot [rank] of buffer
//          (seq & 1) in EVERY peer's exchange region (fire-and-forget NVLink
//          stores), the last CTA bumps the device sequence number and sets
//          flag[rank] = seq in every peer's region (system-scope fences);
//   wait   one CTA polls this rank's flags until every peer published seq
//          (bounded: an error flag instead of a hang);
//   reduce g += sum of the peers' slots (local HBM reads), after which the
//          regular fused SGD + bf16 refresh runs (hg_sgd_refresh).
// Double buffering by seq parity is safe: a rank reuses buffer (s & 1) for
// s + 2 only after every peer published s + 1, which each peer does after its
// reduce of s (stream order).  Region layout: [S int64 flags | pad to 256 |
// 2 x S x n floats].
struct ArRegion {
  int64_t o_flags, o_buf;
};

__device__ __forceinline__ float* ar_slot(uint8_t* region, ArRegion r, int parity, int S, int p,
                                          int64_t n) {
  return reinterpret_cast<float*>(region + r.o_buf) + ((int64_t)parity * S + p) * n;
}

__global__ void __launch_bounds__(256)
k_ar_push(const float* __restrict__ g, int64_t n, const uint64_t* __restrict__ regions, int rank,
          int S, ArRegion r, int64_t* seq, unsigned int* counter) {
  const int64_t s = *seq + 1;
  const int par = (int)(s & 1);
  for (int p = 0; p < S; ++p) {
    if (p == rank) continue;
    float* dst = ar_slot(reinterpret_cast<uint8_t*>(regions[p]), r, par, S, rank, n);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
      dst[i] = g[i];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int t = atomicAdd(counter, 1u);
    if (t == gridDim.x - 1) {  // every CTA's stores are fenced: publish s
      *counter = 0u;
      *seq = s;
      __threadfence_system();
      for (int p = 0; p < S; ++p) {
        if (p == rank) continue;
        volatile int64_t* f =
            reinterpret_cast<volatile int64_t*>(reinterpret_cast<uint8_t*>(regions[p]) + r.o_flags);
        f[rank] = s;
      }
      __threadfence_system();
    }
  }
}

__global__ void k_ar_wait(const uint64_t* __restrict__ regions, int rank, int S, ArRegion r,
                          const int64_t* seq, int* err) {
  if (threadIdx.x != 0) return;
  const int64_t s = *seq;
  volatile int64_t* mine =
      reinterpret_cast<volatile int64_t*>(reinterpret_cast<uint8_t*>(regions[rank]) + r.o_flags);
  for (long long it = 0; it < (1ll << 26); ++it) {
    bool all = true;
    for (int p = 0; p < S; ++p)
      if (p != rank && mine[p] < s) all = false;
    if (all) { __threadfence_system(); return; }
    __nanosleep(64);
  }
  raise_flag(err, HG_EINVARIANT);
}

__global__ void __launch_bounds__(256)
k_ar_reduce(float* __restrict__ g, int64_t n, const uint64_t* __restrict__ regions, int rank,
            int S, ArRegion r, const int64_t* seq) {
  const int par = (int)(*seq & 1);
  uint8_t* mine = reinterpret_cast<uint8_t*>(regions[rank]);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = g[i];
    for (int p = 0; p < S; ++p)
      if (p != rank) v += ar_slot(mine, r, par, S, p, n)[i];
    g[i] = v;
  }
}

}  // namespace hg

using namespace hg;

extern "C" int hg_p2p_region_bytes(int32_t n_ranks, int64_t n, int64_t* bytes) {
  const int64_t flags = ((int64_t)n_ranks * 8 + 255) / 256 * 256;
  *bytes = flags + 2ll * n_ranks * n * 4;
  return HG_OK;
}

extern "C" int hg_p2p_allreduce(float* grads, int64_t n, const uint64_t* regions, int32_t rank,
                                int32_t n_ranks, int64_t* seq, unsigned int* counter, int* err,
                                void* stream) {
  if (n_ranks < 1 || rank < 0 || rank >= n_ranks) return hg_fail(HG_ERANGE, "bad rank");
  if (n_ranks == 1 || n <= 0) return HG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  ArRegion r{0, ((int64_t)n_ranks * 8 + 255) / 256 * 256};
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)nsm);
  count_launch(3);
  k_ar_push<<<grid, 256, 0, s>>>(grads, n, regions, rank, n_ranks, r, seq, counter);
  HG_CUDA_TRY(cudaGetLastError());
  k_ar_wait<<<1, 32, 0, s>>>(regions, rank, n_ranks, r, seq, err);
  HG_CUDA_TRY(cudaGetLastError());
  k_ar_reduce<<<grid, 256, 0, s>>>(grads, n, regions, rank, n_ranks, r, seq);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}
