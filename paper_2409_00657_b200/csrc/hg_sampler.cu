// Bit-exact k-hop micrograph sampling, dedup/relabel and need-chain plan.
//
// Reference semantics:
//   * draw rule  -- _kernels_nb.py:55-86: deg <= fanout keeps all neighbours
//     in CSR order; otherwise slot j gets key (mix64(mix64(state^v)^j) & HI32)|j
//     and the `fanout` smallest keys win, emitted in ascending slot order;
//   * hop loop   -- sampler.py:92-105 (hop h = L-k uses fanout[h-1] and
//     state chain(key, h); layers sorted-unique; pairs = searchsorted);
//   * plan       -- model.py:183-198 (need[k] = union(layers[k], need[k+1]),
//     self_pos / dpos / spos / deg).
//
// B200 design: one CTA (8 warps) owns one root's micrograph in shared memory.
// Per frontier vertex the draw is a *threshold select*: one hashing pass keeps
// only slots whose hash is below a threshold sized for ~fanout+4*sqrt(fanout)+8
// expected survivors (ballot compaction into smem), then the exact `fanout`
// smallest survivors are ranked in smem.  Cost is one mix64 per slot, no sort
// of the hub's adjacency.  Vertices with degree <= 256 are handled by one
// warp; larger hubs by the whole CTA.  A rare under/overflow of the survivor
// buffer bisects the threshold and retries, so the result is always exact.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstdio>

#include <cub/device/device_scan.cuh>

#include "hg_common.cuh"

namespace hg {

#ifndef HG_BUILD_THREADS
#define HG_BUILD_THREADS 256
#endif
constexpr int kBuildThreads = HG_BUILD_THREADS;
#ifndef HG_BUILD_MINB
#define HG_BUILD_MINB 4  // resident build CTAs per SM (64 regs, no spills)
#endif
constexpr int kBuildWarps = kBuildThreads / 32;
constexpr int kBigTask = 256;  // degree above which the whole CTA draws one vertex

// Output descriptors of a group of batches built by one launch (run-ahead over
// several iterations): batch b's roots are [b * n_roots, (b + 1) * n_roots).
struct MgOuts {
  hg_mg_batch b[HG_MAX_GROUP];
};

// The CSR the builds read: one table (single GPU, replicated), or one shard
// per home server mapped over NVLink (partitioned topology, north_star): the
// row of v lives in shard home(v) at local row v - vstart[home(v)]
// (contiguous partitions, e.g. planted blocks), or at row_of[v] with home
// from home_of[v] (arbitrary partitions).
struct CsrView {
  const int64_t* off[HG_MAX_SHARDS];
  const int32_t* tgt[HG_MAX_SHARDS];
  int64_t vstart[HG_MAX_SHARDS + 1];
  const int32_t* home_of;  // NULL: contiguous ranges (vstart)
  const int32_t* row_of;
  int S;
};

__device__ __forceinline__ int csr_row(const CsrView& g, int64_t v, int64_t* lo) {
  int h = 0;
  int64_t r = v;
  if (g.S > 1) {
    if (g.home_of) {
      h = g.home_of[v];
      r = g.row_of[v];
    } else {
      while (h + 1 < g.S && v >= g.vstart[h + 1]) ++h;
      r = v - g.vstart[h];
    }
  }
  const int64_t* off = g.off[h];
  *lo = off[r];
  return (int)(off[r + 1] - *lo) | (h << 26);  // degree < 2^26, shard in the top bits
}
__device__ __forceinline__ int row_deg(int packed) { return packed & ((1 << 26) - 1); }
__device__ __forceinline__ int row_shard(int packed) { return packed >> 26; }

struct MgCarve {
  int L;
  int fanout[HG_MAX_LAYERS];
  int mean[HG_MAX_LAYERS];
  int cap_lay[HG_MAX_LAYERS + 1];
  int cap_need[HG_MAX_LAYERS + 1];
  // shared-memory int offsets
  int sm_lay[HG_MAX_LAYERS + 1], sm_need[HG_MAX_LAYERS + 1];
  int sm_flat[HG_MAX_LAYERS + 1], sm_cnt[HG_MAX_LAYERS + 1], sm_off[HG_MAX_LAYERS + 1],
      sm_deg[HG_MAX_LAYERS + 1];
  int sm_sort, sm_scan, sm_misc, sm_ints;
  int cand_cap, sort_cap;
  int cand_byte_off;  // byte offset of the candidate buffers (8-aligned)
  int smem_bytes;
  // per-root workspace int offsets
  int ws_need[HG_MAX_LAYERS + 1], ws_inl[HG_MAX_LAYERS + 1];
  int ws_self[HG_MAX_LAYERS + 1], ws_rowoff[HG_MAX_LAYERS + 1], ws_nbr[HG_MAX_LAYERS + 1];
  int ws_cnt, ws_root_ints;
};

static int pow2ceil(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

static int isqrt_ceil(int x) {
  int r = 0;
  while (r * r < x) ++r;
  return r;
}

// expected survivors of the threshold pass: fanout + 2 sqrt(fanout) + 4 (a ~2-sigma margin;
// an under- or overflow re-runs the pass with a bisected threshold, so the draw stays
// exact -- the margin only trades retries against the O(m) candidate rank)
int select_mean(int fanout) { return fanout + 2 * isqrt_ceil(fanout) + 4; }

int make_carve(int L, const int32_t* fanout, MgCarve* c) {
  if (L < 1 || L > HG_MAX_LAYERS) return hg_fail(HG_ECONFIG, "n_layers must be 1..%d", HG_MAX_LAYERS);
  *c = MgCarve{};
  c->L = L;
  int max_mean = 0;
  for (int h = 0; h < L; ++h) {
    if (fanout[h] < 1) return hg_fail(HG_ECONFIG, "fanout must be >= 1");
    c->fanout[h] = fanout[h];
    c->mean[h] = select_mean(fanout[h]);
    max_mean = c->mean[h] > max_mean ? c->mean[h] : max_mean;
  }
  c->cap_lay[L] = 1;
  for (int k = L - 1; k >= 0; --k) {
    long long v = (long long)c->cap_lay[k + 1] * c->fanout[L - k - 1];
    if (v > (1 << 16)) return hg_fail(HG_ECONFIG, "micrograph layer capacity %lld too large", v);
    c->cap_lay[k] = (int)v;
  }
  c->cap_need[L] = 1;
  for (int k = L - 1; k >= 0; --k) c->cap_need[k] = c->cap_lay[k] + c->cap_need[k + 1];
  c->cand_cap = pow2ceil(2 * max_mean < 64 ? 64 : 2 * max_mean);
  int mx = 1;
  for (int k = 0; k <= L; ++k) mx = c->cap_need[k] > mx ? c->cap_need[k] : mx;
  c->sort_cap = pow2ceil(mx);
  int o = 0;
  for (int k = 0; k <= L; ++k) { c->sm_lay[k] = o; o += c->cap_lay[k]; }
  for (int k = 0; k <= L; ++k) { c->sm_need[k] = o; o += c->cap_need[k]; }
  for (int h = 1; h <= L; ++h) {
    int k = L - h;
    c->sm_flat[h] = o; o += c->cap_lay[k];
    c->sm_cnt[h] = o; o += c->cap_lay[k + 1];
    c->sm_off[h] = o; o += c->cap_lay[k + 1] + 1;
    c->sm_deg[h] = o; o += c->cap_lay[k + 1];
  }
  c->sm_sort = o; o += c->sort_cap;
  c->sm_scan = o; o += 40;
  c->sm_misc = o; o += 8 + 2 * kBuildWarps + 2 * kBuildWarps;  // counters + T slots
  c->sm_ints = o;
  c->cand_byte_off = ((o * 4 + 15) / 16) * 16;
  c->smem_bytes = c->cand_byte_off + (kBuildWarps + 1) * c->cand_cap * 8;
  if (c->smem_bytes > 227 * 1024)
    return hg_fail(HG_ECONFIG, "micrograph tile needs %d B shared memory (> 227 KB)", c->smem_bytes);
  int w = 0;
  for (int k = 0; k <= L; ++k) {
    c->ws_need[k] = w; w += c->cap_need[k];
    c->ws_inl[k] = w; w += c->cap_need[k];
  }
  for (int k = 1; k <= L; ++k) {
    c->ws_self[k] = w; w += c->cap_need[k];
    c->ws_rowoff[k] = w; w += c->cap_need[k] + 1;
    c->ws_nbr[k] = w; w += c->cap_lay[k - 1];
  }
  c->ws_cnt = w; w += 2 * L + 2;
  c->ws_root_ints = w;
  return HG_OK;
}

// ---------------------------------------------------------------- team select

struct WarpTeam {
  __device__ static int rank() { return lane_id(); }
  __device__ static int size() { return 32; }
  __device__ static int warp_in_team() { return 0; }
  __device__ static void sync() { __syncwarp(); }
};
struct BlockTeam {
  __device__ static int rank() { return threadIdx.x; }
  __device__ static int size() { return blockDim.x; }
  __device__ static int warp_in_team() { return warp_id(); }
  __device__ static void sync() { __syncthreads(); }
};

// Exact "fanout smallest keyed slots" of one frontier vertex, written to out
// in ascending slot order.  cand: team candidate buffer (cap entries);
// ctr / tsh: team-private shared scratch.  Requires d > fo.
template <class Team>
__device__ void team_select(const int32_t* __restrict__ targets, int64_t lo, int d, int fo,
                            int mean, uint64_t hv, int32_t* out, uint64_t* cand, int cap,
                            int* ctr, uint64_t* tsh, int* err) {
  const int lane = lane_id();
  // threshold for ~mean survivors: any value keeps the draw exact (the count
  // check below retries), so a float quotient replaces the 64-bit division
  uint64_t gh = mean >= d ? (1ull << 32)
                          : (uint64_t)__float2ull_rz(__fdividef((float)mean, (float)d) * 4294967296.0f);
  uint64_t lo_b = 0, hi_b = 1ull << 33;
  int m = 0;
  for (int attempt = 0;; ++attempt) {
    if (Team::rank() == 0) *ctr = 0;
    Team::sync();
    // kU slots per lane per pass: independent hashes in flight, and the
    // warp-uniform survivor count skips the shared-counter round trip on the
    // (typical) passes where nothing falls below the threshold
    constexpr int kU = 4;
    const unsigned lt = (1u << lane) - 1u;
    for (int base = Team::warp_in_team() * 32 * kU; base < d; base += Team::size() * kU) {
      bool take[kU];
      uint64_t key[kU];
      unsigned mask[kU];
      int cw = 0;
#pragma unroll
      for (int u = 0; u < kU; ++u) {  // branch-free: slots past d hash too, never taken
        const int j = base + u * 32 + lane;
        const uint64_t h = mix64(hv ^ (uint64_t)j);
        take[u] = j < d && (h >> 32) < gh;
        key[u] = (h & kHi32) | (uint64_t)(uint32_t)j;
        mask[u] = __ballot_sync(0xffffffffu, take[u]);
        cw += __popc(mask[u]);
      }
      if (cw) {
        int off = 0;
        if (lane == 0) off = atomicAdd(ctr, cw);
        off = __shfl_sync(0xffffffffu, off, 0);
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int pos = off + __popc(mask[u] & lt);
          if (take[u] && pos < cap) cand[pos] = key[u];
          off += __popc(mask[u]);
        }
      }
    }
    Team::sync();
    const int cnt = *ctr;
    Team::sync();
    if (cnt >= fo && cnt <= cap) { m = cnt; break; }
    if (attempt > 80) {  // cannot happen for distinct keys; keep shapes valid
      raise_flag(err, HG_EINVARIANT);
      for (int i = Team::rank(); i < fo; i += Team::size()) out[i] = targets[lo + i];
      Team::sync();
      return;
    }
    if (cnt < fo) lo_b = gh; else hi_b = gh;
    if (hi_b == (1ull << 33)) {
      gh = gh * 2 + 1;
      if (gh > (1ull << 32)) gh = 1ull << 32;
    } else {
      gh = (lo_b + hi_b) >> 1;
    }
  }
  // T = fanout-th smallest candidate key
  uint64_t T = 0;
  bool have_t = false;
  if (Team::size() == 32 && m <= 32) {
    // one candidate per lane: rank on the 32-bit hash parts (one compare per
    // candidate, shuffles instead of shared-memory loads) unless two hash
    // parts are equal, where the slot decides (64-bit path below)
    const uint64_t ki = lane < m ? cand[lane] : ~0ull;
    const uint32_t hi = (uint32_t)(ki >> 32);
    const unsigned valid = m >= 32 ? 0xffffffffu : ((1u << m) - 1u);
    const unsigned same = __match_any_sync(0xffffffffu, hi) & valid;
    if (!__any_sync(0xffffffffu, lane < m && __popc(same) > 1)) {
      int rank = 0;
      for (int c = 0; c < m; ++c) rank += __shfl_sync(0xffffffffu, hi, c) < hi;
      const unsigned b = __ballot_sync(0xffffffffu, lane < m && rank == fo - 1);
      T = __shfl_sync(0xffffffffu, ki, __ffs(b) - 1);
      have_t = true;
    }
  }
  if (!have_t) {
    for (int i = Team::rank(); i < m; i += Team::size()) {
      const uint64_t ki = cand[i];
      int rank = 0;
      for (int c = 0; c < m; ++c) rank += cand[c] < ki;
      if (rank == fo - 1) *tsh = ki;
    }
    Team::sync();
    T = *tsh;
  }
  if (Team::size() == 32) {
    // one warp filled cand[] in ascending slot order (passes in slot order,
    // ballot positions lane-ordered): the selected keys' output positions are
    // a running ballot count
    int base = 0;
    for (int i0 = 0; i0 < m; i0 += 32) {
      const int i = i0 + lane;
      const uint64_t ki = i < m ? cand[i] : ~0ull;
      const bool sel = ki <= T;
      const unsigned b = __ballot_sync(0xffffffffu, sel);
      if (sel) out[base + __popc(b & ((1u << lane) - 1u))] = targets[lo + (uint32_t)ki];
      base += __popc(b);
    }
    Team::sync();
    return;
  }
  for (int i = Team::rank(); i < m; i += Team::size()) {
    const uint64_t ki = cand[i];
    if (ki <= T) {
      const uint32_t slot = (uint32_t)ki;
      int pos = 0;
      for (int c = 0; c < m; ++c) {
        const uint64_t kc = cand[c];
        pos += (kc <= T) && ((uint32_t)kc < slot);
      }
      out[pos] = targets[lo + slot];
    }
  }
  Team::sync();
}

// ---------------------------------------------------------------- block sort

// One warp sorts up to 32*E ints held in registers (element i = lane*E + j):
// bitonic network, in-register exchanges for strides < E, shuffles above;
// then writes the distinct values to out and returns their count.  No block
// barriers, which dominate the block-wide network for the small layers of
// (15,10)-style micrographs.
template <int E>
__device__ int warp_sort_unique(const int* in, int n, int* out) {
  const int lane = lane_id();
  int x[E];
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const int i = lane * E + j;
    x[j] = i < n ? in[i] : INT_MAX;
  }
#pragma unroll
  for (int size = 2; size <= 32 * E; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= E) {
        const int lm = stride / E;
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const int i = lane * E + j;
          const int y = __shfl_xor_sync(0xffffffffu, x[j], lm);
          const bool up = (i & size) == 0;
          const bool lower = (i & stride) == 0;
          x[j] = (lower == up) ? min(x[j], y) : max(x[j], y);
        }
      } else {
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const int p = j ^ stride;
          if (p > j) {
            const bool up = ((lane * E + j) & size) == 0;
            const int a = x[j], b = x[p];
            if ((a > b) == up) { x[j] = b; x[p] = a; }
          }
        }
      }
    }
  }
  int prev = __shfl_up_sync(0xffffffffu, x[E - 1], 1);
  if (lane == 0) prev = INT_MIN;
  int cnt = 0;
  bool keep[E];
#pragma unroll
  for (int j = 0; j < E; ++j) {
    keep[j] = x[j] != INT_MAX && x[j] != (j ? x[j - 1] : prev);
    cnt += keep[j];
  }
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int pos = incl - cnt;
#pragma unroll
  for (int j = 0; j < E; ++j)
    if (keep[j]) out[pos++] = x[j];
  return __shfl_sync(0xffffffffu, incl, 31);
}

// Sort buf[0..n) ascending (bitonic over the next power of two, INT_MAX pad)
// then write the distinct values to out; returns the distinct count.
__device__ int block_sort_unique(int* buf, int n, int* out, int* scan) {
  if (n <= 256) {  // one warp, register network
    __shared__ int s_total;
    if (warp_id() == 0) {
      const int t = warp_sort_unique<8>(buf, n, out);
      if (lane_id() == 0) s_total = t;
    }
    __syncthreads();
    const int t = s_total;
    __syncthreads();
    return t;
  }
  int P = 1;
  while (P < n) P <<= 1;
  for (int i = n + threadIdx.x; i < P; i += blockDim.x) buf[i] = INT_MAX;
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < (P >> 1); i += blockDim.x) {
        const int a = 2 * i - (i & (stride - 1));
        const int b = a + stride;
        const bool up = (a & size) == 0;
        const int x = buf[a], y = buf[b];
        if ((x > y) == up) { buf[a] = y; buf[b] = x; }
      }
      __syncthreads();
    }
  }
  const int per = (P + blockDim.x - 1) / blockDim.x;
  const int s = threadIdx.x * per;
  const int e = min(s + per, P);
  int keep = 0;
  for (int i = s; i < e; ++i) {
    const int v = buf[i];
    keep += (v != INT_MAX) && (i == 0 || buf[i - 1] != v);
  }
  int total;
  int pos = block_exclusive_scan(keep, scan, &total);
  for (int i = s; i < e; ++i) {
    const int v = buf[i];
    if ((v != INT_MAX) && (i == 0 || buf[i - 1] != v)) out[pos++] = v;
  }
  __syncthreads();
  return total;
}

// exclusive scan of in[0..n) into out[0..n], out[n] = total (n small)
__device__ int block_scan_small(const int* in, int* out, int n, int* scan) {
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int s = threadIdx.x * per;
  const int e = min(s + per, n);
  int sum = 0;
  for (int i = s; i < e; ++i) sum += in[i];
  int total;
  int pos = block_exclusive_scan(sum, scan, &total);
  for (int i = s; i < e; ++i) { out[i] = pos; pos += in[i]; }
  if (threadIdx.x == 0) out[n] = total;
  __syncthreads();
  return total;
}

__device__ __forceinline__ bool contains(const int* a, int n, int x) {
  const int p = lower_bound(a, n, x);
  return p < n && a[p] == x;
}

// Sorted-unique of buf[0..n) for n <= blockDim.x by ranking: thread i keeps
// buf[i] if no equal value precedes it, then places it at the number of
// distinct smaller values.  Two O(n) passes, 2 barriers, no sorting network.
// `flag` needs n ints of scratch.
__device__ int rank_sort_unique(const int* buf, int n, int* out, int* flag, int* s_total) {
  const int i = threadIdx.x;
  int x = 0;
  bool first = false;
  if (i < n) {
    x = buf[i];
    first = true;
    for (int j = 0; j < i; ++j) first &= buf[j] != x;
    flag[i] = first;
  }
  if (i == 0) *s_total = 0;
  __syncthreads();
  if (first) {
    int pos = 0;
    for (int j = 0; j < n; ++j) pos += flag[j] && buf[j] < x;
    out[pos] = x;
    atomicAdd(s_total, 1);
  }
  __syncthreads();
  const int t = *s_total;
  __syncthreads();
  return t;
}

// out = sorted union of two sorted-unique lists A[0..a) and B[0..b) by merge
// positions (binary searches), B's members of A dropped; b <= blockDim.x.
// `flag` needs b+1 ints of scratch.  Returns the union size.
__device__ int union_sorted(const int* A, int a, const int* B, int b, int* out, int* flag,
                            int* scan) {
  // flag[j] = 1 if B[j] is not in A; exclusive prefix over B
  const int i = threadIdx.x;
  int nd = 0;
  if (i < b) nd = contains(A, a, B[i]) ? 0 : 1;
  int tot_b;
  const int pre = block_exclusive_scan(nd, scan, &tot_b);  // all threads participate
  if (i < b) flag[i] = pre;
  if (i == 0) flag[b] = tot_b;
  __syncthreads();
  for (int k = i; k < a; k += blockDim.x) {
    const int x = A[k];
    out[k + flag[lower_bound(B, b, x)]] = x;
  }
  if (i < b && nd) out[pre + lower_bound(A, a, B[i])] = B[i];
  __syncthreads();
  return a + tot_b;
}

// ---------------------------------------------------------------- build kernel

#ifdef HG_BUILD_PROFILE
__device__ long long g_phase[4096][16];
#define HG_PHASE(i) \
  if (threadIdx.x == 0 && r < 4096) g_phase[r][(i)] = clock64();
#else
#define HG_PHASE(i)
#endif

// One root's micrograph (CTA-wide); r indexes roots / iter_state / ws.
__device__ __forceinline__ void build_root(
    const int r, const CsrView& g,
    int64_t n_vertices, const int64_t* __restrict__ roots, const uint64_t* __restrict__ iter_state,
    int roots_per_state, const MgCarve& c, int32_t* __restrict__ ws, int* err,
    const int32_t* __restrict__ n_roots_dev, int per_batch) {
  extern __shared__ __align__(16) int sm[];
  const int L = c.L;
  // beyond the device count of its batch: an empty micrograph
  if (n_roots_dev && r % per_batch >= n_roots_dev[r / per_batch]) {
    int32_t* w = ws + (size_t)r * c.ws_root_ints;
    if (threadIdx.x <= 2 * L) w[c.ws_cnt + threadIdx.x] = 0;
    return;
  }
  int* scan = sm + c.sm_scan;
  __shared__ int warp_ctr[kBuildWarps + 1];
  __shared__ uint64_t tslots[kBuildWarps + 1];
  uint64_t* cand_base = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(sm) + c.cand_byte_off);

  int64_t root = roots[r];
  if (root < 0 || root >= n_vertices) {
    raise_flag(err, HG_ERANGE);
    root = 0;
  }
  // roots_per_state == 0: iter_state already holds one final stream key per root
  const uint64_t key = roots_per_state > 0
                           ? mix64(iter_state[r / roots_per_state] ^ (uint64_t)root)
                           : iter_state[r];
  __shared__ int nlay[HG_MAX_LAYERS + 1], nneed[HG_MAX_LAYERS + 1], ntot[HG_MAX_LAYERS + 1];
  if (threadIdx.x == 0) {
    sm[c.sm_lay[L]] = (int)root;
    nlay[L] = 1;
  }
  __syncthreads();
  HG_PHASE(0);

  for (int h = 1; h <= L; ++h) {
    const int k = L - h;
    const int F = nlay[k + 1];
    const int fo = c.fanout[h - 1];
    const int mean = c.mean[h - 1];
    const int* front = sm + c.sm_lay[k + 1];
    int* cnt = sm + c.sm_cnt[h];
    int* off = sm + c.sm_off[h];
    int* degs = sm + c.sm_deg[h];
    int* flat = sm + c.sm_flat[h];
    const uint64_t state = mix64(mix64(key) ^ (uint64_t)h);  // chain(key, hop)
    for (int i = threadIdx.x; i < F; i += blockDim.x) {
      int64_t lo;
      const int pk = csr_row(g, front[i], &lo);
      const int d = row_deg(pk);
      degs[i] = pk;
      cnt[i] = d <= fo ? d : fo;
    }
    __syncthreads();
    const int T = block_scan_small(cnt, off, F, scan);
    HG_PHASE(1 + 4 * (h - 1));
    // small tasks: one warp each
    for (int i = warp_id(); i < F; i += kBuildWarps) {
      const int d = row_deg(degs[i]);
      if (d > kBigTask) continue;
      const int v = front[i];
      int64_t lo;
      csr_row(g, v, &lo);
      const int32_t* targets = g.tgt[row_shard(degs[i])];
      int32_t* out = flat + off[i];
      if (d <= fo) {
        for (int j = lane_id(); j < d; j += 32) out[j] = targets[lo + j];
      } else {
        team_select<WarpTeam>(targets, lo, d, fo, mean, mix64(state ^ (uint64_t)v), out,
                              cand_base + (size_t)warp_id() * c.cand_cap, c.cand_cap,
                              warp_ctr + warp_id(), tslots + warp_id(), err);
      }
    }
    __syncthreads();
    HG_PHASE(2 + 4 * (h - 1));
    // hubs: the whole CTA
    for (int i = 0; i < F; ++i) {
      const int d = row_deg(degs[i]);
      if (d <= kBigTask) continue;
      const int v = front[i];
      int64_t lo;
      csr_row(g, v, &lo);
      team_select<BlockTeam>(g.tgt[row_shard(degs[i])], lo, d, fo, mean, mix64(state ^ (uint64_t)v),
                             flat + off[i], cand_base + (size_t)kBuildWarps * c.cand_cap,
                             c.cand_cap, warp_ctr + kBuildWarps, tslots + kBuildWarps, err);
    }
    __syncthreads();
    HG_PHASE(3 + 4 * (h - 1));
    int* sb = sm + c.sm_sort;
    int u;
    if (T <= (int)blockDim.x) {
      __shared__ int s_tot;
      u = rank_sort_unique(flat, T, sm + c.sm_lay[k], sb, &s_tot);
    } else {
      for (int i = threadIdx.x; i < T; i += blockDim.x) sb[i] = flat[i];
      __syncthreads();
      u = block_sort_unique(sb, T, sm + c.sm_lay[k], scan);
    }
    if (threadIdx.x == 0) { nlay[k] = u; ntot[h] = T; }
    __syncthreads();
    HG_PHASE(4 + 4 * (h - 1));
  }

  // need-chain sets: need[L] = [root], need[k] = union(layers[k], need[k+1])
  if (threadIdx.x == 0) { sm[c.sm_need[L]] = sm[c.sm_lay[L]]; nneed[L] = 1; }
  __syncthreads();
  for (int k = L - 1; k >= 0; --k) {
    int* sb = sm + c.sm_sort;
    const int a = nlay[k], b = nneed[k + 1];
    int u;
    if (b < (int)blockDim.x) {  // merge of two sorted-unique lists
      u = union_sorted(sm + c.sm_lay[k], a, sm + c.sm_need[k + 1], b, sm + c.sm_need[k], sb, scan);
    } else {
      for (int i = threadIdx.x; i < a; i += blockDim.x) sb[i] = sm[c.sm_lay[k] + i];
      for (int i = threadIdx.x; i < b; i += blockDim.x) sb[a + i] = sm[c.sm_need[k + 1] + i];
      __syncthreads();
      u = block_sort_unique(sb, a + b, sm + c.sm_need[k], scan);
    }
    if (threadIdx.x == 0) nneed[k] = u;
    __syncthreads();
  }

  HG_PHASE(13);
  // padded per-root outputs
  int32_t* w = ws + (size_t)r * c.ws_root_ints;
  for (int k = 0; k <= L; ++k) {
    const int* need = sm + c.sm_need[k];
    const int* lay = sm + c.sm_lay[k];
    for (int a = threadIdx.x; a < nneed[k]; a += blockDim.x) {
      const int uv = need[a];
      w[c.ws_need[k] + a] = uv;
      w[c.ws_inl[k] + a] = contains(lay, nlay[k], uv) ? 1 : 0;
    }
  }
  for (int k = 1; k <= L; ++k) {
    const int hp = L - k + 1;  // hop whose frontier is layers[k]
    const int* need = sm + c.sm_need[k];
    const int* prev = sm + c.sm_need[k - 1];
    const int* lay = sm + c.sm_lay[k];
    const int* off = sm + c.sm_off[hp];
    const int* flat = sm + c.sm_flat[hp];
    const int nk = nneed[k], np = nneed[k - 1], nl = nlay[k];
    for (int a = threadIdx.x; a < nk; a += blockDim.x) {
      const int uv = need[a];
      w[c.ws_self[k] + a] = lower_bound(prev, np, uv);
      w[c.ws_rowoff[k] + a] = off[lower_bound(lay, nl, uv)];
    }
    if (threadIdx.x == 0) w[c.ws_rowoff[k] + nk] = ntot[hp];
    for (int t = threadIdx.x; t < ntot[hp]; t += blockDim.x)
      w[c.ws_nbr[k] + t] = lower_bound(prev, np, flat[t]);
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k <= L; ++k) w[c.ws_cnt + k] = nneed[k];
    for (int k = 1; k <= L; ++k) w[c.ws_cnt + L + k] = ntot[L - k + 1];
  }
  HG_PHASE(14);
}

// CTA per root, or (gridDim.x < n_roots) a persistent grid striding over the
// roots: capping the resident build CTAs per SM leaves registers for the
// training kernels that run beside the build in the graph loop.
__global__ void __launch_bounds__(kBuildThreads, HG_BUILD_MINB)
k_mg_build(const CsrView g, int64_t n_vertices, const int64_t* __restrict__ roots, int n_roots,
           const uint64_t* __restrict__ iter_state, int roots_per_state, MgCarve c,
           int32_t* __restrict__ ws, int* err, const int32_t* __restrict__ n_roots_dev,
           int per_batch) {
  for (int r = blockIdx.x; r < n_roots; r += gridDim.x) {
    build_root(r, g, n_vertices, roots, iter_state, roots_per_state, c, ws, err,
               n_roots_dev, per_batch);
    __syncthreads();  // shared tiles are reused by the next root
  }
}

// ---------------------------------------------------------------- warp-per-root build (L = 2)
//
// Two-layer micrographs whose layers fit one warp (hop-1 fanout f1 <= 31,
// f1 * f2 <= 256 hop-2 pairs): the configuration the benchmark trains.  A CTA
// of 8 warps builds 8 roots, one warp each, with 3 block barriers per 8 roots
// (the CTA-per-root kernel above pays ~20 per root, and its 8 warps wait at
// every one for the slowest draw):
//   P1  warp: root, key, hop-1 draw (threshold select) -- a hub root (degree
//       > kWarpMaxDeg) is queued and drawn by the whole CTA;
//       warp: sort-unique layer 1, row starts / degrees / pair offsets;
//   P2  the CTA's hop-2 draws (<= 8 x 31 frontier vertices) as one task list
//       pulled dynamically by the 8 warps (shared counter), so a root with
//       heavy frontier vertices does not hold the other seven back; hub
//       vertices are queued and drawn by the whole CTA afterwards;
//   P3  warp: sort-unique layer 0 in registers, need sets by merge positions,
//       in-layer flags, self / neighbour positions by binary search, the
//       per-root workspace rows (same layout as build_root: k_mg_scan and
//       k_mg_finalize are shared).
// Bit-exact with build_root (tests/test_sampler_gpu.py compares both kernels
// and the oracle).
constexpr int kW2Roots = kBuildWarps;   // roots per CTA (one per warp)
constexpr int kW2F1 = 31;               // max hop-1 fanout (need[1] <= 32 = one lane each)
constexpr int kW2P2 = 256;              // max hop-2 pairs per root (warp_sort_unique<8>)
constexpr int kWarpMaxDeg = 1024;       // larger rows are drawn by the whole CTA

struct W2Slot {
  uint64_t st1, st2;      // hop-1 / hop-2 states chain(key, 1), chain(key, 2)
  int64_t lo1[32];        // CSR start of each layer-1 vertex
  int flat1[32];          // hop-1 draws, slot order
  int lay1[32];           // layers[1] (sorted unique)
  int deg1[32];
  int off1[33];           // hop-2 pair offsets per layer-1 vertex
  int need1[32];
  int mflag[33];          // merge prefix of need1 entries absent from layer 0
  int flat2[kW2P2];       // hop-2 draws, frontier order
  int lay0[kW2P2];        // layers[0]
  int need0[kW2P2 + 33];  // need[0] = layers[0] U need[1]
  int root, n_flat1, n_flat2, pad;
};

bool w2_eligible(const MgCarve& c) {
  return c.L == 2 && c.fanout[0] <= kW2F1 && c.cap_lay[0] <= kW2P2;
}

size_t w2_smem(const MgCarve& c) {
  return sizeof(W2Slot) * kW2Roots + (size_t)(kW2Roots + 1) * c.cand_cap * sizeof(uint64_t);
}

__device__ __forceinline__ int warp_incl_scan(int x) {
  const int lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

__global__ void __launch_bounds__(kBuildThreads, 4)
k_mg_build_w2(const CsrView g, int64_t n_vertices, const int64_t* __restrict__ roots, int n_roots,
              const uint64_t* __restrict__ iter_state, int roots_per_state, MgCarve c,
              int32_t* __restrict__ ws, int* err, const int32_t* __restrict__ n_roots_dev,
              int per_batch) {
  extern __shared__ __align__(16) unsigned char w2raw[];
  W2Slot* slots = reinterpret_cast<W2Slot*>(w2raw);
  uint64_t* cand_base = reinterpret_cast<uint64_t*>(w2raw + sizeof(W2Slot) * kW2Roots);
  __shared__ int nl1s[kW2Roots], hub1_list[kW2Roots], hub_list[kW2Roots * 32];
  __shared__ int hub1_cnt, hub_cnt, task_ctr;
  __shared__ int warp_ctr[kW2Roots + 1];
  __shared__ uint64_t tslots[kW2Roots + 1];
  const int w = warp_id(), lane = lane_id();
  const unsigned full = 0xffffffffu;
  W2Slot& S = slots[w];
  const int f1 = c.fanout[0], f2 = c.fanout[1], m1 = c.mean[0], m2 = c.mean[1];
  const int cap = c.cand_cap;
  uint64_t* my_cand = cand_base + (size_t)w * cap;
  uint64_t* cta_cand = cand_base + (size_t)kW2Roots * cap;
  const int groups = (n_roots + kW2Roots - 1) / kW2Roots;
  for (int gi = blockIdx.x; gi < groups; gi += gridDim.x) {
    const int r = gi * kW2Roots + w;
    if (threadIdx.x == 0) { hub1_cnt = 0; hub_cnt = 0; task_ctr = 0; }
    __syncthreads();  // counters reset; the previous group's slots are free
    const bool in_range = r < n_roots;
    const bool empty = in_range && n_roots_dev && r % per_batch >= n_roots_dev[r / per_batch];
    const bool live = in_range && !empty;
    int32_t* wr = ws + (size_t)r * c.ws_root_ints;
    if (empty && lane <= 4) wr[c.ws_cnt + lane] = 0;  // an empty micrograph (2L+1 counts)
    // ---- P1: hop-1 draw of the root
    if (live) {
      int64_t root = roots[r];
      if (root < 0 || root >= n_vertices) {
        if (lane == 0) raise_flag(err, HG_ERANGE);
        root = 0;
      }
      // roots_per_state == 0: iter_state already holds one final stream key per root
      const uint64_t key = roots_per_state > 0
                               ? mix64(iter_state[r / roots_per_state] ^ (uint64_t)root)
                               : iter_state[r];
      const uint64_t k1 = mix64(key);
      const uint64_t st1 = mix64(k1 ^ 1ull);
      int64_t lo;
      const int pk = csr_row(g, root, &lo);
      const int d = row_deg(pk);
      const int32_t* targets = g.tgt[row_shard(pk)];
      if (lane == 0) {
        S.st1 = st1;
        S.st2 = mix64(k1 ^ 2ull);
        S.root = (int)root;
        S.n_flat1 = d <= f1 ? d : f1;
      }
      if (d <= f1) {
        for (int j = lane; j < d; j += 32) S.flat1[j] = targets[lo + j];
      } else if (d <= kWarpMaxDeg) {
        team_select<WarpTeam>(targets, lo, d, f1, m1, mix64(st1 ^ (uint64_t)root), S.flat1,
                              my_cand, cap, warp_ctr + w, tslots + w, err);
      } else if (lane == 0) {
        hub1_list[atomicAdd(&hub1_cnt, 1)] = w;
      }
    }
    __syncthreads();
    const int nh1 = hub1_cnt;
    for (int q = 0; q < nh1; ++q) {  // hub roots: the whole CTA draws
      W2Slot& H = slots[hub1_list[q]];
      const int64_t rt = H.root;
      int64_t lo;
      const int pk = csr_row(g, rt, &lo);
      team_select<BlockTeam>(g.tgt[row_shard(pk)], lo, row_deg(pk), f1, m1,
                             mix64(H.st1 ^ (uint64_t)rt), H.flat1, cta_cand, cap,
                             warp_ctr + kW2Roots, tslots + kW2Roots, err);
    }
    // layer 1, its rows and the hop-2 pair offsets
    int nl1 = 0;
    if (live) {
      __syncwarp();
      nl1 = warp_sort_unique<1>(S.flat1, S.n_flat1, S.lay1);
      __syncwarp();
      int cnt = 0;
      if (lane < nl1) {
        int64_t lo;
        const int pk = csr_row(g, S.lay1[lane], &lo);
        const int d = row_deg(pk);
        S.lo1[lane] = lo;
        S.deg1[lane] = pk;
        cnt = d <= f2 ? d : f2;
      }
      const int incl = warp_incl_scan(cnt);
      S.off1[lane] = incl - cnt;
      if (lane == 31) { S.off1[32] = incl; S.n_flat2 = incl; }
    }
    if (lane == 0) nl1s[w] = nl1;
    __syncthreads();
    // ---- P2: the CTA's hop-2 draws, pulled dynamically by its warps
    const int nb = lane < kW2Roots ? nl1s[lane] : 0;
    const int incl_b = warp_incl_scan(nb);
    const int excl_b = incl_b - nb;
    const int n_tasks = __shfl_sync(full, incl_b, kW2Roots - 1);
    for (;;) {
      int t = 0;
      if (lane == 0) t = atomicAdd(&task_ctr, 1);
      t = __shfl_sync(full, t, 0);
      if (t >= n_tasks) break;
      const unsigned bm = __ballot_sync(full, lane < kW2Roots && excl_b <= t);
      const int ow = 31 - __clz(bm);
      const int i = t - __shfl_sync(full, excl_b, ow);
      W2Slot& Q = slots[ow];
      const int d = row_deg(Q.deg1[i]);
      const int32_t* targets = g.tgt[row_shard(Q.deg1[i])];
      int32_t* out = Q.flat2 + Q.off1[i];
      if (d <= f2) {
        const int64_t lo = Q.lo1[i];
        for (int j = lane; j < d; j += 32) out[j] = targets[lo + j];
      } else if (d <= kWarpMaxDeg) {
        team_select<WarpTeam>(targets, Q.lo1[i], d, f2, m2,
                              mix64(Q.st2 ^ (uint64_t)Q.lay1[i]), out, my_cand, cap,
                              warp_ctr + w, tslots + w, err);
      } else if (lane == 0) {
        hub_list[atomicAdd(&hub_cnt, 1)] = t;
      }
    }
    __syncthreads();
    const int nh = hub_cnt;
    for (int q = 0; q < nh; ++q) {  // hub frontier vertices: the whole CTA draws
      const int t = hub_list[q];
      int ow = 0, base = 0;
      while (base + nl1s[ow] <= t) base += nl1s[ow++];
      W2Slot& Q = slots[ow];
      const int i = t - base;
      team_select<BlockTeam>(g.tgt[row_shard(Q.deg1[i])], Q.lo1[i], row_deg(Q.deg1[i]), f2, m2,
                             mix64(Q.st2 ^ (uint64_t)Q.lay1[i]), Q.flat2 + Q.off1[i], cta_cand,
                             cap, warp_ctr + kW2Roots, tslots + kW2Roots, err);
    }
    if (!live) continue;
    // ---- P3: layer 0, need sets, plan, workspace rows (warp only)
    __syncwarp();
    const int T = S.n_flat2, T1 = S.n_flat1;
    const int nl0 = warp_sort_unique<8>(S.flat2, T, S.lay0);
    const int rt = S.root;
    // need[1] = layers[1] U {root}
    const int p = lower_bound(S.lay1, nl1, rt);
    const bool rin = p < nl1 && S.lay1[p] == rt;
    const int nn1 = nl1 + (rin ? 0 : 1);
    if (lane < nn1) S.need1[lane] = rin ? S.lay1[lane] : (lane < p ? S.lay1[lane] : lane == p ? rt : S.lay1[lane - 1]);
    __syncwarp();
    // need[0] = layers[0] U need[1] by merge positions (need[1] entries not in layers[0] inserted)
    int nd = 0;
    if (lane < nn1) {
      const int x = S.need1[lane];
      const int q = lower_bound(S.lay0, nl0, x);
      nd = (q < nl0 && S.lay0[q] == x) ? 0 : 1;
    }
    const int incl_nd = warp_incl_scan(nd);
    if (lane < nn1) S.mflag[lane] = incl_nd - nd;
    const int tb = __shfl_sync(full, incl_nd, 31);
    if (lane == 0) S.mflag[nn1] = tb;
    __syncwarp();
    const int nn0 = nl0 + tb;
    int32_t* need0_ws = wr + c.ws_need[0];
    int32_t* inl0_ws = wr + c.ws_inl[0];
    for (int a = lane; a < nl0; a += 32) {
      const int x = S.lay0[a];
      const int pos = a + S.mflag[lower_bound(S.need1, nn1, x)];
      S.need0[pos] = x;
      need0_ws[pos] = x;
      inl0_ws[pos] = 1;
    }
    if (nd) {
      const int x = S.need1[lane];
      const int pos = S.mflag[lane] + lower_bound(S.lay0, nl0, x);
      S.need0[pos] = x;
      need0_ws[pos] = x;
      inl0_ws[pos] = 0;
    }
    __syncwarp();
    // layer 1 rows: need[1], in-layer, self positions in need[0], pair ranges
    if (lane < nn1) {
      const int x = S.need1[lane];
      wr[c.ws_need[1] + lane] = x;
      wr[c.ws_inl[1] + lane] = (rin || lane != p) ? 1 : 0;
      wr[c.ws_self[1] + lane] = lower_bound(S.need0, nn0, x);
      wr[c.ws_rowoff[1] + lane] = S.off1[lower_bound(S.lay1, nl1, x)];
    }
    if (lane == 0) {
      wr[c.ws_rowoff[1] + nn1] = T;
      // layer 2 = [root]: need, in-layer, self position in need[1], hop-1 pair range
      wr[c.ws_need[2]] = rt;
      wr[c.ws_inl[2]] = 1;
      wr[c.ws_self[2]] = p;  // lower_bound(need[1], root)
      wr[c.ws_rowoff[2]] = 0;
      wr[c.ws_rowoff[2] + 1] = T1;
      wr[c.ws_cnt + 0] = nn0;
      wr[c.ws_cnt + 1] = nn1;
      wr[c.ws_cnt + 2] = 1;
      wr[c.ws_cnt + 3] = T;   // pairs of layer 1 (hop 2)
      wr[c.ws_cnt + 4] = T1;  // pairs of layer 2 (hop 1)
    }
    for (int t = lane; t < T; t += 32) wr[c.ws_nbr[1] + t] = lower_bound(S.need0, nn0, S.flat2[t]);
    if (lane < T1) wr[c.ws_nbr[2] + lane] = lower_bound(S.need1, nn1, S.flat1[lane]);
  }
}

// Exclusive scans of the per-root counts (one CTA).  cols 0..L: need sizes,
// cols L+1..2L: pair counts of layers 1..L.  Every count is loaded up front
// (one strided gather in flight per thread and column) so the per-column
// scans run from registers and shared memory only.
constexpr int kScanCols = 2 * HG_MAX_LAYERS + 1;
constexpr int kScanPer = 2;  // roots per thread held in registers per 2048-root tile

__global__ void __launch_bounds__(1024)
k_mg_scan(const int32_t* __restrict__ ws, int n_roots, MgCarve c, MgOuts outs) {
  // CTA b scans batch b: roots [b * n_roots, (b + 1) * n_roots) of the workspace
  const hg_mg_batch& out = outs.b[blockIdx.x];
  ws += (size_t)blockIdx.x * n_roots * c.ws_root_ints;
  __shared__ int scan[40];
  __shared__ int32_t* dsts[kScanCols];
  const int L = c.L, ncol = 2 * L + 1;
  if (threadIdx.x < ncol)
    dsts[threadIdx.x] = threadIdx.x <= L ? out.need_off[threadIdx.x] : out.pair_off[threadIdx.x - L];
  __syncthreads();
  int carry[kScanCols];
#pragma unroll
  for (int col = 0; col < kScanCols; ++col) carry[col] = 0;
  for (int base = 0; base < n_roots; base += (int)blockDim.x * kScanPer) {  // tiles of 2048 roots
    const int s0 = base + threadIdx.x * kScanPer;
    int v[kScanCols][kScanPer];
#pragma unroll
    for (int col = 0; col < kScanCols; ++col)
#pragma unroll
      for (int j = 0; j < kScanPer; ++j)
        v[col][j] = (col < ncol && s0 + j < n_roots)
                        ? ws[(size_t)(s0 + j) * c.ws_root_ints + c.ws_cnt + col] : 0;
#pragma unroll
    for (int col = 0; col < kScanCols; ++col) {
      if (col >= ncol) continue;  // uniform across the block
      int32_t* dst = dsts[col];
      int sum = 0;
#pragma unroll
      for (int j = 0; j < kScanPer; ++j) sum += v[col][j];
      int total;
      int pos = carry[col] + block_exclusive_scan(sum, scan, &total);
#pragma unroll
      for (int j = 0; j < kScanPer; ++j) {
        if (s0 + j < n_roots) dst[s0 + j] = pos;
        pos += v[col][j];
      }
      carry[col] += total;
    }
  }
  if (threadIdx.x == 0) {
#pragma unroll
    for (int col = 0; col < kScanCols; ++col) {
      if (col >= ncol) continue;
      int32_t* dst = dsts[col];
      dst[n_roots] = carry[col];
      out.totals[col] = carry[col];
    }
    // pair totals close the CSR-by-destination offsets of each layer
    for (int k = 1; k <= L; ++k) out.nbr_off[k][out.totals[k]] = out.totals[L + k];
  }
}

__global__ void __launch_bounds__(256)
k_mg_finalize(const int32_t* __restrict__ ws, int n_roots, int total, MgCarve c, MgOuts outs) {
  // warp per root of the whole group; root g belongs to batch g / n_roots
  const int gid = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (gid >= total) return;
  const int lane = threadIdx.x & 31;
  const int r = gid % n_roots;
  const hg_mg_batch& out = outs.b[gid / n_roots];
  const int L = c.L;
  const int32_t* w = ws + (size_t)gid * c.ws_root_ints;
  for (int k = 0; k <= L; ++k) {
    const int base = out.need_off[k][r];
    const int nk = w[c.ws_cnt + k];
    for (int a = lane; a < nk; a += 32) {
      out.need_ids[k][base + a] = w[c.ws_need[k] + a];
      out.in_layer[k][base + a] = (int8_t)w[c.ws_inl[k] + a];
    }
    if (k == 0) continue;
    const int pbase = out.pair_off[k][r];
    const int prev_base = out.need_off[k - 1][r];
    for (int a = lane; a < nk; a += 32) {
      out.self_pos[k][base + a] = prev_base + w[c.ws_self[k] + a];
      out.nbr_off[k][base + a] = pbase + w[c.ws_rowoff[k] + a];
      if (k == 1 && out.self_vid1) out.self_vid1[base + a] = w[c.ws_need[1] + a];
    }
    const int pk = w[c.ws_cnt + L + k];
    for (int t = lane; t < pk; t += 32) {
      const int q = w[c.ws_nbr[k] + t];
      out.nbr_idx[k][pbase + t] = prev_base + q;
      if (k == 1 && out.nbr_vid1) out.nbr_vid1[pbase + t] = w[c.ws_need[0] + q];
    }
  }
}

// ---------------------------------------------------------------- drop-in frontier

__global__ void k_frontier_counts(const int64_t* __restrict__ offsets, int64_t n_vertices,
                                  const int64_t* __restrict__ frontier, int64_t f, int fo,
                                  int64_t* counts, int* err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= f) return;
  int64_t v = frontier[i];
  if (v < 0 || v >= n_vertices) { raise_flag(err, HG_ERANGE); counts[i] = 0; return; }
  const int64_t d = offsets[v + 1] - offsets[v];
  counts[i] = d <= fo ? d : fo;
}

__global__ void __launch_bounds__(256)
k_frontier_fill(const int64_t* __restrict__ offsets, const int32_t* __restrict__ targets,
                int64_t n_vertices, const int64_t* __restrict__ frontier, int64_t f, int fo,
                int mean, uint64_t state, const int64_t* __restrict__ pos,
                int64_t* __restrict__ flat, int cand_cap, int* err) {
  extern __shared__ __align__(16) unsigned char smraw[];
  uint64_t* cand = reinterpret_cast<uint64_t*>(smraw) + (size_t)warp_id() * cand_cap;
  int32_t* obuf = reinterpret_cast<int32_t*>(reinterpret_cast<uint64_t*>(smraw) +
                                             (size_t)(blockDim.x / 32) * cand_cap) +
                  (size_t)warp_id() * fo;
  __shared__ int ctr[8];
  __shared__ uint64_t tsh[8];
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + warp_id();
  if (i >= f) return;
  const int64_t v = frontier[i];
  if (v < 0 || v >= n_vertices) return;
  const int64_t lo = offsets[v];
  const int d = (int)(offsets[v + 1] - lo);
  int64_t* out = flat + pos[i];
  if (d <= fo) {
    for (int j = lane_id(); j < d; j += 32) out[j] = targets[lo + j];
    return;
  }
  team_select<WarpTeam>(targets, lo, d, fo, mean, mix64(state ^ (uint64_t)v), obuf, cand,
                        cand_cap, ctr + warp_id(), tsh + warp_id(), err);
  for (int j = lane_id(); j < fo; j += 32) out[j] = obuf[j];
}

}  // namespace hg

using namespace hg;

extern "C" int hg_mg_plan_layout(int32_t n_layers, const int32_t* fanout, hg_mg_layout* out) {
  MgCarve c;
  int st = make_carve(n_layers, fanout, &c);
  if (st) return st;
  *out = hg_mg_layout{};
  out->n_layers = n_layers;
  for (int h = 0; h < n_layers; ++h) out->fanout[h] = fanout[h];
  for (int k = 0; k <= n_layers; ++k) {
    out->cap_lay[k] = c.cap_lay[k];
    out->cap_need[k] = c.cap_need[k];
  }
  out->cand_cap = c.cand_cap;
  out->sort_cap = c.sort_cap;
  out->smem_bytes = c.smem_bytes;
  out->ws_root_ints = c.ws_root_ints;
  return HG_OK;
}

extern "C" int hg_mg_build(const int64_t* offsets, const int32_t* targets, int64_t n_vertices,
                           const int64_t* roots, int32_t n_roots, const uint64_t* iter_state,
                           int32_t roots_per_state, const hg_mg_layout* layout, int32_t* ws,
                           hg_mg_batch* out, int* err_flag, void* stream) {
  return hg_mg_build_n(offsets, targets, n_vertices, roots, n_roots, nullptr, iter_state,
                       roots_per_state, layout, ws, out, err_flag, stream);
}

// 0: the warp-per-root build wherever it applies (w2_eligible), else the CTA-per-root
// build; 1: always the CTA-per-root build (hg_mg_build_mode, used by the parity tests
// that compare the two kernels)
static int g_build_mode = 0;

static CsrView single_view(const int64_t* offsets, const int32_t* targets) {
  CsrView g{};
  g.S = 1;
  g.off[0] = offsets;
  g.tgt[0] = targets;
  return g;
}

static int view_from(const hg_csr_shards* sh, int64_t n_vertices, CsrView* g) {
  if (!sh || sh->n_shards < 1 || sh->n_shards > HG_MAX_SHARDS)
    return hg_fail(HG_ECONFIG, "csr shards: n_shards must be 1..%d", HG_MAX_SHARDS);
  *g = CsrView{};
  g->S = sh->n_shards;
  for (int h = 0; h < g->S; ++h) {
    if (!sh->offsets[h] || !sh->targets[h]) return hg_fail(HG_ECONFIG, "csr shard %d missing", h);
    g->off[h] = sh->offsets[h];
    g->tgt[h] = sh->targets[h];
  }
  g->home_of = sh->home_of;
  g->row_of = sh->row_of;
  if (g->S > 1 && !g->home_of) {
    if (sh->vstart[0] != 0 || sh->vstart[g->S] != n_vertices)
      return hg_fail(HG_ECONFIG, "csr shards: vstart must cover [0, n_vertices)");
    for (int h = 0; h <= g->S; ++h) g->vstart[h] = sh->vstart[h];
  } else if (g->S > 1 && !g->row_of) {
    return hg_fail(HG_ECONFIG, "csr shards: home_of needs row_of");
  }
  return HG_OK;
}

static int build_group(const CsrView& g, int64_t n_vertices,
                       const int64_t* roots, int32_t n_roots, int32_t n_batches,
                       const int32_t* n_roots_dev, const uint64_t* iter_state,
                       int32_t roots_per_state, const hg_mg_layout* layout, int32_t* ws,
                       const hg_mg_batch* outs, int* err_flag, int ctas_per_sm, void* stream) {
  if (n_roots < 0 || roots_per_state < 0) return hg_fail(HG_ERANGE, "bad root count");
  if (n_batches < 1 || n_batches > HG_MAX_GROUP) return hg_fail(HG_ERANGE, "bad batch count %d", n_batches);
  if ((int64_t)n_roots * n_batches > INT32_MAX) return hg_fail(HG_ERANGE, "group too large");
  MgCarve c;
  int st = make_carve(layout->n_layers, layout->fanout, &c);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (n_roots == 0) return HG_OK;
  MgOuts o{};
  for (int b = 0; b < n_batches; ++b) o.b[b] = outs[b];
  HG_CUDA_TRY(cudaFuncSetAttribute(k_mg_build, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   c.smem_bytes));
  const int total = n_roots * n_batches;
  count_launch(3);
  prof_begin(PROF_BUILD, s);
  const int cps = ctas_per_sm;
  int grid = total;
  if (cps > 0) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    grid = std::min(total, nsm * cps);
  }
  if (w2_eligible(c) && g_build_mode != 1) {
    const int w2s = (int)w2_smem(c);
    HG_CUDA_TRY(cudaFuncSetAttribute(k_mg_build_w2, cudaFuncAttributeMaxDynamicSharedMemorySize, w2s));
    const int groups = (total + kW2Roots - 1) / kW2Roots;
    k_mg_build_w2<<<std::min(grid, groups), kBuildThreads, w2s, s>>>(
        g, n_vertices, roots, total, iter_state, roots_per_state, c, ws, err_flag,
        n_roots_dev, n_roots);
  } else {
    k_mg_build<<<grid, kBuildThreads, c.smem_bytes, s>>>(g, n_vertices, roots,
                                                          total, iter_state, roots_per_state, c,
                                                          ws, err_flag, n_roots_dev, n_roots);
  }
  HG_CUDA_TRY(cudaGetLastError());
  k_mg_scan<<<n_batches, 1024, 0, s>>>(ws, n_roots, c, o);
  HG_CUDA_TRY(cudaGetLastError());
  k_mg_finalize<<<(total + 7) / 8, 256, 0, s>>>(ws, n_roots, total, c, o);
  prof_end(PROF_BUILD, s);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_mg_build_n(const int64_t* offsets, const int32_t* targets, int64_t n_vertices,
                             const int64_t* roots, int32_t n_roots, const int32_t* n_roots_dev,
                             const uint64_t* iter_state, int32_t roots_per_state,
                             const hg_mg_layout* layout, int32_t* ws, hg_mg_batch* out,
                             int* err_flag, void* stream) {
  return build_group(single_view(offsets, targets), n_vertices, roots, n_roots, 1, n_roots_dev,
                     iter_state,
                     roots_per_state, layout, ws, out, err_flag, 0, stream);
}

extern "C" int hg_mg_build_group(const int64_t* offsets, const int32_t* targets,
                                 int64_t n_vertices, const int64_t* roots, int32_t n_roots,
                                 int32_t n_batches, const int32_t* n_roots_dev,
                                 const uint64_t* iter_state, int32_t roots_per_state,
                                 const hg_mg_layout* layout, int32_t* ws,
                                 const hg_mg_batch* outs, int* err_flag, int32_t ctas_per_sm,
                                 void* stream) {
  return build_group(single_view(offsets, targets), n_vertices, roots, n_roots, n_batches,
                     n_roots_dev, iter_state, roots_per_state, layout, ws, outs, err_flag,
                     ctas_per_sm, stream);
}

extern "C" int hg_mg_build_group_sharded(const hg_csr_shards* shards, int64_t n_vertices,
                                         const int64_t* roots, int32_t n_roots,
                                         int32_t n_batches, const int32_t* n_roots_dev,
                                         const uint64_t* iter_state, int32_t roots_per_state,
                                         const hg_mg_layout* layout, int32_t* ws,
                                         const hg_mg_batch* outs, int* err_flag,
                                         int32_t ctas_per_sm, void* stream) {
  CsrView g;
  int st = view_from(shards, n_vertices, &g);
  if (st) return st;
  return build_group(g, n_vertices, roots, n_roots, n_batches, n_roots_dev, iter_state,
                     roots_per_state, layout, ws, outs, err_flag, ctas_per_sm, stream);
}

extern "C" int hg_mg_build_mode(int32_t mode) {
  if (mode < 0 || mode > 1) return hg_fail(HG_ERANGE, "build mode must be 0 (auto) or 1 (CTA per root)");
  g_build_mode = mode;
  return HG_OK;
}

extern "C" int hg_sample_frontier(const int64_t* offsets, const int32_t* targets,
                                  int64_t n_vertices, const int64_t* frontier, int64_t n_frontier,
                                  int32_t fanout, uint64_t state, int64_t* counts_out,
                                  int64_t* flat_out, int64_t flat_cap, int64_t* flat_len_host,
                                  void* stream) {
  if (fanout < 1) return hg_fail(HG_ECONFIG, "fanout must be >= 1");
  cudaStream_t s = (cudaStream_t)stream;
  if (n_frontier == 0) { *flat_len_host = 0; return HG_OK; }
  int* err = nullptr;
  int64_t* pos = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  HG_CUDA_TRY(cudaMallocAsync((void**)&err, sizeof(int), s));
  HG_CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(int), s));
  HG_CUDA_TRY(cudaMallocAsync((void**)&pos, (n_frontier + 1) * sizeof(int64_t), s));
  k_frontier_counts<<<(unsigned)((n_frontier + 255) / 256), 256, 0, s>>>(
      offsets, n_vertices, frontier, n_frontier, fanout, counts_out, err);
  HG_CUDA_TRY(cudaGetLastError());
  HG_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts_out, pos, n_frontier, s));
  HG_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, s));
  HG_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts_out, pos, n_frontier, s));
  int64_t last_pos = 0, last_cnt = 0;
  HG_CUDA_TRY(cudaMemcpyAsync(&last_pos, pos + n_frontier - 1, 8, cudaMemcpyDeviceToHost, s));
  HG_CUDA_TRY(cudaMemcpyAsync(&last_cnt, counts_out + n_frontier - 1, 8, cudaMemcpyDeviceToHost, s));
  int herr = 0;
  HG_CUDA_TRY(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, s));
  HG_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t total = last_pos + last_cnt;
  *flat_len_host = total;
  int rc = HG_OK;
  if (herr) rc = hg_fail(herr, "frontier vertex out of range");
  else if (total > flat_cap) rc = hg_fail(HG_ECAPACITY, "flat_out holds %lld < %lld", (long long)flat_cap, (long long)total);
  if (rc == HG_OK) {
    const int mean = select_mean(fanout);
    int cap = pow2ceil(2 * mean < 64 ? 64 : 2 * mean);
    const int warps = 8;
    size_t smem = (size_t)warps * cap * 8 + (size_t)warps * fanout * 4;
    if (smem > 200 * 1024) rc = hg_fail(HG_ECONFIG, "fanout %d too large", fanout);
    else {
      HG_CUDA_TRY(cudaFuncSetAttribute(k_frontier_fill, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
      k_frontier_fill<<<(unsigned)((n_frontier + warps - 1) / warps), warps * 32, smem, s>>>(
          offsets, targets, n_vertices, frontier, n_frontier, fanout, mean, state, pos, flat_out,
          cap, err);
      HG_CUDA_TRY(cudaGetLastError());
    }
  }
  HG_CUDA_TRY(cudaFreeAsync(tmp, s));
  HG_CUDA_TRY(cudaFreeAsync(pos, s));
  HG_CUDA_TRY(cudaFreeAsync(err, s));
  return rc;
}

extern "C" int hg_debug_build_phases(long long* out, int n) {
#ifdef HG_BUILD_PROFILE
  HG_CUDA_TRY(cudaMemcpyFromSymbol(out, hg::g_phase, sizeof(long long) * 16 * (n < 4096 ? n : 4096)));
  return HG_OK;
#else
  return hg_fail(HG_ECONFIG, "built without HG_BUILD_PROFILE");
#endif
}
