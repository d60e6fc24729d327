// Forward / backward of a batch of micrographs (the GNN math of model.py).
//
// Reference: forward model.py:213-247, loss_and_backward model.py:250-287,
// sync_and_update model.py:299-324.  The reference runs one micrograph at a
// time in float64; here a whole cell of roots is one segmented computation:
// every layer is ONE gather+aggregate over the need[k] rows of all roots and
// ONE dense GEMM, because micrographs share nothing but the parameters
// (SURVEY §0.4).  Row numbering is the global one produced by hg_mg_build.
//
// Kernels:
//   k_aggregate    gather rows (features for layer 1, h_{k-1} above) and
//                  build agg_k = [self, mean(nbrs)] (SAGE) or mean(nbrs+self)
//                  (GCN); 16-byte vector loads, several rows per warp
//   gemm (SIMT)    fp32-accumulate tiled GEMM with fused epilogues (bias+ReLU,
//                  ReLU-mask, split-K atomic accumulation for dW)
//   k_softmax_ce   root logits -> loss, dlogits (labels hashed on the fly)
//   k_scatter      transpose of the aggregation for dh_{k-1}
//   k_mask_colsum  dz = dh * (h > 0) and bias gradient
//   k_sgd          fused update + gradient reset + bf16 shadow refresh
#include <cuda_bf16.h>

#include <algorithm>
#include <mutex>
#include <cstdlib>

#include "hg_step.cuh"

namespace hg {


template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<bf16>(bf16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }

// 16-byte vector of T
template <typename T> struct Vec { static constexpr int N = 16 / sizeof(T); };

template <typename T>
__device__ __forceinline__ void load_vec(const T* p, float* v) {
  const uint4 raw = __ldg(reinterpret_cast<const uint4*>(p));
  if constexpr (sizeof(T) == 4) {
    v[0] = __uint_as_float(raw.x); v[1] = __uint_as_float(raw.y);
    v[2] = __uint_as_float(raw.z); v[3] = __uint_as_float(raw.w);
  } else {
    const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
}

// 16 loaded bytes -> VEC floats
template <typename T>
__device__ __forceinline__ void unpack_vec(const uint4 raw, float* v) {
  if constexpr (sizeof(T) == 4) {
    v[0] = __uint_as_float(raw.x); v[1] = __uint_as_float(raw.y);
    v[2] = __uint_as_float(raw.z); v[3] = __uint_as_float(raw.w);
  } else {
    const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
}

// 16-byte vector from shared memory (TMA-staged rows)
template <typename T>
__device__ __forceinline__ void load_vec_s(const T* p, float* v) {
  const uint4 raw = *reinterpret_cast<const uint4*>(p);
  if constexpr (sizeof(T) == 4) {
    v[0] = __uint_as_float(raw.x); v[1] = __uint_as_float(raw.y);
    v[2] = __uint_as_float(raw.z); v[3] = __uint_as_float(raw.w);
  } else {
    const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
}

template <typename T>
__device__ __forceinline__ void store_vec(T* p, const float* v) {
  uint4 raw;
  if constexpr (sizeof(T) == 4) {
    raw.x = __float_as_uint(v[0]); raw.y = __float_as_uint(v[1]);
    raw.z = __float_as_uint(v[2]); raw.w = __float_as_uint(v[3]);
  } else {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162 t = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      w[i] = *reinterpret_cast<const uint32_t*>(&t);
    }
    raw = make_uint4(w[0], w[1], w[2], w[3]);
  }
  *reinterpret_cast<uint4*>(p) = raw;
}

// 16-byte read-only load with an L2 cache policy (createpolicy) and no L1 allocation
__device__ __forceinline__ uint4 ld_evict_first(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

// ------------------------------------------------------------------ aggregate
//
// One group of G = W/VEC lanes (<= 32) per destination row.  For layer 1 the
// source row of need[0] entry i is feat_row[need_ids0[i]] (vertex ids), for
// deeper layers the row index itself.
// Row address of a source entry: layer 1 maps need[0] entry -> vertex ->
// (local table row | owner GPU's table over NVLink); deeper layers index
// h_{k-1} rows directly.
template <typename T>
struct RowSrc {
  const T* src;
  int ld;
  const int32_t* need_ids0;   // layer 1 only
  const int32_t* feat_row;    // vertex -> row (local table, or owner's table with peers)
  const T* const* peers;      // per-home row tables (multi-GPU peer reads) or null
  const int32_t* home;
  const T* stage;             // staged mode: remote rows pre-gathered into HBM
  const int32_t* stage_row;
  int rank;
  bool by_vid;                // index arrays hold vertex ids (layer 1 vid lists)
  const int32_t* handle;      // staged mode: need[0] row handles (hg_resolve_rows) or null
  bool stream;                // source rows read once (feature table): L2 evict-first
  __device__ __forceinline__ const T* row(int i) const {
    if (by_vid) return vrow(i);
    if (handle) {
      const int h = handle[i];
      return h >= 0 ? src + (int64_t)h * ld : stage + (int64_t)(-1 - h) * ld;
    }
    if (!need_ids0) return src + (int64_t)i * ld;
    return vrow(need_ids0[i]);
  }
  // row of vertex v (layer 1 with vertex-id pair lists)
  __device__ __forceinline__ const T* vrow(int v) const {
    if (stage_row) {
      if (home[v] != rank) return stage + (int64_t)stage_row[v] * ld;
      return src + (int64_t)feat_row[v] * ld;
    }
    const int r = feat_row ? feat_row[v] : v;
    const T* base = peers ? peers[home[v]] : src;
    return base + (int64_t)r * ld;
  }
};

// Segments of one launch: blockIdx.y selects a batch (a group of run-ahead
// iterations shares the feature source and is gathered in one launch).
template <typename T>
struct AggSegs {
  const int32_t* self_pos[HG_MAX_GROUP];
  const int32_t* nbr_off[HG_MAX_GROUP];
  const int32_t* nbr_idx[HG_MAX_GROUP];
  const int32_t* n_rows[HG_MAX_GROUP];
  int cap[HG_MAX_GROUP];                // row capacity (nbr_off holds cap + 1 entries)
  T* out[HG_MAX_GROUP];
  const int32_t* handle[HG_MAX_GROUP];  // staged mode: per-batch need[0] row handles
};

#ifndef HG_AGG_U
#define HG_AGG_U 10     // neighbour loads in flight per lane (layer-1 fanout 10 in one round)
#endif
#ifndef HG_AGG_MINB
#define HG_AGG_MINB 3   // CTAs/SM the register budget is sized for (U = 10 -> ~80 registers)
#endif

// One group of G lanes per destination row (G = min(32, 16-byte vectors per
// row)), so a warp carries 32/G rows at once.  A row's neighbour indices are
// read by its lanes in one coalesced load and broadcast by shuffles; each
// lane then issues up to U predicated 16-byte row loads before consuming
// any, so a row's whole neighbour list (fanout <= U) is one DRAM round trip.
// The dependent chain per row is (self_pos, nbr_off) -> (nbr_idx, self row)
// -> neighbour rows -> store; with ~2 rows x U loads in flight per warp the
// ~100K-row gather of a batch keeps >100 KB in flight per SM.
template <typename T, bool SAGE>
__global__ void __launch_bounds__(256, HG_AGG_MINB)
k_aggregate(RowSrc<T> rs_in, AggSegs<T> segs, int W, int out_ld, int pad_cap) {
  constexpr int U = HG_AGG_U;
  pdl_trigger();
  pdl_wait();
  RowSrc<T> rs = rs_in;
  if (segs.handle[blockIdx.y]) rs.handle = segs.handle[blockIdx.y];  // this batch's handles
  const int32_t* __restrict__ self_pos = segs.self_pos[blockIdx.y];
  const int32_t* __restrict__ nbr_off = segs.nbr_off[blockIdx.y];
  const int32_t* __restrict__ nbr_idx = segs.nbr_idx[blockIdx.y];
  const int32_t* __restrict__ n_rows_dev = segs.n_rows[blockIdx.y];
  T* __restrict__ out = segs.out[blockIdx.y];
  constexpr int VEC = Vec<T>::N;
  uint64_t pol = 0;
  if (rs.stream) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  constexpr unsigned FULL = 0xffffffffu;
  if (pad_cap && blockIdx.x == gridDim.x - 1) {
    // the tensor-core dW GEMM reduces over rows up to the next multiple of 64:
    // keep those padding rows zero (folded in here instead of its own launch)
    const int n = *n_rows_dev;
    const int pad = min(pad_cap, (n + 63) / 64 * 64);
    for (int64_t i = threadIdx.x; i < (int64_t)(pad - n) * out_ld; i += blockDim.x)
      out[(int64_t)n * out_ld + i] = from_f<T>(0.f);
  }
  const int nvec = W / VEC;                        // vectors per row
  const int G = nvec >= 32 ? 32 : (nvec >= 16 ? 16 : (nvec >= 8 ? 8 : (nvec >= 4 ? 4 : (nvec >= 2 ? 2 : 1))));
  const int P = 32 / G;                            // rows per warp
  const int lane = threadIdx.x & 31, gi = lane / G, gl = lane % G;
  const int warps = blockDim.x >> 5;
  const int n_rows = *n_rows_dev;
  const int stride = gridDim.x * warps * P;
  // Software pipeline over this warp's rows a, a+stride, ...: the CSR range
  // and self index of row i+2 and the neighbour indices of row i+1 are in
  // flight while row i's source rows load, so the dependent index chain
  // (offsets -> indices -> rows) costs one DRAM round trip per row, not three.
  int a = (blockIdx.x * warps + (threadIdx.x >> 5)) * P + gi;
  // row metadata is loaded for any row inside the capacity (in bounds) and
  // discarded past the device row count, so the first loads do not wait for
  // that count
  const int cap_rows = segs.cap[blockIdx.y];
  auto meta = [&](int r, int& j0, int& deg, int& sidx) {
    j0 = 0; deg = 0; sidx = 0;
    if (r < cap_rows) {
      j0 = nbr_off[r];
      deg = nbr_off[r + 1] - j0;
      sidx = self_pos[r];
    }
  };
  auto valid_meta = [&](int r, int& j0, int& deg, int& sidx) {
    if (r >= n_rows) { j0 = 0; deg = 0; sidx = 0; }
  };
  int j0, deg, sidx, j0n, degn, sidxn;
  meta(a, j0, deg, sidx);
  meta(a + stride, j0n, degn, sidxn);
  valid_meta(a, j0, deg, sidx);
  valid_meta(a + stride, j0n, degn, sidxn);
  int idx = gl < min(G, deg) ? nbr_idx[j0 + gl] : 0;
  while (__any_sync(FULL, a < n_rows)) {
    const bool row_ok = a < n_rows;
    // prefetch: indices of the next row, range of the one after
    const int idxn = gl < min(G, degn) ? nbr_idx[j0n + gl] : 0;
    int j0nn, degnn, sidxnn;
    meta(a + 2 * stride, j0nn, degnn, sidxnn);
    valid_meta(a + 2 * stride, j0nn, degnn, sidxnn);
    const T* sp = rs.row(row_ok ? sidx : 0);
    const int max_deg = __reduce_max_sync(FULL, deg);
    T* o = out + (int64_t)a * out_ld;
    for (int c0 = 0; c0 < nvec; c0 += G) {
      const int cv = c0 + gl;
      const bool act = row_ok && cv < nvec;
      const int col = cv * VEC;
      float acc[VEC];
#pragma unroll
      for (int i = 0; i < VEC; ++i) acc[i] = 0.f;
      // the self row stays packed (16 bytes) through the neighbour loop
      const uint4 self_raw = act ? __ldg(reinterpret_cast<const uint4*>(sp + col)) : make_uint4(0, 0, 0, 0);
      for (int jb = 0; jb < max_deg; jb += G) {       // neighbour chunks of G indices
        const int ix = jb == 0 ? idx : (gl < deg - jb ? nbr_idx[j0 + jb + gl] : 0);
        const int cnt = min(G, deg - jb);              // this group's neighbours in the chunk
        const int rounds = min(G, max_deg - jb);       // warp-uniform
        for (int t0 = 0; t0 < rounds; t0 += U) {
          uint4 x[U];
#pragma unroll
          for (int t = 0; t < U; ++t) {
            const int v = __shfl_sync(FULL, ix, (gi * G + ((t0 + t) & (G - 1))) & 31);
            if (act && t0 + t < cnt)
              x[t] = rs.stream ? ld_evict_first(rs.row(v) + col, pol)
                               : __ldg(reinterpret_cast<const uint4*>(rs.row(v) + col));
            else x[t] = make_uint4(0, 0, 0, 0);
          }
#pragma unroll
          for (int t = 0; t < U; ++t) {
            if constexpr (sizeof(T) == 4) {
              acc[0] += __uint_as_float(x[t].x); acc[1] += __uint_as_float(x[t].y);
              acc[2] += __uint_as_float(x[t].z); acc[3] += __uint_as_float(x[t].w);
            } else {
              const uint32_t w[4] = {x[t].x, x[t].y, x[t].z, x[t].w};
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                acc[2 * i] += __uint_as_float(w[i] << 16);
                acc[2 * i + 1] += __uint_as_float(w[i] & 0xFFFF0000u);
              }
            }
          }
        }
      }
      if (!act) continue;
      float self[VEC];
      unpack_vec<T>(self_raw, self);
      if constexpr (SAGE) {
        float nb[VEC];
        const float inv = deg > 0 ? 1.0f / (float)deg : 0.f;
#pragma unroll
        for (int i = 0; i < VEC; ++i) nb[i] = deg > 0 ? acc[i] * inv : self[i];
        store_vec(o + col, self);
        store_vec(o + W + col, nb);
      } else {
        const float inv = 1.0f / (float)(deg + 1);
#pragma unroll
        for (int i = 0; i < VEC; ++i) acc[i] = (acc[i] + self[i]) * inv;
        store_vec(o + col, acc);
      }
    }
    a += stride;
    j0 = j0n; deg = degn; sidx = sidxn; idx = idxn;
    j0n = j0nn; degn = degnn; sidxn = sidxnn;
  }
}

// ------------------------------------------------------------------ SIMT GEMM
//
// C[m,n] = sum_k A(m,k) B(k,n); A(m,k) = AT ? A[k*lda+m] : A[m*lda+k],
// B(k,n) = BT ? B[n*ldb+k] : B[k*ldb+n].  M or K may be device-resident
// (row counts of the batch).  fp32 accumulation.
enum Epi { EPI_STORE = 0, EPI_BIAS_RELU = 1, EPI_MASK = 2, EPI_ATOMIC = 3 };

constexpr int BM = 64, BN = 64, BK = 16;

template <typename TA, bool AT, bool BT, int EPI, typename TC, typename TM>
__global__ void __launch_bounds__(256)
k_gemm(const TA* __restrict__ A, int lda, const float* __restrict__ B, int ldb, TC* C, int ldc,
       const int32_t* M_dev, int M_host, int N, const int32_t* K_dev, int K_host,
       const float* __restrict__ bias, const TM* __restrict__ mask, int ldm) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int M = M_dev ? *M_dev : M_host;
  const int K = K_dev ? *K_dev : K_host;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= M) return;
  // split along K (gridDim.z)
  const int kchunk = ((K + gridDim.z - 1) / gridDim.z + BK - 1) / BK * BK;
  const int kb = blockIdx.z * kchunk;
  const int ke = min(K, kb + kchunk);
  if (kb >= ke) return;
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  float acc[4][4] = {};
  for (int k0 = kb; k0 < ke; k0 += BK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + i * 256;
      int r, kk;
      if (AT) { kk = e / BM; r = e % BM; } else { r = e / BK; kk = e % BK; }
      const int gm = m0 + r, gk = k0 + kk;
      float v = 0.f;
      if (gm < M && gk < ke) v = to_f(AT ? A[(int64_t)gk * lda + gm] : A[(int64_t)gm * lda + gk]);
      As[kk][r] = v;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + i * 256;
      int c, kk;
      if (BT) { c = e / BK; kk = e % BK; } else { kk = e / BN; c = e % BN; }
      const int gn = n0 + c, gk = k0 + kk;
      float v = 0.f;
      if (gn < N && gk < ke) v = BT ? B[(int64_t)gn * ldb + gk] : B[(int64_t)gk * ldb + gn];
      Bs[kk][c] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      float v = acc[i][j];
      if constexpr (EPI == EPI_BIAS_RELU) {
        v = fmaxf(v + bias[gn], 0.f);
        C[(int64_t)gm * ldc + gn] = from_f<TC>(v);
      } else if constexpr (EPI == EPI_MASK) {
        v = to_f(mask[(int64_t)gm * ldm + gn]) > 0.f ? v : 0.f;
        C[(int64_t)gm * ldc + gn] = from_f<TC>(v);
      } else if constexpr (EPI == EPI_ATOMIC) {
        atomicAdd(reinterpret_cast<float*>(C) + (int64_t)gm * ldc + gn, v);
      } else {
        C[(int64_t)gm * ldc + gn] = from_f<TC>(v);
      }
    }
  }
}

// ------------------------------------------------------------------ loss

// warp per root: softmax-CE on the root logits (model.py:253-259); logits are
// overwritten with dlogits = softmax - onehot(label).
__global__ void k_softmax_ce(float* __restrict__ logits, int C, const int64_t* __restrict__ roots,
                             int n_roots, const int32_t* __restrict__ n_dev, uint64_t label_state,
                             const int32_t* __restrict__ labels, float* __restrict__ loss,
                             bf16* __restrict__ dl_lowp, int ldp) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x * (blockDim.x / 32) + warp_id();
  if (r >= n_roots) return;
  const int lane = lane_id();
  float* x = logits + (int64_t)r * C;
  // the independent loads first -- the device root count, the label source
  // and the row's logits (<= 8 per lane) -- so they share one round trip
  // (capacity rows hold stale logits; they are only read, then zeroed)
  constexpr int kPer = 8;
  const int n = n_dev ? *n_dev : n_roots;
  const int64_t root = labels ? 0 : roots[r];
  const int lab_in = labels ? labels[r] : 0;
  float xv[kPer];
  const bool regs = C <= 32 * kPer;
#pragma unroll
  for (int t = 0; t < kPer; ++t) {
    const int c = lane + 32 * t;
    xv[t] = regs && c < C ? x[c] : -INFINITY;
  }
  if (r >= n) {  // capacity rows past the device root count: no loss, no gradient
    for (int c = lane; c < C; c += 32) x[c] = 0.f;
    if (dl_lowp)
      for (int c = lane; c < ldp; c += 32) dl_lowp[(int64_t)r * ldp + c] = __float2bfloat16_rn(0.f);
    if (lane == 0) loss[r] = 0.f;
    return;
  }
  float mx = -INFINITY;
  if (regs) {
#pragma unroll
    for (int t = 0; t < kPer; ++t) mx = fmaxf(mx, xv[t]);
  } else {
    for (int c = lane; c < C; c += 32) mx = fmaxf(mx, x[c]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float s = 0.f;
  if (regs) {
#pragma unroll
    for (int t = 0; t < kPer; ++t)
      if (lane + 32 * t < C) s += expf(xv[t] - mx);
  } else {
    for (int c = lane; c < C; c += 32) s += expf(x[c] - mx);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const int label = labels ? lab_in : (int)(mix64(label_state ^ (uint64_t)root) % (uint64_t)C);
  const float xl = x[label];
  __syncwarp();
  const float inv = 1.0f / s;
  if (regs) {
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int c = lane + 32 * t;
      if (c >= C) break;
      const float g = expf(xv[t] - mx) * inv - (c == label ? 1.f : 0.f);
      x[c] = g;
      if (dl_lowp) dl_lowp[(int64_t)r * ldp + c] = __float2bfloat16_rn(g);
    }
  } else {
    for (int c = lane; c < C; c += 32) {
      const float g = expf(x[c] - mx) * inv - (c == label ? 1.f : 0.f);
      x[c] = g;
      if (dl_lowp) dl_lowp[(int64_t)r * ldp + c] = __float2bfloat16_rn(g);
    }
  }
  if (dl_lowp)
    for (int c = C + lane; c < ldp; c += 32) dl_lowp[(int64_t)r * ldp + c] = __float2bfloat16_rn(0.f);
  if (lane == 0) loss[r] = logf(s) - (xl - mx);
}

// out[r][c] = bf16(W[r][c]) for c < cols, 0 for cols <= c < ld (K-major operand
// with a 16-byte-aligned row pitch for TMA)
__global__ void k_pad_bf16(const float* __restrict__ W, int rows, int cols, bf16* __restrict__ out,
                           int ld) {
  const int64_t total = (int64_t)rows * ld;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / ld), c = (int)(i % ld);
    out[i] = __float2bfloat16_rn(c < cols ? W[(int64_t)r * cols + c] : 0.f);
  }
}

// Fused classifier head (model.py:246, 253-265): per root, logits = h_L @ W_c
// (no bias), softmax-CE with the label hashed on the fly, dlogits, then
// dz_L = (dlogits @ W_cᵀ) * (h_L > 0) and the bias gradient of layer L.
// One warp per root; W_c staged once per CTA in shared memory with an odd
// row pitch so both the class-parallel and the hidden-parallel loops are
// bank-conflict free.
template <typename T>
__global__ void __launch_bounds__(256)
k_head(const T* __restrict__ hL, const float* __restrict__ Wc, int H, int C,
       const int64_t* __restrict__ roots, int n_cap, const int32_t* __restrict__ n_dev,
       uint64_t label_state, const int32_t* __restrict__ labels, float* __restrict__ dlogits,
       float* __restrict__ loss,
       float* __restrict__ dz, bf16* __restrict__ dz_lowp, int cap_rows, float* __restrict__ gb,
       int backward) {
  extern __shared__ float sm[];
  const int n_roots = n_dev ? *n_dev : n_cap;
  for (int i = n_roots + blockIdx.x * blockDim.x + threadIdx.x; i < n_cap;
       i += gridDim.x * blockDim.x)
    loss[i] = 0.f;  // capacity rows past the device root count
  const int pitch = C | 1;
  float* ws = sm;                                   // [H][pitch]
  float* gbs = ws + (size_t)H * pitch;              // [H]
  float* rowbuf = gbs + H;                          // [8][H]
  float* dlbuf = rowbuf + 8 * H;                    // [8][C]
  for (int h = warp_id(); h < H; h += blockDim.x / 32)
    for (int c = lane_id(); c < C; c += 32) ws[h * pitch + c] = Wc[(int64_t)h * C + c];
  for (int i = threadIdx.x; i < H; i += blockDim.x) gbs[i] = 0.f;
  __syncthreads();
  const int w = warp_id(), lane = lane_id();
  float* hrow = rowbuf + w * H;
  float* dl = dlbuf + w * C;
  for (int r = blockIdx.x * 8 + w; r < n_roots; r += gridDim.x * 8) {
    for (int h = lane; h < H; h += 32) hrow[h] = to_f(hL[(int64_t)r * H + h]);
    __syncwarp();
    float mx = -INFINITY;
    for (int c = lane; c < C; c += 32) {
      float acc = 0.f;
      for (int h = 0; h < H; ++h) acc = fmaf(hrow[h], ws[h * pitch + c], acc);
      dl[c] = acc;
      if (!backward) dlogits[(int64_t)r * C + c] = acc;  // forward only: the logits themselves
      mx = fmaxf(mx, acc);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float s = 0.f;
    for (int c = lane; c < C; c += 32) s += expf(dl[c] - mx);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const int label = labels ? labels[r]
                             : (int)(mix64(label_state ^ (uint64_t)roots[r]) % (uint64_t)C);
    __syncwarp();
    const float xl = dl[label];
    __syncwarp();
    const float inv = 1.0f / s;
    for (int c = lane; c < C; c += 32) {
      const float g = expf(dl[c] - mx) * inv - (c == label ? 1.f : 0.f);
      dl[c] = g;
      if (backward) dlogits[(int64_t)r * C + c] = g;
    }
    if (lane == 0) loss[r] = logf(s) - (xl - mx);
    __syncwarp();
    if (backward) {
      for (int h = lane; h < H; h += 32) {
        float acc = 0.f;
        for (int c = 0; c < C; ++c) acc = fmaf(dl[c], ws[h * pitch + c], acc);
        const float v = hrow[h] > 0.f ? acc : 0.f;
        dz[(int64_t)r * H + h] = v;
        if (dz_lowp) dz_lowp[(int64_t)r * H + h] = __float2bfloat16_rn(v);
        atomicAdd(gbs + h, v);
      }
    }
    __syncwarp();
  }
  if (backward && dz_lowp && blockIdx.x == 0) {  // zero padding rows for the tensor-core dW
    const int pad = min(cap_rows, (n_roots + 63) / 64 * 64);
    for (int64_t i = (int64_t)n_roots * H + threadIdx.x; i < (int64_t)pad * H; i += blockDim.x)
      dz_lowp[i] = __float2bfloat16_rn(0.f);
  }
  __syncthreads();
  if (backward)
    for (int h = threadIdx.x; h < H; h += blockDim.x) atomicAdd(gb + h, gbs[h]);
}

// ------------------------------------------------------------------ backward

// Transpose of k_aggregate (model.py:266-285): warp per destination row.
template <bool SAGE>
__global__ void __launch_bounds__(256)
k_scatter(const float* __restrict__ dagg, int ld, const int32_t* __restrict__ self_pos,
          const int32_t* __restrict__ nbr_off, const int32_t* __restrict__ nbr_idx,
          const int32_t* __restrict__ n_rows_dev, int W, float* __restrict__ dh) {
  const int n_rows = *n_rows_dev;
  const int a = blockIdx.x * (blockDim.x / 32) + warp_id();
  if (a >= n_rows) return;
  const int lane = lane_id();
  const int s = self_pos[a];
  const int j0 = nbr_off[a], j1 = nbr_off[a + 1];
  const int deg = j1 - j0;
  const float* g = dagg + (int64_t)a * ld;
  if constexpr (SAGE) {
    const float inv = deg > 0 ? 1.0f / (float)deg : 0.f;
    for (int c = lane; c < W; c += 32) {
      const float gs = g[c], gn = g[W + c];
      atomicAdd(dh + (int64_t)s * W + c, deg > 0 ? gs : gs + gn);
      if (deg > 0) {
        const float v = gn * inv;
        for (int j = j0; j < j1; ++j) atomicAdd(dh + (int64_t)nbr_idx[j] * W + c, v);
      }
    }
  } else {
    const float inv = 1.0f / (float)(deg + 1);
    for (int c = lane; c < W; c += 32) {
      const float v = g[c] * inv;
      atomicAdd(dh + (int64_t)s * W + c, v);
      for (int j = j0; j < j1; ++j) atomicAdd(dh + (int64_t)nbr_idx[j] * W + c, v);
    }
  }
}

// Fused backward of one aggregation layer, one root's micrograph at a time:
// dh_{k-1} = scatterᵀ(dagg_k) (the transpose of k_aggregate), then
// dz = dh * (h_{k-1} > 0), its bf16 copy for the tensor-core GEMMs, the f32
// copy when a SIMT GEMM still needs it, and the bias-gradient column sums.
// A root's need[k-1] rows are contiguous and every self/neighbour index of
// its need[k] rows points inside them (k_mg_finalize), so the scatter runs in
// shared memory with each thread owning whole columns: no atomics, no zeroing
// pass, one read of dagg and h, one write of dz.  Replaces k_zero_rows +
// k_scatter + k_mask_colsum when root_rows[k-1] * H floats fit in smem.
template <bool SAGE, typename T>
__global__ void __launch_bounds__(256)
k_scatter_root(const float* __restrict__ dagg, int ld, const int32_t* __restrict__ need_off_p,
               const int32_t* __restrict__ need_off_c, const int32_t* __restrict__ self_pos,
               const int32_t* __restrict__ nbr_off, const int32_t* __restrict__ nbr_idx,
               int n_roots, int H, const T* __restrict__ h, float* __restrict__ dh_out,
               bf16* __restrict__ lowp, float* __restrict__ gb,
               const int32_t* __restrict__ n_rows_dev, int cap_rows) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float acc[];  // [root_rows x H]
  // each thread owns columns c and c + blockDim.x (H <= 2 * blockDim.x)
  float colsum0 = 0.f, colsum1 = 0.f;
  for (int r = blockIdx.x; r < n_roots; r += gridDim.x) {
    const int q0 = need_off_p[r], nq = need_off_p[r + 1] - q0;
    const int p0 = need_off_c[r], p1 = need_off_c[r + 1];
    for (int c = threadIdx.x; c < H; c += blockDim.x) {
      float colsum = 0.f;
      for (int i = 0; i < nq; ++i) acc[i * H + c] = 0.f;
      for (int p = p0; p < p1; ++p) {
        const int s = self_pos[p] - q0;
        const int j0 = nbr_off[p], j1 = nbr_off[p + 1];
        const int deg = j1 - j0;
        const float* g = dagg + (int64_t)p * ld;
        if constexpr (SAGE) {
          const float gs = g[c], gn = g[H + c];
          acc[s * H + c] += deg > 0 ? gs : gs + gn;
          const float v = deg > 0 ? gn / (float)deg : 0.f;
          for (int j = j0; j < j1; ++j) acc[(nbr_idx[j] - q0) * H + c] += v;
        } else {
          const float v = g[c] / (float)(deg + 1);
          acc[s * H + c] += v;
          for (int j = j0; j < j1; ++j) acc[(nbr_idx[j] - q0) * H + c] += v;
        }
      }
      for (int i = 0; i < nq; ++i) {
        const int64_t o = (int64_t)(q0 + i) * H + c;
        const float v = to_f(h[o]) > 0.f ? acc[i * H + c] : 0.f;
        if (dh_out) dh_out[o] = v;
        if (lowp) lowp[o] = __float2bfloat16_rn(v);
        colsum += v;
      }
      if (c == threadIdx.x) colsum0 += colsum;
      else colsum1 += colsum;
    }
  }
  if (threadIdx.x < H) atomicAdd(gb + threadIdx.x, colsum0);
  if (threadIdx.x + blockDim.x < H) atomicAdd(gb + threadIdx.x + blockDim.x, colsum1);
  // the dW GEMM reduces over rows up to the next multiple of 64: zero the padding
  if (lowp && blockIdx.x == 0) {
    const int n_rows = *n_rows_dev;
    const int pad = min(cap_rows, (n_rows + 63) / 64 * 64);
    for (int64_t i = (int64_t)n_rows * H + threadIdx.x; i < (int64_t)pad * H; i += blockDim.x)
      lowp[i] = __float2bfloat16_rn(0.f);
  }
}

// Top-layer special case of k_scatter_root (k == L, need[L] = [root]): every
// need[L-1] row of root r is either the root's self row or one of its sampled
// neighbours, each exactly once (layers are deduplicated, no self-loops), so
// the transpose of the aggregation is a per-row map -- SAGE: self row gets
// dagg[r, :H] (+ dagg[r, H:] when deg == 0), a neighbour dagg[r, H:] / deg;
// GCN: every row dagg[r] / (deg + 1) -- with the same arithmetic as the
// scatter.  One warp per row, 8 columns per lane: two dependent round trips
// per CTA instead of the per-column loops over rows and pairs.
template <bool SAGE, typename T>
__global__ void __launch_bounds__(256)
k_scatter_top(const float* __restrict__ dagg, int ld, const int32_t* __restrict__ need_off_p,
              const int32_t* __restrict__ need_off_c, const int32_t* __restrict__ self_pos,
              const int32_t* __restrict__ nbr_off, const int8_t* __restrict__ in_layer,
              int n_roots, int H,
              const T* __restrict__ h, float* __restrict__ dh_out, bf16* __restrict__ lowp,
              float* __restrict__ gb, const int32_t* __restrict__ n_rows_dev, int cap_rows) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[8][257];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = lane * 8;
  const bool lane_on = c0 < H;
  float cs[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) cs[j] = 0.f;
  const int n_rows = *n_rows_dev;
  // warp per root (its <= 1 + f1 need[L-1] rows), four rows' loads in flight
  // at a time
  for (int r = blockIdx.x * 8 + warp; r < n_roots; r += gridDim.x * 8) {
    const int q0 = need_off_p[r], nq = need_off_p[r + 1] - q0;
    const int rowL = need_off_c[r];
    if (!lane_on || nq == 0 || need_off_c[r + 1] - rowL != 1) continue;  // empty micrograph
    // software pipeline: the h rows of the next four need[L-1] rows (and their
    // in-layer flags) are in flight while this batch is computed; the first
    // batch's loads share a round trip with the self / degree / dagg loads
    constexpr int NV = sizeof(T) == 4 ? 2 : 1;  // 16-byte vectors per lane row
    uint4 raw[4][NV];
    int8_t inl[4];
    auto fetch = [&](int i0) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int u = q0 + min(i0 + t, nq - 1);
#pragma unroll
        for (int v = 0; v < NV; ++v)
          raw[t][v] = __ldg(reinterpret_cast<const uint4*>(h + (int64_t)u * H + c0) + v);
        inl[t] = in_layer[u];
      }
    };
    fetch(0);
    const int srow = self_pos[rowL];
    const int deg = nbr_off[rowL + 1] - nbr_off[rowL];
    const float* g = dagg + (int64_t)rowL * ld;
    float gs[8], gn[8];
#pragma unroll
    for (int j = 0; j < 8; j += 4) {
      const float4 a = *reinterpret_cast<const float4*>(g + c0 + j);
      gs[j] = a.x; gs[j + 1] = a.y; gs[j + 2] = a.z; gs[j + 3] = a.w;
      if constexpr (SAGE) {
        const float4 b = *reinterpret_cast<const float4*>(g + H + c0 + j);
        gn[j] = b.x; gn[j + 1] = b.y; gn[j + 2] = b.z; gn[j + 3] = b.w;
      }
    }
    for (int i0 = 0; i0 < nq; i0 += 4) {
      float hv[4][8];
      int8_t il[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
#pragma unroll
        for (int v = 0; v < NV; ++v) unpack_vec<T>(raw[t][v], hv[t] + v * (8 / NV));
        il[t] = inl[t];
      }
      if (i0 + 4 < nq) fetch(i0 + 4);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (i0 + t >= nq) break;
        const int u = q0 + i0 + t;
        // a row is the root's self row and/or one of its sampled neighbours (both
        // with a self-loop); the neighbour rows are exactly layers[L-1] (in_layer)
        const bool self = u == srow, nbr = il[t] != 0;
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float x;
          if constexpr (SAGE)
            x = (self ? (deg > 0 ? gs[j] : gs[j] + gn[j]) : 0.f) + (nbr ? gn[j] / (float)deg : 0.f);
          else
            x = gs[j] * ((float)((int)self + (int)nbr) / (float)(deg + 1));
          v[j] = hv[t][j] > 0.f ? x : 0.f;
          cs[j] += v[j];
        }
        const int64_t o = (int64_t)u * H + c0;
        if (dh_out) {
          *reinterpret_cast<float4*>(dh_out + o) = make_float4(v[0], v[1], v[2], v[3]);
          *reinterpret_cast<float4*>(dh_out + o + 4) = make_float4(v[4], v[5], v[6], v[7]);
        }
        if (lowp) store_vec(lowp + o, v);
      }
    }
  }
  if (lane_on)
#pragma unroll
    for (int j = 0; j < 8; ++j) red[warp][c0 + j] = cs[j];
  __syncthreads();
  for (int c = threadIdx.x; c < H; c += blockDim.x) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][c];
    atomicAdd(gb + c, t);
  }
  // the dW GEMM reduces over rows up to the next multiple of 64: zero the padding
  if (lowp && blockIdx.x == 0) {
    const int pad = min(cap_rows, (n_rows + 63) / 64 * 64);
    for (int64_t i = (int64_t)n_rows * H + threadIdx.x; i < (int64_t)pad * H; i += blockDim.x)
      lowp[i] = __float2bfloat16_rn(0.f);
  }
}

// dz = dh * (h > 0) in place; gb[c] += sum_rows dz[., c]
// Optional bf16 copy of dz for the tensor-core dW GEMM, whose row reduction
// reads up to the next multiple of 64 rows: those padding rows are zeroed.
template <typename T>
__global__ void __launch_bounds__(256)
k_mask_colsum(float* __restrict__ dh, const T* __restrict__ h, const int32_t* __restrict__ n_rows_dev,
              int H, float* __restrict__ gb, bf16* __restrict__ lowp, int cap_rows) {
  pdl_trigger();
  pdl_wait();
  const int n_rows = *n_rows_dev;
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int r0 = blockIdx.y * 8 + (threadIdx.x >> 5);
  float s = 0.f;
  if (c < H) {
    for (int r = r0; r < n_rows; r += gridDim.y * 8) {
      const int64_t i = (int64_t)r * H + c;
      float v = dh[i];
      v = to_f(h[i]) > 0.f ? v : 0.f;
      dh[i] = v;
      if (lowp) lowp[i] = __float2bfloat16_rn(v);
      s += v;
    }
    if (lowp) {
      const int pad = min(cap_rows, (n_rows + 63) / 64 * 64);
      for (int r = n_rows + r0; r < pad; r += gridDim.y * 8) lowp[(int64_t)r * H + c] = __float2bfloat16_rn(0.f);
    }
  }
  __shared__ float red[8][33];
  red[threadIdx.x >> 5][threadIdx.x & 31] = s;
  __syncthreads();
  if (threadIdx.x < 32 && c < H) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][threadIdx.x];
    atomicAdd(gb + c, t);
  }
}

// column sums of an already-masked matrix (bias grad of the top layer)
__global__ void __launch_bounds__(256)
k_colsum(const float* __restrict__ x, const int32_t* __restrict__ n_rows_dev, int n_rows_host,
         int H, float* __restrict__ gb, bf16* __restrict__ lowp, int cap_rows) {
  const int n_rows = n_rows_dev ? *n_rows_dev : n_rows_host;
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int r0 = blockIdx.y * 8 + (threadIdx.x >> 5);
  float s = 0.f;
  if (c < H) {
    for (int r = r0; r < n_rows; r += gridDim.y * 8) {
      const float v = x[(int64_t)r * H + c];
      if (lowp) lowp[(int64_t)r * H + c] = __float2bfloat16_rn(v);
      s += v;
    }
    if (lowp) {
      const int pad = min(cap_rows, (n_rows + 63) / 64 * 64);
      for (int r = n_rows + r0; r < pad; r += gridDim.y * 8) lowp[(int64_t)r * H + c] = __float2bfloat16_rn(0.f);
    }
  }
  __shared__ float red[8][33];
  red[threadIdx.x >> 5][threadIdx.x & 31] = s;
  __syncthreads();
  if (threadIdx.x < 32 && c < H) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][threadIdx.x];
    atomicAdd(gb + c, t);
  }
}

// WT[c][r] = bf16(W[r][c]): K-major B operand of the tensor-core layer GEMM
__global__ void k_transpose_bf16(const float* __restrict__ W, int rows, int cols,
                                 bf16* __restrict__ WT, bf16* __restrict__ Wplain) {
  __shared__ float tile[32][33];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    const float v = (r < rows && c < cols) ? W[(int64_t)r * cols + c] : 0.f;
    tile[i][threadIdx.x] = v;
    if (Wplain && r < rows && c < cols) Wplain[(int64_t)r * cols + c] = __float2bfloat16_rn(v);
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (c < cols && r < rows) WT[(int64_t)c * rows + r] = __float2bfloat16_rn(tile[threadIdx.x][i]);
  }
}

// zero rows [n_rows, min(roundup64(n_rows), cap)) of a bf16 [rows x W] matrix
__global__ void k_zero_pad_rows(bf16* __restrict__ x, const int32_t* __restrict__ n_rows_dev, int W,
                                int cap_rows) {
  const int n = *n_rows_dev;
  const int pad = min(cap_rows, (n + 63) / 64 * 64);
  const int64_t total = (int64_t)(pad - n) * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    x[(int64_t)n * W + i] = __float2bfloat16_rn(0.f);
}

__global__ void k_zero_rows(float* __restrict__ x, const int32_t* __restrict__ n_rows_dev, int W) {
  const int64_t total = (int64_t)(*n_rows_dev) * W;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < total;
       i += (int64_t)gridDim.x * blockDim.x * 4) {
    if (i + 4 <= total) *reinterpret_cast<float4*>(x + i) = make_float4(0.f, 0.f, 0.f, 0.f);
    else for (int64_t j = i; j < total; ++j) x[j] = 0.f;
  }
}

// Where each parameter's bf16 operand copies live (the step's layout).
// SGD + gradient reset, then the parameters' bf16 operand copies, in one
// launch over 32 x 32 tiles of every weight matrix (f32 reads/writes and the
// straight bf16 copy coalesced along columns; the transposed copy staged in
// shared memory so its writes are coalesced too), plus elementwise blocks for
// the biases.  Replaces three transposes and a pad per step.
__global__ void __launch_bounds__(256)
k_sgd_refresh(float* __restrict__ p, float* __restrict__ g, float lr, float inv_batch, int update,
              SgdPlan P) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  if (t >= P.n_tiles) {  // biases: elementwise
    for (int64_t i = P.plain_lo + (int64_t)(t - P.n_tiles) * blockDim.x + threadIdx.x;
         i < P.plain_hi; i += (int64_t)(gridDim.x - P.n_tiles) * blockDim.x) {
      if (update) {
        p[i] -= lr * (g[i] * inv_batch);
        g[i] = 0.f;
      }
    }
    return;
  }
  __shared__ bf16 tile[32][34];
  int mi = 0;
  while (mi + 1 < P.n_mats && P.m[mi + 1].tile0 <= t) ++mi;
  const SgdMat& M = P.m[mi];
  const int lt = t - M.tile0, tr = lt / M.tiles_c, tc = lt % M.tiles_c;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int r = tr * 32 + ty + 8 * j, c = tc * 32 + tx;
    if (r < M.rows && c < M.cols) {
      const int64_t i = M.off + (int64_t)r * M.cols + c;
      float v = p[i];
      if (update) {
        v -= lr * (g[i] * inv_batch);
        p[i] = v;
        g[i] = 0.f;
      }
      const bf16 b = __float2bfloat16_rn(v);
      if (M.sdst) M.sdst[(int64_t)r * M.sld + c] = b;
      tile[ty + 8 * j][tx] = b;
    }
  }
  if (!M.tdst) return;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = tc * 32 + ty + 8 * j, r = tr * 32 + tx;
    if (r < M.rows && c < M.cols) M.tdst[(int64_t)c * M.tld + r] = tile[tx][ty + 8 * j];
  }
}

__global__ void k_sgd(float* __restrict__ p, float* __restrict__ g, bf16* __restrict__ shadow,
                      int64_t n, float lr, float inv_batch) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float step = g[i] * inv_batch;
    const float v = p[i] - lr * step;
    p[i] = v;
    g[i] = 0.f;
    if (shadow) shadow[i] = __float2bfloat16_rn(v);
  }
}

// ------------------------------------------------------------------ launchers

int umma_gemm(const void* A, int64_t lda, bool a_mn, const void* B, int64_t ldb, bool b_mn,
              void* C, int64_t ldc, int M, int N, int K, const int32_t* M_dev,
              const int32_t* K_dev, int epi, const float* bias, int split, cudaStream_t s);
int umma_gemm_mask(const void* A, int64_t lda, const void* B, int64_t ldb, __nv_bfloat16* C,
                   int64_t ldc, int M, int N, int K, const int32_t* M_dev,
                   const __nv_bfloat16* mask, int ldm, float* colsum, cudaStream_t s);
int umma_top(const void* agg, const void* WlT, const void* Wb, const float* bias, const void* WcT,
             const void* Wcp, void* h, void* dl, void* dz, float* dagg, int cap, int H, int C,
             int inL, const int32_t* M_dev, const int64_t* roots, uint64_t label_state,
             const int32_t* labels, float* loss, float* gb, cudaStream_t s);
int umma_head_ce(const void* A, int64_t lda, const void* B, int64_t ldb, float* logits, int C,
                 int n_cap, int K, const int32_t* M_dev, const int64_t* roots, uint64_t label_state,
                 float* loss, __nv_bfloat16* dl_lowp, int ldp, cudaStream_t s);

static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (!g_num_sms) g_num_sms = 148;
  }
  return g_num_sms;
}

template <typename TA, bool AT, bool BT, int EPI, typename TC, typename TM>
static void gemm(cudaStream_t s, const TA* A, int lda, const float* B, int ldb, TC* C, int ldc,
                 const int32_t* M_dev, int M_cap, int N, const int32_t* K_dev, int K_cap,
                 const float* bias, const TM* mask, int ldm, int split) {
  dim3 grid((N + BN - 1) / BN, (M_cap + BM - 1) / BM, split);
  count_launch();
  k_gemm<TA, AT, BT, EPI, TC, TM><<<grid, 256, 0, s>>>(A, lda, B, ldb, C, ldc, M_dev, M_cap, N,
                                                       K_dev, K_cap, bias, mask, ldm);
}

// Layer-k gather + aggregate (k == 1 reads features: local table, staged
// remote rows or peer tables).  pad: zero the rows up to the next 64 for the
// tensor-core weight-gradient reduction.
// hg_set_side_budget: layer-1 feature rows are streamed with an L2
// evict-first policy so the gather (the largest HBM stream of the loop) does
// not evict the training chain's working set from L2
static int g_agg_stream = 1;

template <typename T>
static RowSrc<T> row_src(const hg_step_desc* d, int k) {
  const T* src = k == 1 ? (const T*)d->features : (const T*)d->h[k - 1];
  const int Wd = k == 1 ? d->feat_ld : d->hidden;
  // layer 1: pair lists by vertex id (one dependent load fewer per source row),
  // or, staged with resolved handles, need-index lists into the handles
  const bool hnd = k == 1 && d->row_handle && d->stage_base;
  const bool vid = k == 1 && d->mg.nbr_vid1 && d->mg.self_vid1 && !hnd;
  return RowSrc<T>{src, Wd, k == 1 ? d->mg.need_ids[0] : nullptr, k == 1 ? d->feat_row : nullptr,
                   k == 1 ? (const T* const*)d->feat_peers : nullptr, d->feat_home,
                   (const T*)d->stage_base, k == 1 ? d->stage_row : nullptr, d->rank, vid,
                   hnd ? d->row_handle : nullptr, k == 1 && g_agg_stream != 0};
}

// Layer-k gather + aggregate for n steps sharing one row source (k == 1
// reads features: local table, staged remote rows or peer tables; n > 1 only
// for layer 1 of run-ahead groups).  pad: zero the rows up to the next 64 for
// the tensor-core weight-gradient reduction.
// resident CTAs per SM of a grouped (run-ahead) layer-1 gather: it runs beside
// the training branch, so it must leave registers for the training kernels
// (hg_set_side_budget)
static int g_agg_group_ctas = HG_AGG_MINB;

template <typename T>
static void launch_aggregate_n(const hg_step_desc* const* ds, int n, int k, cudaStream_t s,
                               bool pad) {
  const hg_step_desc* d = ds[0];
  const int H = d->hidden;
  const int Wd = k == 1 ? d->feat_ld : H;
  AggSegs<T> segs{};
  int cap = 1;
  for (int b = 0; b < n; ++b) {
    const hg_step_desc* e = ds[b];
    const bool hnd = k == 1 && e->row_handle && e->stage_base;
    const bool vid = k == 1 && e->mg.nbr_vid1 && e->mg.self_vid1 && !hnd;
    segs.handle[b] = hnd ? e->row_handle : nullptr;
    segs.self_pos[b] = vid ? e->mg.self_vid1 : e->mg.self_pos[k];
    segs.nbr_off[b] = e->mg.nbr_off[k];
    segs.nbr_idx[b] = vid ? e->mg.nbr_vid1 : e->mg.nbr_idx[k];
    segs.n_rows[b] = e->mg.totals + k;
    segs.cap[b] = e->max_rows[k];
    segs.out[b] = (T*)e->agg[k];
    cap = std::max(cap, e->max_rows[k]);
  }
  // rows per CTA: 8 warps x (32 / lanes per row); blocks past the device row count exit
  const int nvec = Wd / (16 / (int)sizeof(T));
  const int lanes = nvec >= 32 ? 32 : nvec >= 16 ? 16 : nvec >= 8 ? 8 : nvec >= 4 ? 4 : nvec >= 2 ? 2 : 1;
  const int rows_per_cta = 8 * (32 / lanes);
  // a group of segments: one resident wave split over them, warps loop over
  // their rows (the software pipeline pays off); one segment: a warp per
  // row group over the capacity (every row's chain in flight at once)
  const int wave = n > 1 ? std::max(1, num_sms() * g_agg_group_ctas / n) : num_sms() * 32;
  dim3 grid(std::max(1, std::min((cap + rows_per_cta - 1) / rows_per_cta, wave)), n);
  const int pad_cap = pad && sizeof(T) == 2 ? d->max_rows[k] : 0;
  prof_begin(k == 1 ? PROF_AGG1 : PROF_AGG2, s);
  count_launch();
  if (d->arch == 1)
    launch_pdl(k_aggregate<T, true>, dim3(grid), dim3(256), 0, s, row_src<T>(d, k), segs, Wd, d->in_dim[k], pad_cap);
  else
    launch_pdl(k_aggregate<T, false>, dim3(grid), dim3(256), 0, s, row_src<T>(d, k), segs, Wd, d->in_dim[k], pad_cap);
  prof_end(k == 1 ? PROF_AGG1 : PROF_AGG2, s);
}

template <typename T>
static void launch_aggregate(const hg_step_desc* d, int k, cudaStream_t s, bool pad) {
  launch_aggregate_n<T>(&d, 1, k, s, pad);
}

constexpr size_t kScatterSmem = 96 * 1024;

template <typename T>
static void scatter_root_attrs() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(k_scatter_root<true, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kScatterSmem);
  cudaFuncSetAttribute(k_scatter_root<false, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kScatterSmem);
  done = true;
}

// Variant switch (hg_set_fused_head): 1 puts the softmax-CE in the tcgen05 head
// GEMM's epilogue (umma_head_ce; tested, measured slower on B200 -- the head
// GEMM has only n_roots / 128 CTAs, the separate kernel a warp per root).
static int g_fused_head = 0;
static bool fused_head_on() { return g_fused_head != 0; }
// Opt-in (hg_set_fused_top): training steps run the top of the network
// (layer-L GEMM through the dX GEMM of layer L) as one kernel per 128 roots
// (k_umma_top).  Measured on B200 at the papers shape (phase timestamps,
// scripts/bench_train.py HG_TOP_TRACE=1): 27 us per launch against ~19.5 us
// for the six split kernels in the replayed graph -- each CTA streams all
// four weight operands (~870 KB) through one SM and runs 128 rows of
// epilogue work (softmax, masks, column sums) on that SM, where the split
// kernels spread both over 24-128 CTAs.  The parity tests run both paths.
static int g_fused_top = 0;

// bf16 dz operand of layer k (per-layer region when lowp_layered)
static inline bf16* dz_lowp(const hg_step_desc* d, int k) {
  int64_t rows = 0;
  if (d->lowp_layered)
    for (int j = 1; j < k; ++j) rows += d->max_rows[j];
  return (bf16*)d->lowp_scratch + rows * d->hidden;
}

// Forked stream of the backward pass: weight-gradient GEMMs (gW_c, gW_k for
// k >= 2) depend on nothing later in the step but the final SGD, so they run
// beside the dX -> scatter chain (joined at the end of the step; event
// fork/join is captured as graph edges).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t ev[2 * HG_MAX_LAYERS + 4];
};
static SideStream* side_stream() {
  static std::mutex mu;
  static SideStream per_dev[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  SideStream& ss = per_dev[dev & 63];
  if (!ss.s) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&ss.s, cudaStreamNonBlocking, hi) != cudaSuccess) return nullptr;
    for (auto& e : ss.ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  }
  return &ss;
}

template <typename T>
static int run_step(const hg_step_desc* d, int n_roots, cudaStream_t s, bool backward) {
  const int L = d->n_layers;
  const bool sage = d->arch == 1;
  const int H = d->hidden, C = d->n_classes;
  const int32_t* tot = d->mg.totals;  // N_0..N_L on device
  const int nb = num_sms() * 4;
  // tensor-core path: bf16 operands, H a multiple of 64 up to 256 (one N tile)
  const bool tc = sizeof(T) == 2 && d->use_tc && H % 64 == 0 && H <= 256;
  scatter_root_attrs<T>();
  // forked weight-gradient GEMMs (one side stream; joined before returning)
  SideStream* side = backward && tc ? side_stream() : nullptr;
  int n_fork = 0;
  auto fork = [&]() -> cudaStream_t {
    if (!side || n_fork >= 2 * HG_MAX_LAYERS + 2) return s;
    cudaEventRecord(side->ev[n_fork], s);
    cudaStreamWaitEvent(side->s, side->ev[n_fork], 0);
    ++n_fork;
    return side->s;
  };
  auto join = [&]() {
    if (!n_fork) return;
    cudaEventRecord(side->ev[n_fork], side->s);
    cudaStreamWaitEvent(s, side->ev[n_fork], 0);
    n_fork = 0;
  };
  const int Cp = (C + 63) / 64 * 64;
  const bool tc_head = tc && C <= 256 && d->WcT && d->Wcp && d->dl_lowp;
  // fused top (k_umma_top): layer-L linear, head, softmax-CE, dz_L, dagg_L
  const bool top_fused = backward && tc_head && g_fused_top && L >= 2 &&
                         (d->in_dim[L] == H || d->in_dim[L] == 2 * H) && d->Wb[L] &&
                         C <= 192;
  // ---- forward
  prof_begin(PROF_STEP, s);
  if (tc && !d->lowp_fresh) {
    for (int k = 1; k <= L; ++k) {
      dim3 g((H + 31) / 32, (d->in_dim[k] + 31) / 32), b(32, 8);
      count_launch();
      k_transpose_bf16<<<g, b, 0, s>>>(d->W[k], d->in_dim[k], H, (bf16*)d->Wlp[k],
                                       backward && k >= 2 ? (bf16*)d->Wb[k] : nullptr);
    }
  }
  for (int k = 1; k <= L; ++k) {
    if (k > 1 || !d->agg1_ready) launch_aggregate<T>(d, k, s, tc && backward);
    if (k == L && top_fused) {
      if (!d->lowp_fresh) {
        dim3 g((C + 31) / 32, (H + 31) / 32), b(32, 8);
        count_launch(2);
        k_transpose_bf16<<<g, b, 0, s>>>(d->Wc, H, C, (bf16*)d->WcT, nullptr);
        k_pad_bf16<<<64, 256, 0, s>>>(d->Wc, H, C, (bf16*)d->Wcp, Cp);
      }
      int st = umma_top(d->agg[L], d->Wlp[L], d->Wb[L], d->b[L], d->WcT, d->Wcp, d->h[L],
                        d->dl_lowp, dz_lowp(d, L), d->dagg, d->max_rows[L], H, C, d->in_dim[L],
                        tot + L, d->roots, d->label_state, d->labels, d->loss, d->gb[L], s);
      if (st) { join(); return st; }
      // gW_c += h_Lᵀ dlogits, beside the rest of the backward
      const int split = std::max(1, std::min(16, n_roots / 256));
      st = umma_gemm(d->h[L], H, true, d->dl_lowp, Cp, true, d->gWc, C, H, C, n_roots, nullptr,
                     tot + L, 2, nullptr, split, fork());
      if (st) { join(); return st; }
      break;
    }
    if (k == 1) prof_begin(PROF_GEMM1, s);
    if (tc) {
      int st = umma_gemm(d->agg[k], d->in_dim[k], false, d->Wlp[k], d->in_dim[k], false, d->h[k], H,
                         d->max_rows[k], H, d->in_dim[k], tot + k, nullptr, 1, d->b[k], 1, s);
      if (st) { join(); return st; }
    } else {
      gemm<T, false, false, EPI_BIAS_RELU, T, T>(s, (const T*)d->agg[k], d->in_dim[k], d->W[k], H,
                                                 (T*)d->h[k], H, tot + k, d->max_rows[k], H,
                                                 nullptr, d->in_dim[k], d->b[k], nullptr, 0, 1);
    }
    if (k == 1) prof_end(PROF_GEMM1, s);
  }
  // classifier head (model.py:246, 253-265)
  if (top_fused) {
    // done by k_umma_top
  } else if (tc_head) {
    // logits = h_L @ W_c on tcgen05 (B = W_cᵀ bf16, K-major); softmax-CE writes
    // dlogits (f32 in place + bf16 padded copy for the backward GEMMs)
    if (!d->lowp_fresh) {
      dim3 g((C + 31) / 32, (H + 31) / 32), b(32, 8);
      count_launch(2);
      k_transpose_bf16<<<g, b, 0, s>>>(d->Wc, H, C, (bf16*)d->WcT, nullptr);
      k_pad_bf16<<<64, 256, 0, s>>>(d->Wc, H, C, (bf16*)d->Wcp, Cp);
    }
    // root rows: n_roots is the capacity, the device count N_L the actual roots
    int st;
    if (C <= 192 && fused_head_on() && !d->labels) {
      st = umma_head_ce(d->h[L], H, d->WcT, H, d->logits, C, n_roots, H, tot + L, d->roots,
                        d->label_state, d->loss, (bf16*)d->dl_lowp, Cp, s);
      if (st) { join(); return st; }
    } else {
    st = umma_gemm(d->h[L], H, false, d->WcT, H, false, d->logits, C, n_roots, C, H,
                       tot + L, nullptr, 0, nullptr, 1, s);
    if (st) { join(); return st; }
    count_launch();
    launch_pdl(k_softmax_ce, dim3((n_roots + 7) / 8), dim3(256), 0, s, d->logits, C, d->roots, n_roots, tot + L,
                                                   d->label_state, d->labels, d->loss,
                                                   (bf16*)d->dl_lowp, Cp);
    }
    if (backward) {
      // dz_L = bf16((dlogits @ W_cᵀ) * (h_L > 0)) and gb_L += its column sums, in
      // the dz GEMM's epilogue (no f32 dh_L round trip, no k_mask_colsum); the
      // rows past the root count come out zero for the dW GEMM's reduction
      // (the f32 dh_L is still produced where a SIMT dX GEMM of layer L would read it)
      if (L == 1 || (d->in_dim[L] % 64 == 0 && d->Wb[L])) {
        // rows up to the next multiple of 64 (within the capacity): the dW GEMM's
        // reduction reads them, so they are stored (as zeros past the root count)
        const int mrows = std::min(d->max_rows[L], (n_roots + 63) / 64 * 64);
        st = umma_gemm_mask(d->dl_lowp, Cp, d->Wcp, Cp, dz_lowp(d, L), H, mrows, H, Cp, tot + L,
                            (const bf16*)d->h[L], H, d->gb[L], s);
        if (st) { join(); return st; }
      } else {
        st = umma_gemm(d->dl_lowp, Cp, false, d->Wcp, Cp, false, d->dh[L], H, n_roots, H, Cp,
                       tot + L, nullptr, 0, nullptr, 1, s);
        if (st) { join(); return st; }
        dim3 g((H + 31) / 32, 16);
        count_launch();
        launch_pdl(k_mask_colsum<T>, dim3(g), dim3(256), 0, s, d->dh[L], (const T*)d->h[L], tot + L,
                   H, d->gb[L], dz_lowp(d, L), d->max_rows[L]);
      }
      // gW_c += h_Lᵀ dlogits (both MN-major, reduction over the roots), forked
      const int split = std::max(1, std::min(16, n_roots / 256));
      st = umma_gemm(d->h[L], H, true, d->dl_lowp, Cp, true, d->gWc, C, H, C, n_roots,
                     nullptr, tot + L, 2, nullptr, split, fork());
      if (st) { join(); return st; }
    }
  } else {
    const size_t smem = ((size_t)H * (C | 1) + H + 8 * H + 8 * C) * sizeof(float);
    static size_t smem_set = 0;
    if (smem > 48 * 1024 && smem > smem_set) {
      cudaFuncSetAttribute(k_head<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      smem_set = smem;
    }
    const int grid = std::max(1, std::min(num_sms(), (n_roots + 7) / 8));
    count_launch();
    k_head<T><<<grid, 256, smem, s>>>((const T*)d->h[L], d->Wc, H, C, d->roots, n_roots,
                                      tot + L, d->label_state, d->labels, d->logits, d->loss,
                                      d->dh[L],
                                      tc ? dz_lowp(d, L) : nullptr, d->max_rows[L],
                                      d->gb[L], backward ? 1 : 0);
  }
  if (!backward) { prof_end(PROF_STEP, s); return HG_OK; }
  // ---- backward (model.py:262-285)
  const int split_r = std::max(1, std::min(32, n_roots / 64));
  // gWc += h_L^T dlogits
  if (!tc_head)
    gemm<T, true, false, EPI_ATOMIC, float, T>(s, (const T*)d->h[L], H, d->logits, C, d->gWc, C,
                                               nullptr, H, C, tot + L, n_roots, nullptr, nullptr,
                                               0, split_r);
  for (int k = L; k >= 1; --k) {
    // gW_k += agg_k^T dz_k   (reduction over the N_k rows, split across CTAs)
    if (k == 1) prof_begin(PROF_DW1, s);
    if (tc) {
      // both operands MN-major straight from their row-major buffers
      const int kblocks = (d->max_rows[k] + 63) / 64;
      const int tiles = (d->in_dim[k] + 127) / 128;
      int split = (kblocks + 5) / 6;
      split = std::max(1, std::min(split, std::max(1, num_sms() / tiles)));
      // layers >= 2 (own dz region): beside the dX -> scatter chain
      cudaStream_t ws = k >= 2 && d->lowp_layered ? fork() : s;
      int st = umma_gemm(d->agg[k], d->in_dim[k], true, dz_lowp(d, k), H, true, d->gW[k], H,
                         d->in_dim[k], H, d->max_rows[k], nullptr, tot + k, 2, nullptr, split, ws);
      if (st) { join(); return st; }
    } else {
      gemm<T, true, false, EPI_ATOMIC, float, T>(s, (const T*)d->agg[k], d->in_dim[k], d->dh[k], H,
                                                 d->gW[k], H, nullptr, d->in_dim[k], H, tot + k,
                                                 d->max_rows[k], nullptr, nullptr, 0,
                                                 k == L ? split_r : d->split_k);
    }
    if (k == 1) { prof_end(PROF_DW1, s); break; }  // layer-1 dX is unused (features are not trainable)
    // dagg_k = dz_k W_k^T
    if (k == L && top_fused) {
      // written by k_umma_top
    } else if (tc && d->in_dim[k] % 64 == 0 && d->Wb[k]) {
      int st = umma_gemm(dz_lowp(d, k), H, false, d->Wb[k], H, false, d->dagg, d->in_dim[k],
                         d->max_rows[k], d->in_dim[k], H, tot + k, nullptr, 0, nullptr, 1, s);
      if (st) { join(); return st; }
    } else {
      gemm<float, false, true, EPI_STORE, float, T>(s, d->dh[k], H, d->W[k], H, d->dagg,
                                                    d->in_dim[k], tot + k, d->max_rows[k],
                                                    d->in_dim[k], nullptr, H, nullptr, nullptr, 0,
                                                    1);
    }
    if (k == L && H % 8 == 0 && H <= 256) {
      // top layer: per-row map, no scatter (k_scatter_top)
      const bool tc_dx = tc && d->in_dim[k - 1] % 64 == 0 && d->Wb[k - 1];
      const bool want_f32 = !tc || (k - 1 >= 2 && !tc_dx);
      const int grid = std::max(1, std::min((n_roots + 7) / 8, num_sms() * 4));
      count_launch();
      auto kern = sage ? k_scatter_top<true, T> : k_scatter_top<false, T>;
      launch_pdl(kern, dim3(grid), dim3(256), 0, s, (const float*)d->dagg, d->in_dim[k],
                 (const int32_t*)d->mg.need_off[k - 1], (const int32_t*)d->mg.need_off[k],
                 (const int32_t*)d->mg.self_pos[k], (const int32_t*)d->mg.nbr_off[k],
                 (const int8_t*)d->mg.in_layer[k - 1], n_roots, H,
                 (const T*)d->h[k - 1], want_f32 ? d->dh[k - 1] : nullptr,
                 tc ? dz_lowp(d, k - 1) : nullptr, d->gb[k - 1], tot + (k - 1),
                 d->max_rows[k - 1]);
      continue;
    }
    const size_t root_smem = (size_t)d->root_rows[k - 1] * H * sizeof(float);
    if (d->root_rows[k - 1] > 0 && root_smem <= kScatterSmem && H <= 512) {
      // f32 dz is only needed where a SIMT GEMM consumes it (layer k-1's dX)
      const bool tc_dx = tc && d->in_dim[k - 1] % 64 == 0 && d->Wb[k - 1];
      const bool want_f32 = !tc || (k - 1 >= 2 && !tc_dx);
      const int grid = n_roots;  // one CTA per root: every root's latency chain in flight at once
      count_launch();
      if (sage)
        launch_pdl(k_scatter_root<true, T>, dim3(grid), dim3(256), root_smem, s, 
            d->dagg, d->in_dim[k], d->mg.need_off[k - 1], d->mg.need_off[k], d->mg.self_pos[k],
            d->mg.nbr_off[k], d->mg.nbr_idx[k], n_roots, H, (const T*)d->h[k - 1],
            want_f32 ? d->dh[k - 1] : nullptr, tc ? dz_lowp(d, k - 1) : nullptr,
            d->gb[k - 1], tot + (k - 1), d->max_rows[k - 1]);
      else
        launch_pdl(k_scatter_root<false, T>, dim3(grid), dim3(256), root_smem, s, 
            d->dagg, d->in_dim[k], d->mg.need_off[k - 1], d->mg.need_off[k], d->mg.self_pos[k],
            d->mg.nbr_off[k], d->mg.nbr_idx[k], n_roots, H, (const T*)d->h[k - 1],
            want_f32 ? d->dh[k - 1] : nullptr, tc ? dz_lowp(d, k - 1) : nullptr,
            d->gb[k - 1], tot + (k - 1), d->max_rows[k - 1]);
      continue;
    }
    count_launch(3);
    k_zero_rows<<<nb, 256, 0, s>>>(d->dh[k - 1], tot + (k - 1), H);
    const int grid = (d->max_rows[k] + 7) / 8;
    if (sage)
      k_scatter<true><<<grid, 256, 0, s>>>(d->dagg, d->in_dim[k], d->mg.self_pos[k],
                                           d->mg.nbr_off[k], d->mg.nbr_idx[k], tot + k, H,
                                           d->dh[k - 1]);
    else
      k_scatter<false><<<grid, 256, 0, s>>>(d->dagg, d->in_dim[k], d->mg.self_pos[k],
                                            d->mg.nbr_off[k], d->mg.nbr_idx[k], tot + k, H,
                                            d->dh[k - 1]);
    dim3 g((H + 31) / 32, 64);
    launch_pdl(k_mask_colsum<T>, dim3(g), dim3(256), 0, s, d->dh[k - 1], (const T*)d->h[k - 1], tot + (k - 1), H,
                                       d->gb[k - 1], tc ? dz_lowp(d, k - 1) : nullptr,
                                       d->max_rows[k - 1]);
  }
  join();
  prof_end(PROF_STEP, s);
  return HG_OK;
}

static int validate(const hg_step_desc* d, int n_roots) {
  if (d->n_layers < 1 || d->n_layers > HG_MAX_LAYERS) return hg_fail(HG_ECONFIG, "bad n_layers");
  if (n_roots < 1 || n_roots > d->max_roots) return hg_fail(HG_ERANGE, "bad n_roots %d", n_roots);
  if (d->feat_ld % 8 || d->hidden % 8) return hg_fail(HG_ECONFIG, "feat_ld and hidden must be multiples of 8");
  if (d->act_dtype != 0 && d->act_dtype != 1) return hg_fail(HG_ECONFIG, "bad act_dtype");
  return HG_OK;
}

}  // namespace hg

using namespace hg;

extern "C" int hg_set_fused_top(int32_t on) {
  hg::g_fused_top = on != 0;
  return HG_OK;
}

extern "C" int hg_set_side_budget(int32_t agg_ctas_per_sm, int32_t agg_stream) {
  if (agg_ctas_per_sm < 1 || agg_ctas_per_sm > HG_AGG_MINB)
    return hg_fail(HG_ECONFIG, "agg_ctas_per_sm must be 1..%d", HG_AGG_MINB);
  g_agg_group_ctas = agg_ctas_per_sm;
  g_agg_stream = agg_stream != 0;
  return HG_OK;
}

extern "C" int hg_set_fused_head(int32_t on) {
  g_fused_head = on ? 1 : 0;
  return HG_OK;
}

extern "C" int hg_train_step(const hg_step_desc* d, int32_t n_roots, void* stream) {
  int st = validate(d, n_roots);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  st = d->act_dtype == 0 ? run_step<float>(d, n_roots, s, true) : run_step<bf16>(d, n_roots, s, true);
  if (st) return st;
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_step_prologue(const hg_step_desc* d, int32_t n_roots, int32_t backward,
                                void* stream) {
  return hg_step_prologue_group(&d, 1, backward, stream);
}

extern "C" int hg_step_prologue_group(const hg_step_desc* const* ds, int32_t n, int32_t backward,
                                      void* stream) {
  if (n < 1 || n > HG_MAX_GROUP) return hg_fail(HG_ERANGE, "bad group size %d", n);
  const hg_step_desc* d = ds[0];
  for (int b = 0; b < n; ++b) {
    int st = validate(ds[b], ds[b]->max_roots);
    if (st) return st;
    const hg_step_desc* e = ds[b];
    if (e->features != d->features || e->feat_row != d->feat_row || e->feat_ld != d->feat_ld ||
        e->stage_base != d->stage_base || e->stage_row != d->stage_row ||
        e->feat_peers != d->feat_peers || e->act_dtype != d->act_dtype || e->arch != d->arch ||
        (e->row_handle && e->stage_base) != (d->row_handle && d->stage_base) ||
        e->in_dim[1] != d->in_dim[1] || e->max_rows[1] != d->max_rows[1])
      return hg_fail(HG_ECONFIG, "grouped prologue: steps must share the feature source");
  }
  cudaStream_t s = (cudaStream_t)stream;
  const bool tc = d->act_dtype == 1 && d->use_tc && d->hidden % 64 == 0 && d->hidden <= 256;
  if (d->act_dtype == 0) launch_aggregate_n<float>(ds, n, 1, s, false);
  else launch_aggregate_n<bf16>(ds, n, 1, s, tc && backward);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_forward(const hg_step_desc* d, int32_t n_roots, void* stream) {
  int st = validate(d, n_roots);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  st = d->act_dtype == 0 ? run_step<float>(d, n_roots, s, false) : run_step<bf16>(d, n_roots, s, false);
  if (st) return st;
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

// The SGD + bf16-refresh plan of a step's parameters (flat buffer layout
// W_1..W_L, b_1..b_L, W_c; model.py:299-324): one 32 x 32 tile list over the
// weight matrices with the destinations of their bf16 operand copies.
int hg::make_sgd_plan(const hg_step_desc* d, float* params, int64_t n, SgdPlan* out) {
  const int L = d->n_layers, H = d->hidden, C = d->n_classes, Cp = (C + 63) / 64 * 64;
  SgdPlan P{};
  int tiles = 0;
  auto add = [&](int64_t off, int rows, int cols, bf16* tdst, int64_t tld, bf16* sdst,
                 int64_t sld) {
    SgdMat& M = P.m[P.n_mats++];
    M.off = off; M.rows = rows; M.cols = cols;
    M.tdst = tdst; M.tld = tld; M.sdst = sdst; M.sld = sld;
    M.tiles_c = (cols + 31) / 32;
    M.tile0 = tiles;
    tiles += ((rows + 31) / 32) * M.tiles_c;
  };
  for (int k = 1; k <= L; ++k) {
    const int64_t off = d->W[k] - params;
    if (off < 0 || off + (int64_t)d->in_dim[k] * H > n)
      return hg_fail(HG_ECONFIG, "layer %d weights outside the flat parameter buffer", k);
    // Wlp: Wᵀ [H x in_k] (K-major B of the forward GEMM); Wb: W (B of the dX GEMM, k >= 2)
    add(off, d->in_dim[k], H, (bf16*)d->Wlp[k], d->in_dim[k], k >= 2 ? (bf16*)d->Wb[k] : nullptr, H);
  }
  const int64_t off_c = d->Wc - params;
  if (off_c < 0 || off_c + (int64_t)H * C > n)
    return hg_fail(HG_ECONFIG, "classifier outside the flat parameter buffer");
  add(off_c, H, C, (bf16*)d->WcT, H, (bf16*)d->Wcp, Cp);  // WcT [C x H], Wcp [H x Cp]
  P.n_tiles = tiles;
  // the biases sit between the last layer weight and the classifier
  P.plain_lo = d->b[1] - params;
  P.plain_hi = d->b[L] - params + H;
  if (P.plain_lo < 0 || P.plain_hi > n || P.plain_hi < P.plain_lo)
    return hg_fail(HG_ECONFIG, "biases outside the flat parameter buffer");
  *out = P;
  return HG_OK;
}

extern "C" int hg_sgd_refresh(const hg_step_desc* d, float* params, float* grads, int64_t n,
                              float lr, float inv_batch, int32_t update, void* stream) {
  if (n <= 0) return HG_OK;
  if (!d->WcT || !d->Wcp) return hg_fail(HG_ECONFIG, "hg_sgd_refresh needs the bf16 head operands");
  SgdPlan P{};
  int st = make_sgd_plan(d, params, n, &P);
  if (st) return st;
  const int grid = P.n_tiles + 4;
  count_launch();
  prof_begin(PROF_SGD, (cudaStream_t)stream);
  launch_pdl(k_sgd_refresh, dim3(grid), dim3(256), 0, (cudaStream_t)stream, params, grads, lr,
             inv_batch, update, P);
  prof_end(PROF_SGD, (cudaStream_t)stream);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

extern "C" int hg_sgd_update(float* params, float* grads, void* shadow_bf16, int64_t n, float lr,
                             float inv_batch, void* stream) {
  if (n <= 0) return HG_OK;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  count_launch();
  prof_begin(PROF_SGD, (cudaStream_t)stream);
  launch_pdl(k_sgd, dim3(grid), dim3(256), 0, (cudaStream_t)stream, params, grads, (bf16*)shadow_bf16, n, lr, inv_batch);
  prof_end(PROF_SGD, (cudaStream_t)stream);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}
