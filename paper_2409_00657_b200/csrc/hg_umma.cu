// bf16 GEMM on the 5th-generation tensor cores: TMA -> smem (128B swizzle)
// -> tcgen05.mma (one elected thread) -> fp32 accumulator in TMEM ->
// tcgen05.ld epilogue.  The layer linear of the SAGE/GCN step (model.py:236,
// agg @ W + b; backward aggᵀ dz, model.py:263) is the only dense
// contraction of the path; this kernel runs it.
//
//   C[M x N] = A(m,k) * B(k,n), fp32 accumulate
//   A K-major : A is [M x K] row-major          A MN-major : A is [K x M] row-major
//   B K-major : B is [N x K] row-major          B MN-major : B is [K x N] row-major
//
// One CTA owns a 128 x BN_T (<= 256) output tile, 4-warp CTA:
//   warp 0 lane 0 : TMA producer (kStages-deep mbarrier ring)
//   warp 1 lane 0 : MMA issuer (4 x UMMA_K=16 per 64-wide K block)
//   warp 2        : TMEM allocator
//   warps 0..3    : epilogue (TMEM lane quadrant = warp % 4 = output rows)
// K may be split across gridDim.z (the weight-gradient reduction over graph
// rows); split partials are accumulated with vector float atomics.
// Row counts can be device-resident (micrograph batches vary per step): rows
// beyond the device count are masked in the epilogue, and producers keep the
// padding rows of reduction operands zero.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "hg_tc.cuh"

namespace hg {

// Pipeline depth: 4 stages, 3 for 256-wide tiles (144 KB instead of 192 KB of
// shared memory, so a GEMM CTA fits on an SM beside the build CTAs that run
// concurrently in the graph loop; the K ranges here are 4-8 blocks, and the
// 128 KB f32 epilogue staging still fits).
#ifndef HG_UMMA_STAGES_256
#define HG_UMMA_STAGES_256 3
#endif
__host__ __device__ constexpr int stages_for(int bn) { return bn >= 256 ? HG_UMMA_STAGES_256 : 4; }

enum UEpi { UEPI_STORE_F32 = 0, UEPI_BIAS_RELU_BF16 = 1, UEPI_ATOMIC_F32 = 2, UEPI_SOFTMAX_CE = 3,
            UEPI_MASK_BF16 = 4 };

struct UmmaArgs {
  int M, N, K;               // host-known sizes (M/K may be overridden on device)
  const int32_t* M_dev;      // optional device row count for M (A K-major) ...
  const int32_t* K_dev;      // ... or for K (reduction over rows, MN-major operands)
  void* C;
  int64_t ldc;
  const float* bias;
  int tma_epi;               // 1: epilogue through smem + TMA store/reduce (map_c valid)
  // UEPI_SOFTMAX_CE (classifier head, model.py:253-265): one N tile holds a
  // root's whole logit row, so the epilogue thread of that row does the
  // softmax-CE: loss, dlogits (f32 in C) and the bf16 padded copy.
  const int64_t* roots;
  uint64_t label_state;
  float* loss;
  __nv_bfloat16* dl_lowp;
  int ldp;                   // dl_lowp row pitch (classes rounded up to 64)
  int n_cap;                 // capacity rows: [M_dev, n_cap) get zeros
  int late_m;                // host: every capacity tile fits one wave, M_dev read late
  // UEPI_MASK_BF16 (dz of the top layer, model.py:266-272): C = bf16(acc * (h > 0)),
  // colsum[c] += sum over the rows of the masked values (bias gradient)
  const __nv_bfloat16* mask;  // h [rows x ldm] bf16
  int ldm;
  float* colsum;
};

// Rows [r0, r1) of the head outputs past the device root count: no loss, no gradient.
__device__ __forceinline__ void head_zero_row(const UmmaArgs& a, int row) {
  float* x = reinterpret_cast<float*>(a.C) + (int64_t)row * a.ldc;
  for (int c = 0; c < a.N; ++c) x[c] = 0.f;
  for (int c = 0; c < a.ldp; ++c) a.dl_lowp[(int64_t)row * a.ldp + c] = __float2bfloat16_rn(0.f);
  a.loss[row] = 0.f;
}

#ifndef HG_UMMA_THREADS
#define HG_UMMA_THREADS 256
#endif
constexpr int kUmmaThreads = HG_UMMA_THREADS;  // 4 warps (roles + epilogue) or 8 (two epilogue warps per lane quadrant)
constexpr int kEpiPerQ = kUmmaThreads / 128;

template <bool A_MN, bool B_MN, int BN_T, int EPI>
__global__ void __launch_bounds__(kUmmaThreads, 1)
k_umma_gemm(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
            const __grid_constant__ CUtensorMap map_c, UmmaArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-aligned stage ring
  // 1024-byte aligned by pointer arithmetic on the shared array (an integer
  // round trip would turn every access into a generic one)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int A_BYTES = BM_T * BK_T * 2;
  constexpr int B_BYTES = BN_T * BK_T * 2;
  constexpr int STAGE = A_BYTES + B_BYTES;
  constexpr int kStages = stages_for(BN_T);
  constexpr uint32_t kTmemCols = BN_T <= 32 ? 32 : BN_T <= 64 ? 64 : BN_T <= 128 ? 128 : 256;
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages], done_bar;
  __shared__ uint32_t tmem_base_sh;
  __shared__ float bias_s[EPI == UEPI_BIAS_RELU_BF16 ? BN_T : 1];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM_T, n0 = blockIdx.y * BN_T;
  pdl_trigger();
  // prologue that reads nothing a predecessor writes -- barrier init and the
  // tensor-map prefetch -- overlaps the previous kernel's tail (programmatic
  // dependent launch); everything after pdl_wait() may read its outputs
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  pdl_wait();
  // Forward GEMMs (device row count, host K): the row count only matters to
  // the epilogue, so the mainloop starts without waiting for that dependent
  // load -- every capacity tile runs (one wave), tiles past the count skip
  // their stores.  Reductions (device K) need K before the first load.
  constexpr bool kSoftmax = EPI == UEPI_SOFTMAX_CE;
  const bool late_m = args.late_m && args.M_dev && !args.K_dev && !kSoftmax;
  // issued now, first consumed in the epilogue when late_m
  const int M_ld = args.M_dev ? __ldcg(args.M_dev) : args.M;
  int M = late_m ? args.M : M_ld;
  const int K = args.K_dev ? *args.K_dev : args.K;
  // K range of this split, in 64-wide blocks
  const int kblocks = (K + BK_T - 1) / BK_T;
  const int per = (kblocks + gridDim.z - 1) / gridDim.z;
  const int kb0 = blockIdx.z * per;
  const int kb1 = min(kblocks, kb0 + per);
  if ((!late_m && m0 >= M) || kb0 >= kb1) {  // whole CTA exits together (before any TMEM is held)
    if constexpr (EPI == UEPI_SOFTMAX_CE)
      if (m0 >= M)
        for (int row = m0 + threadIdx.x; row < min(m0 + BM_T, args.n_cap); row += blockDim.x)
          head_zero_row(args, row);
    return;
  }
  const int nk = kb1 - kb0;
  if constexpr (EPI == UEPI_BIAS_RELU_BF16) {
    for (int c = threadIdx.x; c < BN_T; c += blockDim.x)
      bias_s[c] = n0 + c < args.N ? args.bias[n0 + c] : 0.f;
  }
  // TMEM is allocated only after the predecessor completed: a CTA holding TMEM
  // while waiting could starve a still-running predecessor CTA of its columns
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    for (int i = 0; i < nk; ++i) {
      const int s = i % kStages;
      if (i >= kStages) mbar_wait(&empty_bar[s], ((i / kStages) - 1) & 1);
      uint8_t* sa = smem + s * STAGE;
      uint8_t* sb = sa + A_BYTES;
      const int k0 = (kb0 + i) * BK_T;
      mbar_expect_tx(&full_bar[s], STAGE);
      if (A_MN) {
#pragma unroll
        for (int b = 0; b < BM_T / 64; ++b) tma_load_2d(sa + b * 64 * 128, &map_a, &full_bar[s], m0 + 64 * b, k0);
      } else {
        tma_load_2d(sa, &map_a, &full_bar[s], k0, m0);
      }
      if (B_MN) {
#pragma unroll
        for (int b = 0; b < BN_T / 64; ++b) tma_load_2d(sb + b * 64 * 128, &map_b, &full_bar[s], n0 + 64 * b, k0);
      } else {
        tma_load_2d(sb, &map_b, &full_bar[s], k0, n0);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer
    constexpr uint32_t idesc = make_idesc(BN_T, A_MN, B_MN);
    for (int i = 0; i < nk; ++i) {
      const int s = i % kStages;
      mbar_wait(&full_bar[s], (i / kStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t sa = smem_u32(smem + s * STAGE);
      const uint32_t sb = sa + A_BYTES;
#pragma unroll
      for (int kk = 0; kk < BK_T / 16; ++kk) {
        // K-major: +32 B per 16-wide K step inside the swizzle row (LBO unused)
        // MN-major: rows are K; 16 rows = two 1024-B atoms; LBO = 64-wide MN block
        const uint64_t ad = A_MN ? make_desc(sa + kk * 2048, 64 * 128, 1024)
                                 : make_desc(sa + kk * 32, 16, 1024);
        const uint64_t bd = B_MN ? make_desc(sb + kk * 2048, 64 * 128, 1024)
                                 : make_desc(sb + kk * 32, 16, 1024);
        umma_bf16(tmem, ad, bd, idesc, (i > 0 || kk > 0) ? 1u : 0u);
      }
      umma_commit(&empty_bar[s]);  // frees the stage when these MMAs retire
    }
    umma_commit(&done_bar);
  }
  // ---------------- epilogue: TMEM lane quadrant wq = warp % 4; on the TMA path
  // the kEpiPerQ warps of a quadrant take alternate column chunks, the other
  // paths use warps 0-3
  __syncwarp();
  const int wq = warp & 3, half = warp >> 2;
  const bool epi_on = half == 0 || (EPI != UEPI_SOFTMAX_CE && args.tma_epi);
  M = M_ld;
  if (epi_on) {
  mbar_wait(&done_bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = m0 + wq * 32 + lane;
  const bool valid = row < M;
  if constexpr (EPI == UEPI_SOFTMAX_CE) {
    // one TMEM sweep (4 loads in flight, warp-uniform) copies each thread's
    // logit row into the idle pipeline smem (odd pitch: bank-conflict free);
    // max / sum-exp / gradient then run from smem, and the warp stores its
    // 32 rows coalesced
    const uint32_t tb = tmem + ((uint32_t)(warp * 32) << 16);
    const int C = args.N;
    const int P = C | 1;
    float* stg = reinterpret_cast<float*>(smem) + warp * 32 * P;
    float* mine = stg + lane * P;
#pragma unroll 1
    for (int cb = 0; cb < C; cb += 64) {
      uint32_t r[64];
#pragma unroll
      for (int q = 0; q < 64; q += 16) tmem_ld16_issue(tb + cb + q, r + q);
#pragma unroll
      for (int q = 0; q < 64; q += 16) tmem_wait16(r + q);
#pragma unroll
      for (int j = 0; j < 64; ++j)
        if (cb + j < C) mine[cb + j] = __uint_as_float(r[j]);
    }
    const int label = valid ? (int)(mix64(args.label_state ^ (uint64_t)args.roots[row]) % (uint64_t)C) : 0;
    float mx = -INFINITY, sum = 0.f;
    for (int c = 0; c < C; ++c) mx = fmaxf(mx, mine[c]);
    const float xl = mine[label];
    for (int c = 0; c < C; ++c) sum += expf(mine[c] - mx);
    const float inv = 1.0f / sum;
    for (int c = 0; c < C; ++c)
      mine[c] = valid ? expf(mine[c] - mx) * inv - (c == label ? 1.f : 0.f) : 0.f;
    if (valid) args.loss[row] = logf(sum) - (xl - mx);
    else if (row < args.n_cap) args.loss[row] = 0.f;
    __syncwarp();
    const int r0 = m0 + warp * 32;
    for (int i = 0; i < 32 && r0 + i < args.n_cap; ++i) {
      float* xo = reinterpret_cast<float*>(args.C) + (int64_t)(r0 + i) * args.ldc;
      __nv_bfloat16* lo = args.dl_lowp + (int64_t)(r0 + i) * args.ldp;
      for (int c = lane; c < args.ldp; c += 32) {
        const float g = c < C ? stg[i * P + c] : 0.f;
        if (c < C) xo[c] = g;
        lo[c] = __float2bfloat16_rn(g);
      }
    }
  } else if (args.tma_epi) {
    // Coalesced epilogue: each warp stages its 32 rows x (128-byte column
    // chunk) in the now idle pipeline smem, 128B-swizzled, and one lane hands
    // the box to TMA (store, or f32 add-reduce in L2 for split-K partials).
    // Rows past the device count are written as zeros (inside the capacity).
    constexpr bool kBf16Out = EPI == UEPI_BIAS_RELU_BF16 || EPI == UEPI_MASK_BF16;
    constexpr int EB = kBf16Out ? 2 : 4;
    constexpr int CW = 128 / EB;             // columns per 128-byte row
    constexpr int NCH = (BN_T + CW - 1) / CW;
    constexpr int NCW = (NCH + kEpiPerQ - 1) / kEpiPerQ;  // chunks per warp
    uint8_t* stage = smem + warp * (NCW * 4096);
    // A warp whose 32 rows all lie past the device count still stores (zeros):
    // the weight-gradient GEMMs reduce over rows up to the next multiple of 64
    // and read those padding rows (a reduce-add of zeros would only cost time)
    const bool warp_rows = m0 < M && (EPI != UEPI_ATOMIC_F32 || m0 + wq * 32 < M);
#pragma unroll 1
    for (int ch = half; ch < NCH; ch += kEpiPerQ) {
      const int c = ch * CW;
      if (n0 + c >= args.N || !warp_rows) break;
      uint32_t rr[CW];
#pragma unroll
      for (int q = 0; q < CW; q += 16)
        tmem_ld16_issue(tmem + ((uint32_t)(wq * 32) << 16) + c + q, rr + q);
#pragma unroll
      for (int q = 0; q < CW; q += 16) tmem_wait16(rr + q);
      uint8_t* box = stage + (ch / kEpiPerQ) * 4096 + lane * 128;
      if constexpr (EPI == UEPI_MASK_BF16) {
        // this row's 64 h columns (loads in flight together), mask, bf16,
        // and the column sums of the masked values (butterfly over the warp's
        // 32 rows, one atomic per column per warp)
        const __nv_bfloat16* hp = args.mask + (int64_t)(valid ? row : 0) * args.ldm + n0 + c;
        uint4 hraw[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) hraw[u] = *reinterpret_cast<const uint4*>(hp + u * 8);
#pragma unroll
        for (int g16 = 0; g16 < 4; ++g16) {
          float v[16];
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int u = g16 * 2 + h2;
            const uint32_t hw[4] = {hraw[u].x, hraw[u].y, hraw[u].z, hraw[u].w};
            uint32_t pk[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const float m0 = __uint_as_float(hw[t] << 16), m1 = __uint_as_float(hw[t] & 0xFFFF0000u);
              const float x0 = valid && m0 > 0.f ? __uint_as_float(rr[u * 8 + 2 * t]) : 0.f;
              const float x1 = valid && m1 > 0.f ? __uint_as_float(rr[u * 8 + 2 * t + 1]) : 0.f;
              v[h2 * 8 + 2 * t] = x0;
              v[h2 * 8 + 2 * t + 1] = x1;
              pk[t] = pack_bf2(x0, x1);
            }
            *reinterpret_cast<uint4*>(box + ((u ^ (lane & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
          const float cs = colsum16(v, lane);
          const int col = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 +
                          ((lane >> 1) & 1);
          if ((lane & 1) == 0 && n0 + c + g16 * 16 + col < args.N)
            atomicAdd(args.colsum + n0 + c + g16 * 16 + col, cs);
        }
      } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        uint4 v;
        if constexpr (EPI == UEPI_BIAS_RELU_BF16) {
          uint32_t pk[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int cc = c + u * 8 + 2 * j;
            const float x0 = valid ? fmaxf(__uint_as_float(rr[u * 8 + 2 * j]) + bias_s[cc], 0.f) : 0.f;
            const float x1 = valid ? fmaxf(__uint_as_float(rr[u * 8 + 2 * j + 1]) + bias_s[cc + 1], 0.f) : 0.f;
            const __nv_bfloat162 t = __floats2bfloat162_rn(x0, x1);
            pk[j] = *reinterpret_cast<const uint32_t*>(&t);
          }
          v = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        } else {
          v = valid ? make_uint4(rr[u * 4], rr[u * 4 + 1], rr[u * 4 + 2], rr[u * 4 + 3])
                    : make_uint4(0, 0, 0, 0);
        }
        *reinterpret_cast<uint4*>(box + ((u ^ (lane & 7)) << 4)) = v;
      }
      }  // not UEPI_MASK_BF16
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        tma_store_2d<EPI == UEPI_ATOMIC_F32>(&map_c, stage + (ch / kEpiPerQ) * 4096, n0 + c, m0 + wq * 32);
    }
    if (lane == 0) {
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncwarp();
  } else {
  constexpr int CH = BN_T % 64 == 0 ? 64 : 16;  // columns per TMEM round trip
#pragma unroll 1
  for (int cb = 0; cb < BN_T; cb += CH) {
    uint32_t rr[CH];
#pragma unroll
    for (int q = 0; q < CH; q += 16)
      tmem_ld16_issue(tmem + ((uint32_t)(warp * 32) << 16) + cb + q, rr + q);
#pragma unroll
    for (int q = 0; q < CH; q += 16) tmem_wait16(rr + q);
#pragma unroll
  for (int q = 0; q < CH; q += 16) {
    const uint32_t* r = rr + q;
    const int c = cb + q;
    if (!valid) continue;
    const int col = n0 + c;
    if (col >= args.N) continue;
    if constexpr (EPI == UEPI_BIAS_RELU_BF16) {
      __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(args.C) + (int64_t)row * args.ldc + col;
      uint32_t pk[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float x0 = fmaxf(__uint_as_float(r[2 * j]) + args.bias[col + 2 * j], 0.f);
        const float x1 = fmaxf(__uint_as_float(r[2 * j + 1]) + args.bias[col + 2 * j + 1], 0.f);
        const __nv_bfloat162 t = __floats2bfloat162_rn(x0, x1);
        pk[j] = *reinterpret_cast<const uint32_t*>(&t);
      }
      reinterpret_cast<uint4*>(out)[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      reinterpret_cast<uint4*>(out)[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
    } else if constexpr (EPI == UEPI_ATOMIC_F32) {
      float* out = reinterpret_cast<float*>(args.C) + (int64_t)row * args.ldc + col;
      const int nv = min(16, args.N - col);  // partial last chunk (N not a multiple of 16)
      if (nv == 16 && (args.ldc & 3) == 0) {  // float4 only on 16-byte aligned rows
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          atomicAdd(reinterpret_cast<float4*>(out + j),
                    make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])));
      } else {
        for (int j = 0; j < nv; ++j) atomicAdd(out + j, __uint_as_float(r[j]));
      }
    } else {
      float* out = reinterpret_cast<float*>(args.C) + (int64_t)row * args.ldc + col;
      const int nv = min(16, args.N - col);
      if (nv == 16 && (args.ldc & 3) == 0) {
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(out + j) =
              make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                          __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
      } else {
        for (int j = 0; j < nv; ++j) out[j] = __uint_as_float(r[j]);
      }
    }
  }
  }
  }  // row-per-thread epilogue
  }  // epi_on
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
}

// ------------------------------------------------------------------ host side

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                             const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                             const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 2D bf16 tensor map: inner dim (contiguous) x outer dim, row pitch in elements.
int make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t pitch,
                    uint32_t box_inner, uint32_t box_outer, int elem_bytes) {
  struct Key {
    const void* p; uint64_t a, b, c; uint32_t d, e; int f;
    bool operator==(const Key& o) const {
      return p == o.p && a == o.a && b == o.b && c == o.c && d == o.d && e == o.e && f == o.f;
    }
  };
  struct H {
    size_t operator()(const Key& k) const {
      return std::hash<const void*>()(k.p) ^ (k.a * 1315423911u) ^ (k.b << 7) ^ (k.c << 13) ^
             ((uint64_t)k.d << 29) ^ ((uint64_t)k.e << 41);
    }
  };
  static std::mutex mu;
  static std::unordered_map<Key, CUtensorMap, H> cache;
  Key key{base, inner, outer, pitch, box_inner, box_outer, elem_bytes};
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) { *m = it->second; return HG_OK; }
  EncodeFn enc = encoder();
  if (!enc) return hg_fail(HG_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {pitch * (uint64_t)elem_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return hg_fail(HG_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  cache.emplace(key, *m);
  return HG_OK;
}

template <bool A_MN, bool B_MN, int BN_T, int EPI>
static int launch_t(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
                    const UmmaArgs& a, int split, cudaStream_t s) {
  constexpr int smem = stages_for(BN_T) * (BM_T * BK_T * 2 + BN_T * BK_T * 2) + 1024;
  auto kern = k_umma_gemm<A_MN, B_MN, BN_T, EPI>;
  static bool attr = false;
  if (!attr) {
    HG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  dim3 grid((a.M + BM_T - 1) / BM_T, (a.N + BN_T - 1) / BN_T, split);
  count_launch();
  HG_CUDA_TRY(launch_pdl(kern, grid, dim3(kUmmaThreads), smem, s, ma, mb, mc, a));
  return HG_OK;
}

// Generic entry: shapes are capacities (M/K) when *_dev counts are given.
static int umma_gemm_ex(const void* A, int64_t lda, bool a_mn, const void* B, int64_t ldb,
                        bool b_mn, void* C, int64_t ldc, int M, int N, int K,
                        const int32_t* M_dev, const int32_t* K_dev, int epi, const float* bias,
                        int split, const __nv_bfloat16* mask, int ldm, float* colsum,
                        cudaStream_t s) {
  if (N <= 0 || (N > 256 && N % 256)) return hg_fail(HG_ECONFIG, "umma N must be <= 256 or a multiple of 256");
  // N tile (grid.y covers the rest): the widest tile that still spreads the
  // problem over about half the SMs -- small-M GEMMs (one micrograph batch of
  // roots) otherwise run on a handful of SMs, each streaming all of B
  int bn = N > 256 ? 256 : (N + 63) / 64 * 64;
  {
    const int mt = (M + BM_T - 1) / BM_T;
    auto ctas = [&](int b) { return mt * ((N + b - 1) / b) * std::max(split, 1); };
    static int sms = [] {
      int dev = 0, n = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
      return n > 0 ? n : 148;
    }();
    while (bn > 64 && ctas(bn) < sms / 2) bn = bn == 192 ? 128 : bn / 2;
  }
  if (lda % 8 || ldb % 8) return hg_fail(HG_ECONFIG, "umma leading dims must be multiples of 8");
  CUtensorMap ma, mb;
  int st;
  // A: K-major [M x K] -> inner K; MN-major [K x M] -> inner M
  if (a_mn) st = make_map(&ma, A, (uint64_t)M, (uint64_t)K, lda, 64, BK_T);
  else st = make_map(&ma, A, (uint64_t)K, (uint64_t)M, lda, BK_T, BM_T);
  if (st) return st;
  if (b_mn) st = make_map(&mb, B, (uint64_t)N, (uint64_t)K, ldb, 64, BK_T);
  else st = make_map(&mb, B, (uint64_t)K, (uint64_t)N, ldb, BK_T, (uint32_t)bn);
  if (st) return st;
  // TMA epilogue when C's rows are 16-byte aligned (else row-per-thread stores)
  CUtensorMap mc;
  const int eb = (epi == UEPI_BIAS_RELU_BF16 || epi == UEPI_MASK_BF16) ? 2 : 4;
  int tma_epi = ((uintptr_t)C % 16 == 0 && (ldc * eb) % 16 == 0) ? 1 : 0;
  if (tma_epi && make_map(&mc, C, (uint64_t)N, (uint64_t)M, ldc, 128 / eb, 32, eb) != HG_OK) {
    tma_epi = 0;
  }
  if (!tma_epi) memset(&mc, 0, sizeof(mc));
  if (epi == UEPI_MASK_BF16 && !tma_epi)
    return hg_fail(HG_ECONFIG, "masked dz epilogue needs 16-byte aligned bf16 rows");
  UmmaArgs a{M, N, K, M_dev, K_dev, C, ldc, bias, tma_epi};
  a.mask = mask;
  a.ldm = ldm;
  a.colsum = colsum;
  {
    // late row count only while every capacity tile fits one wave: tiles past
    // the count then run on otherwise idle SMs; beyond a wave they would queue
    // (multi-GPU capacities hold several batches' rows)
    static int sms_ = [] {
      int dev = 0, n = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
      return n > 0 ? n : 148;
    }();
    const int64_t ctas = (int64_t)((M + BM_T - 1) / BM_T) * ((N + bn - 1) / bn) * std::max(split, 1);
    a.late_m = ctas <= sms_ ? 1 : 0;
  }

#define HG_UMMA_CASE(AM, BMJ, BNV, E)                                                       \
  if (a_mn == AM && b_mn == BMJ && bn == BNV && epi == E)                                   \
    return launch_t<AM, BMJ, BNV, E>(ma, mb, mc, a, split, s);
#define HG_UMMA_N(AM, BMJ, E) \
  HG_UMMA_CASE(AM, BMJ, 64, E) HG_UMMA_CASE(AM, BMJ, 128, E) HG_UMMA_CASE(AM, BMJ, 192, E) HG_UMMA_CASE(AM, BMJ, 256, E)
  HG_UMMA_N(false, false, UEPI_BIAS_RELU_BF16)
  HG_UMMA_N(false, false, UEPI_STORE_F32)
  HG_UMMA_N(true, true, UEPI_ATOMIC_F32)
  HG_UMMA_N(true, true, UEPI_STORE_F32)
  HG_UMMA_N(false, false, UEPI_MASK_BF16)
#undef HG_UMMA_N
#undef HG_UMMA_CASE
  return hg_fail(HG_ECONFIG, "unsupported umma variant (a_mn=%d b_mn=%d N=%d epi=%d)", (int)a_mn,
                 (int)b_mn, N, epi);
}

int umma_gemm(const void* A, int64_t lda, bool a_mn, const void* B, int64_t ldb, bool b_mn,
              void* C, int64_t ldc, int M, int N, int K, const int32_t* M_dev,
              const int32_t* K_dev, int epi, const float* bias, int split, cudaStream_t s) {
  return umma_gemm_ex(A, lda, a_mn, B, ldb, b_mn, C, ldc, M, N, K, M_dev, K_dev, epi, bias, split,
                      nullptr, 0, nullptr, s);
}

// dz = bf16((A @ B) * (mask > 0)) with colsum += the masked column sums (both
// operands K-major): the top layer's dz GEMM with k_mask_colsum folded in.
int umma_gemm_mask(const void* A, int64_t lda, const void* B, int64_t ldb, __nv_bfloat16* C,
                   int64_t ldc, int M, int N, int K, const int32_t* M_dev,
                   const __nv_bfloat16* mask, int ldm, float* colsum, cudaStream_t s) {
  return umma_gemm_ex(A, lda, false, B, ldb, false, C, ldc, M, N, K, M_dev, nullptr,
                      UEPI_MASK_BF16, nullptr, 1, mask, ldm, colsum, s);
}

// Classifier head with the softmax-CE fused into the epilogue: logits
// [n_cap x C] = h_L [n_cap x K] @ W_c (B = W_cᵀ bf16, K-major), C <= 192 so
// one N tile covers every class.  Replaces umma_gemm + k_softmax_ce.
int umma_head_ce(const void* A, int64_t lda, const void* B, int64_t ldb, float* logits, int C,
                 int n_cap, int K, const int32_t* M_dev, const int64_t* roots, uint64_t label_state,
                 float* loss, __nv_bfloat16* dl_lowp, int ldp, cudaStream_t s) {
  if (C <= 0 || C > 192) return hg_fail(HG_ECONFIG, "fused head needs 1 <= classes <= 192");
  if (lda % 8 || ldb % 8) return hg_fail(HG_ECONFIG, "umma leading dims must be multiples of 8");
  CUtensorMap ma, mb, mc;
  int st = make_map(&ma, A, (uint64_t)K, (uint64_t)n_cap, lda, BK_T, BM_T);
  if (st) return st;
  st = make_map(&mb, B, (uint64_t)K, (uint64_t)C, ldb, BK_T, 192u);
  if (st) return st;
  memset(&mc, 0, sizeof(mc));
  UmmaArgs a{n_cap, C, K, M_dev, nullptr, logits, C, nullptr, 0,
             roots, label_state, loss, dl_lowp, ldp, n_cap};
  return launch_t<false, false, 192, UEPI_SOFTMAX_CE>(ma, mb, mc, a, 1, s);
}


// ------------------------------------------------------------ fused top step
// The top of the step for one 128-root tile in ONE kernel (model.py:236-285
// for k = L plus the head): five dependent GEMM/epilogue stages that used to
// be six launches (layer-L GEMM, head GEMM, softmax-CE, dz GEMM, mask +
// column sums, dX GEMM), each a latency-bound grid of <= 32 CTAs.
//   1. acc[0,H)      = agg_L  @ W_L            -> h_L = bf16(relu(. + b_L))
//   2. acc[H,H+Cn)   = h_L    @ W_c            -> softmax-CE: loss, dlogits (bf16)
//   3. acc[0,H)      = dl     @ W_cᵀ           -> dz_L = . * (h_L > 0), gb_L += colsum
//   4. acc[0,inL)    = dz_L   @ W_Lᵀ           -> dagg_L (f32, for k_scatter_top)
// h_L, dl and dz_L live in shared memory in the UMMA K-major 128B-swizzled
// layout (each is the next stage's A operand) and leave through TMA stores
// (h_L, dl and dz_L for the weight-gradient GEMMs, dagg_L for the scatter).
// Warp roles: warp 0 lane 0 streams every stage's weight tiles through a
// 2-deep ring (it runs ahead into the next stage while an epilogue runs),
// warp 1 lane 0 issues the MMAs, warps 2-17 are the epilogue (TMEM lane
// quadrant = warp % 4, one root row per lane, four warps per quadrant splitting
// the columns; a thread-per-row epilogue on four warps spent ~30 us of
// dependent per-thread work on the softmax and masks).  Numerics are the split
// kernels' (same operands, same rounding points); only the order of the
// softmax and column sums differs.
struct TopArgs {
  int n_cap;               // root capacity (rows of every operand)
  const int32_t* M_dev;    // device root count N_L
  int H, C, Cn, Cp, inL;   // hidden, classes, classes rounded to 16 / to 64, layer-L input width
  const float* bias;       // b_L [H]
  const int64_t* roots;
  uint64_t label_state;
  const int32_t* labels;   // explicit labels or null (hashed)
  float* loss;             // [n_cap]
  float* gb;               // gb_L [H] (accumulated)
  int64_t* trace;          // optional phase timestamps of CTA 0 (hg_top_trace)
};
static int64_t* g_top_trace = nullptr;

__device__ __forceinline__ void top_stamp(const TopArgs& a, int i) {
  if (a.trace && blockIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[i] = (int64_t)t;
  }
}

constexpr int kTopSlices = 4;                      // epilogue warps per TMEM lane quadrant
constexpr int kTopEpiWarps = 4 * kTopSlices;
constexpr int kTopThreads = 64 + 32 * kTopEpiWarps;  // producer + MMA warps + epilogue
constexpr int kTopA = BM_T * BK_T * 2;         // 16 KB
constexpr int kTopStage = kTopA + 256 * BK_T * 2;  // + 32 KB B tile

__device__ __forceinline__ void epi_sync() {  // the epilogue warps only
  asm volatile("bar.sync 1, %0;" ::"n"(32 * kTopEpiWarps) : "memory");
}
__global__ void __launch_bounds__(kTopThreads, 1)
k_umma_top(const __grid_constant__ CUtensorMap map_agg, const __grid_constant__ CUtensorMap map_w,
           const __grid_constant__ CUtensorMap map_wct, const __grid_constant__ CUtensorMap map_wcp,
           const __grid_constant__ CUtensorMap map_wb, const __grid_constant__ CUtensorMap map_h,
           const __grid_constant__ CUtensorMap map_dl, const __grid_constant__ CUtensorMap map_dz,
           const __grid_constant__ CUtensorMap map_dagg, TopArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned by pointer arithmetic on the shared array (an integer
  // round trip would turn every access into a generic one)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // Layout: slots 0-1 [0, 96K) always; dl at 96K; h_L / dz_L at
  // max(96K + |dl|, 144K).  The load ring has four 48 KB slots while the first
  // GEMM runs (slots 2-3 overlay dl and h_L, both idle then), three during the
  // head and dX GEMMs (slot 2 overlays dl) and two during the dz GEMM (dl is
  // its A operand): phase p's loads cycle over top_slot(p, i).
  uint8_t* dls = smem + 2 * kTopStage;
  uint8_t* hs = smem + max(2 * kTopStage + (a.Cp / 64) * 16384, 3 * kTopStage);
  __shared__ __align__(8) uint64_t full_bar[4], empty_bar[4];
  __shared__ __align__(8) uint64_t acc_bar[4], opnd_bar[3];
  __shared__ uint32_t tmem_base_sh;
  __shared__ float bias_s[256];
  __shared__ float red[4][256];
  __shared__ float part[2][kTopSlices][BM_T];  // per-slice softmax max / sum-exp
  __shared__ float xl_s[BM_T];                 // label logit per row

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM_T;
  const int H = a.H, C = a.C, Cn = a.Cn, Cp = a.Cp, inL = a.inL;
  pdl_trigger();
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int p = 0; p < 4; ++p) mbar_init(&acc_bar[p], 1);
    for (int p = 0; p < 3; ++p) mbar_init(&opnd_bar[p], 32 * kTopEpiWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    const CUtensorMap* maps[5] = {&map_agg, &map_w, &map_wct, &map_wcp, &map_wb};
    for (auto m : maps)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
  }
  pdl_wait();
  const int M = *a.M_dev;
  if (m0 >= M) {  // no roots in this tile: zero its loss rows, no TMEM taken
    for (int r = m0 + threadIdx.x; r < min(m0 + BM_T, a.n_cap); r += blockDim.x) a.loss[r] = 0.f;
    return;
  }
  for (int c = threadIdx.x; c < H; c += blockDim.x) bias_s[c] = a.bias[c];
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;
  const int kb_in = inL / 64, kb_h = H / 64, kb_c = Cp / 64, n_half = (inL + 255) / 256;
  // slot of the i-th load of phase p (see the layout above)
  auto top_slot = [](int p, int i) { return p == 0 ? i & 3 : p == 2 ? i & 1 : (i + 2) % 3; };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: every stage's tiles, in MMA order
      int uses[4] = {0, 0, 0, 0}, n = 0;
      top_stamp(a, 0);
      auto acquire = [&](int p, int i, uint32_t bytes) -> uint8_t* {
        const int s = top_slot(p, i);
        if (uses[s] > 0) mbar_wait(&empty_bar[s], (uses[s] - 1) & 1);
        ++uses[s];
        if (n < 31) top_stamp(a, 1 + n);
        ++n;
        mbar_expect_tx(&full_bar[s], bytes);
        return smem + s * kTopStage;
      };
      for (int kb = 0; kb < kb_in; ++kb) {
        uint8_t* st = acquire(0, kb, kTopA + H * 128);
        tma_load_2d(st, &map_agg, &full_bar[top_slot(0, kb)], kb * 64, m0);
        tma_load_2d(st + kTopA, &map_w, &full_bar[top_slot(0, kb)], kb * 64, 0);
      }
      for (int kb = 0; kb < kb_h; ++kb) {
        uint8_t* st = acquire(1, kb, Cn * 128);
        tma_load_2d(st + kTopA, &map_wct, &full_bar[top_slot(1, kb)], kb * 64, 0);
      }
      for (int kb = 0; kb < kb_c; ++kb) {
        uint8_t* st = acquire(2, kb, H * 128);
        tma_load_2d(st + kTopA, &map_wcp, &full_bar[top_slot(2, kb)], kb * 64, 0);
      }
      mbar_wait(&acc_bar[2], 0);  // slot 2 overlays dl, the dz GEMM's A operand
      for (int hf = 0, i = 0; hf < n_half; ++hf) {
        const int nb = min(256, inL - hf * 256);
        for (int kb = 0; kb < kb_h; ++kb, ++i) {
          uint8_t* st = acquire(3, i, nb * 128);
          tma_load_2d(st + kTopA, &map_wb, &full_bar[top_slot(3, i)], kb * 64, hf * 256);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      int uses[4] = {0, 0, 0, 0}, n = 0;
      auto consume = [&](int p, int i) -> uint32_t {
        const int s = top_slot(p, i);
        mbar_wait(&full_bar[s], uses[s] & 1);
        ++uses[s];
        if (n < 32) top_stamp(a, 32 + n);
        ++n;
        asm volatile("tcgen05.fence::after_thread_sync;");
        return smem_u32(smem + s * kTopStage);
      };
      auto mma_k64 = [&](uint32_t d, uint32_t sa, uint32_t sb, uint32_t idesc, bool first) {
#pragma unroll
        for (int kk = 0; kk < BK_T / 16; ++kk)
          umma_bf16(d, make_desc(sa + kk * 32, 16, 1024), make_desc(sb + kk * 32, 16, 1024), idesc,
                    (!first || kk > 0) ? 1u : 0u);
      };
      // 1. agg_L @ W_L  -> TMEM [0, H)
      for (int kb = 0; kb < kb_in; ++kb) {
        const uint32_t st = consume(0, kb);
        mma_k64(tmem, st, st + kTopA, make_idesc(H, false, false), kb == 0);
        umma_commit(&empty_bar[top_slot(0, kb)]);
      }
      umma_commit(&acc_bar[0]);
      // 2. h_L @ W_c  -> TMEM [H, H + Cn)
      mbar_wait(&opnd_bar[0], 0);
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int kb = 0; kb < kb_h; ++kb) {
        const uint32_t st = consume(1, kb);
        mma_k64(tmem + H, smem_u32(hs + kb * 16384), st + kTopA, make_idesc(Cn, false, false), kb == 0);
        umma_commit(&empty_bar[top_slot(1, kb)]);
      }
      umma_commit(&acc_bar[1]);
      // 3. dl @ W_cᵀ  -> TMEM [0, H)
      mbar_wait(&opnd_bar[1], 0);
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int kb = 0; kb < kb_c; ++kb) {
        const uint32_t st = consume(2, kb);
        mma_k64(tmem, smem_u32(dls + kb * 16384), st + kTopA, make_idesc(H, false, false), kb == 0);
        umma_commit(&empty_bar[top_slot(2, kb)]);
      }
      umma_commit(&acc_bar[2]);
      // 4. dz_L @ W_Lᵀ  -> TMEM [0, inL), 256 columns per MMA
      mbar_wait(&opnd_bar[2], 0);
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int hf = 0, i = 0; hf < n_half; ++hf) {
        const int nb = min(256, inL - hf * 256);
        for (int kb = 0; kb < kb_h; ++kb, ++i) {
          const uint32_t st = consume(3, i);
          mma_k64(tmem + hf * 256, smem_u32(hs + kb * 16384), st + kTopA, make_idesc(nb, false, false),
                  kb == 0);
          umma_commit(&empty_bar[top_slot(3, i)]);
        }
      }
      umma_commit(&acc_bar[3]);
    }
  } else {
    // ---------------- epilogue warps 2..17: four per TMEM lane quadrant q (one
    // root row per lane), the columns dealt out over the four (slice j)
    const int q = warp & 3, j = (warp - 2) >> 2;
    const int et = (warp - 2) * 32 + lane;  // 0..511
    const int rl = q * 32 + lane;           // row in the tile
    const int row = m0 + rl;
    const bool valid = row < M;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    const bool leader = warp == 2 && lane == 0;
    if (leader) top_stamp(a, 72);
    // 1. h_L = bf16(relu(acc + b)) -> hs (A operand of 2, TMA store to h_L)
    mbar_wait(&acc_bar[0], 0);
    if (leader) top_stamp(a, 64);
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c32 = j; c32 < H / 32; c32 += kTopSlices) {
      uint32_t r[32];
      tmem_ld16_issue(tl + c32 * 32, r);
      tmem_ld16_issue(tl + c32 * 32 + 16, r + 16);
      tmem_wait16(r);
      tmem_wait16(r + 16);
      uint8_t* base = hs + (c32 >> 1) * 16384;
#pragma unroll
      for (int uu = 0; uu < 4; ++uu) {
        const int u = (c32 & 1) * 4 + uu;
        uint32_t pk[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int c = c32 * 32 + uu * 8 + 2 * t;
          const float x0 = valid ? fmaxf(__uint_as_float(r[uu * 8 + 2 * t]) + bias_s[c], 0.f) : 0.f;
          const float x1 = valid ? fmaxf(__uint_as_float(r[uu * 8 + 2 * t + 1]) + bias_s[c + 1], 0.f) : 0.f;
          pk[t] = pack_bf2(x0, x1);
        }
        *reinterpret_cast<uint4*>(base + sw128(rl, u)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    mbar_arrive(&opnd_bar[0]);
    if (leader) top_stamp(a, 65);
    epi_sync();
    if (leader) {
      for (int c64 = 0; c64 < kb_h; ++c64) tma_store_2d<false>(&map_h, hs + c64 * 16384, c64 * 64, m0);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    // 2. softmax-CE over the C logits of this row (model.py:253-259); each
    //    slice takes 16-column groups g = j, j + 4, ...; max and sum-exp are
    //    combined across the four slices in shared memory
    mbar_wait(&acc_bar[1], 0);
    if (leader) top_stamp(a, 66);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tcl = tl + H;
    // this slice's 16-column groups g = j + 4t held in registers across the
    // three passes (one TMEM sweep, one exponential per logit)
    constexpr int kG = 192 / 16 / kTopSlices;
    float xv[kG][16];
    float mx = -INFINITY;
    // (C is uniform: only the last group needs per-column guards)
#pragma unroll
    for (int t = 0; t < kG; ++t) {
      const int c16 = (j + kTopSlices * t) * 16;
      if (c16 < Cn) {
        uint32_t r[16];
        tmem_ld16(tcl + c16, r);
#pragma unroll
        for (int e = 0; e < 16; ++e) xv[t][e] = __uint_as_float(r[e]);
        if (c16 + 16 <= C) {
#pragma unroll
          for (int e = 0; e < 16; ++e) mx = fmaxf(mx, xv[t][e]);
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (c16 + e < C) mx = fmaxf(mx, xv[t][e]);
        }
      }
    }
    if (leader) top_stamp(a, 73);
    part[0][j][rl] = mx;
    const int label = valid ? (a.labels ? a.labels[row]
                                        : (int)(mix64(a.label_state ^ (uint64_t)a.roots[row]) %
                                                (uint64_t)C))
                            : -1;
    if (leader) top_stamp(a, 74);
    epi_sync();
    if (leader) top_stamp(a, 75);
    mx = fmaxf(fmaxf(part[0][0][rl], part[0][1][rl]), fmaxf(part[0][2][rl], part[0][3][rl]));
    float sum = 0.f;
#pragma unroll
    for (int t = 0; t < kG; ++t) {
      const int c16 = (j + kTopSlices * t) * 16;
      if (c16 < Cn) {
        const unsigned lo = (unsigned)(label - c16);
        if (lo < 16u) {  // this row's label logit (one group per row)
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (e == (int)lo) xl_s[rl] = xv[t][e];
        }
        if (c16 + 16 <= C) {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            xv[t][e] = __expf(xv[t][e] - mx);
            sum += xv[t][e];
          }
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            xv[t][e] = c16 + e < C ? __expf(xv[t][e] - mx) : 0.f;
            sum += xv[t][e];
          }
        }
      }
    }
    part[1][j][rl] = sum;
    if (leader) top_stamp(a, 76);
    epi_sync();
    if (leader) top_stamp(a, 77);
    sum = (part[1][0][rl] + part[1][1][rl]) + (part[1][2][rl] + part[1][3][rl]);
    const float inv = valid ? 1.0f / sum : 0.f;  // capacity rows: dlogits 0
    // dlogits = softmax - onehot(label), bf16 into dl (the onehot term is
    // applied to the one label column afterwards)
#pragma unroll
    for (int t = 0; t < kG; ++t) {
      const int c16 = (j + kTopSlices * t) * 16;
      if (c16 >= Cp) continue;
      uint32_t pk[8];
      if (c16 + 16 <= C) {
#pragma unroll
        for (int q2 = 0; q2 < 8; ++q2) pk[q2] = pack_bf2(xv[t][2 * q2] * inv, xv[t][2 * q2 + 1] * inv);
      } else if (c16 < Cn) {
#pragma unroll
        for (int q2 = 0; q2 < 8; ++q2)
          pk[q2] = pack_bf2(c16 + 2 * q2 < C ? xv[t][2 * q2] * inv : 0.f,
                            c16 + 2 * q2 + 1 < C ? xv[t][2 * q2 + 1] * inv : 0.f);
      } else {
#pragma unroll
        for (int q2 = 0; q2 < 8; ++q2) pk[q2] = 0u;
      }
      uint8_t* base = dls + (c16 / 64) * 16384;
      const int u0 = (c16 % 64) / 8;
      *reinterpret_cast<uint4*>(base + sw128(rl, u0)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      *reinterpret_cast<uint4*>(base + sw128(rl, u0 + 1)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      if ((unsigned)(label - c16) < 16u) {
        const float g = __expf(xl_s[rl] - mx) * inv - 1.f;
        *reinterpret_cast<__nv_bfloat16*>(dls + (label / 64) * 16384 + sw128(rl, (label % 64) / 8) +
                                          (label % 8) * 2) = __float2bfloat16_rn(g);
      }
    }
    if (leader) top_stamp(a, 78);
    if (j == 0) {
      if (valid) a.loss[row] = logf(sum) - (xl_s[rl] - mx);
      else if (row < a.n_cap) a.loss[row] = 0.f;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    mbar_arrive(&opnd_bar[1]);
    if (leader) top_stamp(a, 67);
    epi_sync();
    if (leader) {
      for (int c64 = 0; c64 < kb_c; ++c64) tma_store_2d<false>(&map_dl, dls + c64 * 16384, c64 * 64, m0);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    // 3. dz_L = (dl @ W_cᵀ) * (h_L > 0) in place of h_L in hs; gb_L column sums
    mbar_wait(&acc_bar[2], 0);
    if (leader) top_stamp(a, 68);
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (leader) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // h_L store has read hs
    epi_sync();
    for (int c32 = j; c32 < H / 32; c32 += kTopSlices) {
      uint32_t r[32];
      tmem_ld16_issue(tl + c32 * 32, r);
      tmem_ld16_issue(tl + c32 * 32 + 16, r + 16);
      tmem_wait16(r);
      tmem_wait16(r + 16);
      uint8_t* base = hs + (c32 >> 1) * 16384;
#pragma unroll
      for (int g16 = 0; g16 < 2; ++g16) {
        float v[16];
#pragma unroll
        for (int uu = 0; uu < 2; ++uu) {
          const int ul = g16 * 2 + uu;          // unit within the 32 columns
          const int u = (c32 & 1) * 4 + ul;     // unit within the 64-column chunk
          uint4 hv = *reinterpret_cast<const uint4*>(base + sw128(rl, u));
          const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
          uint32_t pk[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const __nv_bfloat162 hb = *reinterpret_cast<const __nv_bfloat162*>(&hw[t]);
            const float x0 = valid && __low2float(hb) > 0.f ? __uint_as_float(r[ul * 8 + 2 * t]) : 0.f;
            const float x1 = valid && __high2float(hb) > 0.f ? __uint_as_float(r[ul * 8 + 2 * t + 1]) : 0.f;
            v[uu * 8 + 2 * t] = x0;
            v[uu * 8 + 2 * t + 1] = x1;
            pk[t] = pack_bf2(x0, x1);
          }
          *reinterpret_cast<uint4*>(base + sw128(rl, u)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
        const float cs = colsum16(v, lane);
        const int col = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
        if ((lane & 1) == 0) red[q][c32 * 32 + g16 * 16 + col] = cs;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    mbar_arrive(&opnd_bar[2]);
    if (leader) top_stamp(a, 69);
    epi_sync();
    if (leader) {
      for (int c64 = 0; c64 < kb_h; ++c64) tma_store_2d<false>(&map_dz, hs + c64 * 16384, c64 * 64, m0);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    for (int c = et; c < H; c += 32 * kTopEpiWarps)
      atomicAdd(a.gb + c, (red[0][c] + red[1][c]) + (red[2][c] + red[3][c]));
    // 4. dagg_L -> global f32 in 16 KB boxes (128 rows x 32 columns): the four
    //    warps of slice j (one per lane quadrant) fill a box, one of them
    //    hands it to TMA; two boxes per slice in flight
    mbar_wait(&acc_bar[3], 0);
    if (leader) top_stamp(a, 70);
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (leader) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // dl / dz stores done
    epi_sync();
    {
      uint8_t* stg = smem + j * 2 * 16384;  // slots 0-2 (idle now)
      const bool issuer = q == 2 && lane == 0;  // warp 2 + 4j
      int n = 0;
      for (int b = j; b < inL / 32; b += kTopSlices, ++n) {
        uint8_t* buf = stg + (n & 1) * 16384;
        if (n >= 2) {
          if (issuer) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          asm volatile("bar.sync %0, 128;" ::"r"(2 + j) : "memory");
        }
        uint32_t r[32];
        tmem_ld16_issue(tl + b * 32, r);
        tmem_ld16_issue(tl + b * 32 + 16, r + 16);
        tmem_wait16(r);
        tmem_wait16(r + 16);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          *reinterpret_cast<uint4*>(buf + sw128(rl, u)) =
              make_uint4(r[u * 4], r[u * 4 + 1], r[u * 4 + 2], r[u * 4 + 3]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync %0, 128;" ::"r"(2 + j) : "memory");
        if (issuer) {
          tma_store_2d<false>(&map_dagg, buf, b * 32, m0);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    if (leader) top_stamp(a, 71);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// Host side of k_umma_top.  Shapes: agg_L [cap x inL] bf16, W_L operand WlT
// [H x inL] (= W_Lᵀ, K-major), W_L straight copy Wb [inL x H], WcT [C x H],
// Wcp [H x Cp] (W_c zero-padded), h_L [cap x H] bf16, dl [cap x Cp] bf16,
// dz_L [cap x H] bf16, dagg [cap x inL] f32.
int umma_top(const void* agg, const void* WlT, const void* Wb, const float* bias, const void* WcT,
             const void* Wcp, void* h, void* dl, void* dz, float* dagg, int cap, int H, int C,
             int inL, const int32_t* M_dev, const int64_t* roots, uint64_t label_state,
             const int32_t* labels, float* loss, float* gb, cudaStream_t s) {
  const int Cn = (C + 15) / 16 * 16, Cp = (C + 63) / 64 * 64;
  if (H % 64 || H < 64 || H > 256) return hg_fail(HG_ECONFIG, "fused top: hidden must be 64..256, a multiple of 64");
  if (C < 1 || Cp > 192 || H + Cn > 512) return hg_fail(HG_ECONFIG, "fused top: needs 1 <= classes <= 192");
  if (inL % 64 || inL > 512) return hg_fail(HG_ECONFIG, "fused top: bad layer input width %d", inL);
  if (cap < 1) return HG_OK;
  CUtensorMap m_agg, m_w, m_wct, m_wcp, m_wb, m_h, m_dl, m_dz, m_dagg;
  int st;
  if ((st = make_map(&m_agg, agg, inL, cap, inL, BK_T, BM_T))) return st;
  if ((st = make_map(&m_w, WlT, inL, H, inL, BK_T, H))) return st;
  if ((st = make_map(&m_wct, WcT, H, C, H, BK_T, Cn))) return st;
  if ((st = make_map(&m_wcp, Wcp, Cp, H, Cp, BK_T, H))) return st;
  if ((st = make_map(&m_wb, Wb, H, inL, H, BK_T, std::min(256, inL)))) return st;
  if ((st = make_map(&m_h, h, H, cap, H, BK_T, BM_T))) return st;
  if ((st = make_map(&m_dl, dl, Cp, cap, Cp, BK_T, BM_T))) return st;
  if ((st = make_map(&m_dz, dz, H, cap, H, BK_T, BM_T))) return st;
  if ((st = make_map(&m_dagg, dagg, inL, cap, inL, 32, BM_T, 4))) return st;
  TopArgs a{cap, M_dev, H, C, Cn, Cp, inL, bias, roots, label_state, labels, loss, gb, g_top_trace};
  const int hs_off = std::max(2 * kTopStage + (Cp / 64) * 16384, 3 * kTopStage);
  const int smem = std::max(hs_off + (H / 64) * 16384, 4 * kTopStage) + 1024;
  static int attr = 0;
  if (smem > attr) {
    HG_CUDA_TRY(cudaFuncSetAttribute(k_umma_top, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = smem;
  }
  count_launch();
  HG_CUDA_TRY(launch_pdl(k_umma_top, dim3((cap + BM_T - 1) / BM_T), dim3(kTopThreads), smem, s, m_agg,
                         m_w, m_wct, m_wcp, m_wb, m_h, m_dl, m_dz, m_dagg, a));
  return HG_OK;
}

}  // namespace hg

// Debug: phase timestamps (%globaltimer ns) of CTA 0 of every later
// k_umma_top launch into trace[0..72) (null = off).  [0] producer start,
// [1+i] load i issued, [32+i] load i landed, [64..71] epilogue phases.
extern "C" int hg_top_trace(int64_t* trace) {
  hg::g_top_trace = trace;
  return HG_OK;
}

extern "C" int hg_gemm_bf16(const void* A, int64_t lda, int a_mn_major, const void* B, int64_t ldb,
                            int b_mn_major, void* C, int64_t ldc, int32_t M, int32_t N, int32_t K,
                            int32_t epi, const float* bias, int32_t split, void* stream) {
  if (M <= 0 || K <= 0) return HG_OK;
  return hg::umma_gemm(A, lda, a_mn_major != 0, B, ldb, b_mn_major != 0, C, ldc, M, N, K, nullptr,
                       nullptr, epi, bias, split < 1 ? 1 : split, (cudaStream_t)stream);
}
