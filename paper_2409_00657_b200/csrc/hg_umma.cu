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

#include "hg_common.cuh"

namespace hg {

// Pipeline depth: 4 stages, 3 for 256-wide tiles (144 KB instead of 192 KB of
// shared memory, so a GEMM CTA fits on an SM beside the build CTAs that run
// concurrently in the graph loop; the K ranges here are 4-8 blocks, and the
// 128 KB f32 epilogue staging still fits).
#ifndef HG_UMMA_STAGES_256
#define HG_UMMA_STAGES_256 3
#endif
__host__ __device__ constexpr int stages_for(int bn) { return bn >= 256 ? HG_UMMA_STAGES_256 : 4; }
constexpr int BM_T = 128;
constexpr int BK_T = 64;  // one 128-byte swizzle row of bf16

enum UEpi { UEPI_STORE_F32 = 0, UEPI_BIAS_RELU_BF16 = 1, UEPI_ATOMIC_F32 = 2, UEPI_SOFTMAX_CE = 3 };

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// smem box -> global (plain store or f32 add-reduction in L2), bulk-group completion
template <bool REDUCE>
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* smem_src, int c0,
                                             int c1) {
  if constexpr (REDUCE)
    asm volatile(
        "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];"
        ::"l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
        : "memory");
  else
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
                 : "memory");
}

// UMMA shared-memory descriptor, 128B swizzle (sm_100 version 1).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, M = 128
__host__ __device__ constexpr uint32_t make_idesc(int n, bool a_mn, bool b_mn) {
  return (1u << 4)                       // D format f32
         | (1u << 7)                     // A bf16
         | (1u << 10)                    // B bf16
         | ((a_mn ? 1u : 0u) << 15)      // A major
         | ((b_mn ? 1u : 0u) << 16)      // B major
         | ((uint32_t)(n >> 3) << 17)    // N >> 3
         | ((uint32_t)(128 >> 4) << 24); // M >> 4
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Issue a 16-column TMEM load without waiting; tmem_wait16 completes it and
// ties the registers to the wait so no use is scheduled before it.
__device__ __forceinline__ void tmem_ld16_issue(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
      " [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait16(uint32_t* r) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]),
                 "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]),
                 "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
      " [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

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
};

// Rows [r0, r1) of the head outputs past the device root count: no loss, no gradient.
__device__ __forceinline__ void head_zero_row(const UmmaArgs& a, int row) {
  float* x = reinterpret_cast<float*>(a.C) + (int64_t)row * a.ldc;
  for (int c = 0; c < a.N; ++c) x[c] = 0.f;
  for (int c = 0; c < a.ldp; ++c) a.dl_lowp[(int64_t)row * a.ldp + c] = __float2bfloat16_rn(0.f);
  a.loss[row] = 0.f;
}

template <bool A_MN, bool B_MN, int BN_T, int EPI>
__global__ void __launch_bounds__(128, 1)
k_umma_gemm(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
            const __grid_constant__ CUtensorMap map_c, UmmaArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-aligned stage ring
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~(uintptr_t)1023);
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
  const int M = args.M_dev ? *args.M_dev : args.M;
  const int K = args.K_dev ? *args.K_dev : args.K;
  // K range of this split, in 64-wide blocks
  const int kblocks = (K + BK_T - 1) / BK_T;
  const int per = (kblocks + gridDim.z - 1) / gridDim.z;
  const int kb0 = blockIdx.z * per;
  const int kb1 = min(kblocks, kb0 + per);
  if (m0 >= M || kb0 >= kb1) {  // whole CTA exits together (before any TMEM is held)
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
  // ---------------- epilogue: all 4 warps, TMEM lane quadrant = warp
  __syncwarp();
  mbar_wait(&done_bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = m0 + warp * 32 + lane;
#ifdef HG_UMMA_NOEPI  // timing experiment: main loop only
  const bool valid = false;
  if (false) {
#else
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
#endif
    // Coalesced epilogue: each warp stages its 32 rows x (128-byte column
    // chunk) in the now idle pipeline smem, 128B-swizzled, and one lane hands
    // the box to TMA (store, or f32 add-reduce in L2 for split-K partials).
    // Rows past the device count are written as zeros (inside the capacity).
    constexpr int EB = EPI == UEPI_BIAS_RELU_BF16 ? 2 : 4;
    constexpr int CW = 128 / EB;             // columns per 128-byte row
    constexpr int NCH = (BN_T + CW - 1) / CW;
    uint8_t* stage = smem + warp * (NCH * 4096);
    const bool warp_rows = m0 + warp * 32 < M;
#pragma unroll 1
    for (int ch = 0; ch < NCH; ++ch) {
      const int c = ch * CW;
      if (n0 + c >= args.N || !warp_rows) break;
      uint32_t rr[CW];
#pragma unroll
      for (int q = 0; q < CW; q += 16)
        tmem_ld16_issue(tmem + ((uint32_t)(warp * 32) << 16) + c + q, rr + q);
#pragma unroll
      for (int q = 0; q < CW; q += 16) tmem_wait16(rr + q);
      uint8_t* box = stage + ch * 4096 + lane * 128;
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
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        tma_store_2d<EPI == UEPI_ATOMIC_F32>(&map_c, stage + ch * 4096, n0 + c, m0 + warp * 32);
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
static int make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t pitch,
                    uint32_t box_inner, uint32_t box_outer, int elem_bytes = 2) {
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
  HG_CUDA_TRY(launch_pdl(kern, grid, dim3(128), smem, s, ma, mb, mc, a));
  return HG_OK;
}

// Generic entry: shapes are capacities (M/K) when *_dev counts are given.
int umma_gemm(const void* A, int64_t lda, bool a_mn, const void* B, int64_t ldb, bool b_mn,
              void* C, int64_t ldc, int M, int N, int K, const int32_t* M_dev,
              const int32_t* K_dev, int epi, const float* bias, int split, cudaStream_t s) {
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
  const int eb = epi == UEPI_BIAS_RELU_BF16 ? 2 : 4;
  int tma_epi = ((uintptr_t)C % 16 == 0 && (ldc * eb) % 16 == 0) ? 1 : 0;
  if (tma_epi && make_map(&mc, C, (uint64_t)N, (uint64_t)M, ldc, 128 / eb, 32, eb) != HG_OK) {
    tma_epi = 0;
  }
  if (!tma_epi) memset(&mc, 0, sizeof(mc));
  UmmaArgs a{M, N, K, M_dev, K_dev, C, ldc, bias, tma_epi};

#define HG_UMMA_CASE(AM, BMJ, BNV, E)                                                       \
  if (a_mn == AM && b_mn == BMJ && bn == BNV && epi == E)                                   \
    return launch_t<AM, BMJ, BNV, E>(ma, mb, mc, a, split, s);
#define HG_UMMA_N(AM, BMJ, E) \
  HG_UMMA_CASE(AM, BMJ, 64, E) HG_UMMA_CASE(AM, BMJ, 128, E) HG_UMMA_CASE(AM, BMJ, 192, E) HG_UMMA_CASE(AM, BMJ, 256, E)
  HG_UMMA_N(false, false, UEPI_BIAS_RELU_BF16)
  HG_UMMA_N(false, false, UEPI_STORE_F32)
  HG_UMMA_N(true, true, UEPI_ATOMIC_F32)
  HG_UMMA_N(true, true, UEPI_STORE_F32)
#undef HG_UMMA_N
#undef HG_UMMA_CASE
  return hg_fail(HG_ECONFIG, "unsupported umma variant (a_mn=%d b_mn=%d N=%d epi=%d)", (int)a_mn,
                 (int)b_mn, N, epi);
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

}  // namespace hg

extern "C" int hg_gemm_bf16(const void* A, int64_t lda, int a_mn_major, const void* B, int64_t ldb,
                            int b_mn_major, void* C, int64_t ldc, int32_t M, int32_t N, int32_t K,
                            int32_t epi, const float* bias, int32_t split, void* stream) {
  if (M <= 0 || K <= 0) return HG_OK;
  return hg::umma_gemm(A, lda, a_mn_major != 0, B, ldb, b_mn_major != 0, C, ldc, M, N, K, nullptr,
                       nullptr, epi, bias, split < 1 ? 1 : split, (cudaStream_t)stream);
}
