// Persistent training step: one launch per iteration for the two-layer
// tensor-core step (model.py:213-329 for L = 2, bf16 operands).
//
// The split path (hg_dense.cu run_step) is ~13 dependent launches per
// iteration -- GEMMs of 24-128 CTAs, gathers, softmax, masks, scatter, SGD --
// each paying launch, CTA setup, TMEM allocation and pipeline fill, so the
// chain is latency bound (62.6 us per 1024-root papers step, ~6x the time
// its HBM traffic and tensor work need).  This kernel runs the same chain as
// phases of ONE grid of one CTA per SM, separated by grid-wide barriers, with
// the TMEM accumulator, the mbarrier ring and the tensor maps set up once:
//
//   P1  h1   = bf16(relu(agg1 @ W1 + b1))               GEMM  (tcgen05)
//   P2  agg2 = [h1[self] | mean h1[nbrs]]               gather (SIMT)
//   P3  h2   = bf16(relu(agg2 @ W2 + b2))               GEMM
//   P4  logits = h2 @ Wc                                GEMM
//   P5  loss, dlogits (f32 + bf16)                      softmax-CE (SIMT)
//   P6  dz2 = (dl @ Wcᵀ) * (h2 > 0), gb2 += colsum      GEMM, masked epilogue
//       gWc += h2ᵀ dl                                   GEMM, split-K TMA reduce-add
//   P7  dagg2 = dz2 @ W2ᵀ                               GEMM
//       gW2 += agg2ᵀ dz2                                GEMM, split-K
//   P8  dz1 = scatterᵀ(dagg2) * (h1 > 0), gb1           scatter (SIMT, k_scatter_top's map)
//   P9  gW1 += agg1ᵀ dz1                                GEMM, split-K
//   P10 SGD + gradient reset + bf16 operand refresh     SIMT (k_sgd_refresh's tiles)
//
// Arithmetic is the split kernels' (same operands, rounding points and
// accumulation order per output element); only the order of the atomic
// column sums and split-K reductions differs.
//
// GEMM phases: warp 0 lane 0 streams A/B k-blocks (TMA, 128B swizzle) through
// a ring of up to four slots, warp 1 lane 0 issues tcgen05.mma into the TMEM
// accumulator, warps 4-7 drain it (TMEM lane quadrant = warp & 3) through
// per-warp double-buffered store boxes handed to TMA (store, or f32 add-
// reduction for split-K weight gradients).  The MMA of the next tile waits
// on a TMEM-empty barrier, so a CTA's loads run ahead into its next tile
// while the epilogue drains.  SIMT phases use all eight warps.
//
// Co-residency: the grid barriers need every CTA resident.  The kernel is
// sized (128 KB dynamic shared memory, <= 88 registers) to fit on an SM
// beside the run-ahead side branch at its budget (2 build CTAs, 2 gather
// CTAs per SM); a CTA that cannot be placed yet only delays the step until
// the side kernels retire some CTAs (they never wait on this kernel).
#include <algorithm>
#include <mutex>

#include "hg_step.cuh"
#include "hg_tc.cuh"

namespace hg {

enum PEpi { PE_BIAS_RELU_BF16 = 0, PE_STORE_F32 = 1, PE_REDUCE_F32 = 2, PE_MASK_BF16 = 3 };

constexpr int kPThreads = 256;
constexpr int kPRing = 96 * 1024;
constexpr int kPBox = 4096;  // one 32-row x 128-byte store box
constexpr int kPSmem = kPRing + 4 * 2 * kPBox;
constexpr int kPMaxGemm = 8;
constexpr int kPMaxRegs = 128;

struct PGemm {
  int ma, mb, mc;           // tensor-map slots of A, B, C
  int a_mn, b_mn, bn;       // operand majors, N tile
  int M, N, K;              // C rows (capacity when M_dev), C columns, reduction length
  const int32_t* M_dev;     // device row count of C (A K-major) or null
  const int32_t* K_dev;     // device reduction length (MN-major operands) or null
  int m_tiles, n_tiles, split;
  int epi;
  const float* bias;        // PE_BIAS_RELU_BF16
  const bf16* mask;         // PE_MASK_BF16: h (bf16, row pitch N)
  float* colsum;            // PE_MASK_BF16: bias gradient
};
__host__ __device__ __forceinline__ int pg_items(const PGemm& g) {
  return g.m_tiles * g.n_tiles * g.split;
}

struct PArgs {
  CUtensorMap maps[3 * kPMaxGemm];
  PGemm g[kPMaxGemm];
  int sage, H, C, Cp, in2;
  int R, cap1, cap2;
  const int32_t* tot;       // N_0..N_2 (device)
  // P2
  const bf16* h1;
  bf16* agg2;
  const int32_t* self2;
  const int32_t* noff2;
  const int32_t* nidx2;
  // P5
  float* logits;
  const int64_t* roots;
  uint64_t label_state;
  const int32_t* labels;
  float* loss;
  bf16* dl;
  // P8
  const float* dagg;
  const int32_t* need_off1;
  const int32_t* need_off2;
  const int8_t* inl1;
  bf16* dz1;
  float* gb1;
  // P10
  int update;
  float* params;
  float* grads;
  float lr, inv_batch;
  SgdPlan plan;
  unsigned int* bar;        // [0] barrier arrivals, [1] exits
  int64_t* trace;           // debug (hg_persist_trace): per CTA [32] %globaltimer stamps, or null
};

struct PTile {
  int m0, n0, kb0, kb1;
};

__device__ __forceinline__ bool p_tile(const PGemm& G, int item, PTile& t) {
  const int mt = item % G.m_tiles;
  const int rest = item / G.m_tiles;
  const int nt = rest % G.n_tiles, z = rest / G.n_tiles;
  t.m0 = mt * BM_T;
  t.n0 = nt * G.bn;
  const int M = G.M_dev ? *G.M_dev : G.M;
  if (t.m0 >= M) return false;
  const int K = G.K_dev ? *G.K_dev : G.K;
  const int kblocks = (K + BK_T - 1) / BK_T;
  const int per = (kblocks + G.split - 1) / G.split;
  t.kb0 = z * per;
  t.kb1 = min(kblocks, t.kb0 + per);
  return t.kb0 < t.kb1;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier number `idx` (1, 2, ...): every CTA's global and TMA
// writes before it are visible to every CTA's loads and TMA reads after it.
__device__ __forceinline__ void p_stamp(int64_t* trace, int i) {
  if (trace) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    trace[blockIdx.x * 64 + i] = (int64_t)t;
  }
}

__device__ __forceinline__ void p_grid_sync(unsigned* ctr, unsigned idx, int64_t* trace) {
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    p_stamp(trace, 2 * idx);
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    const unsigned target = idx * gridDim.x;
    while (ld_acquire(ctr) < target) {
    }
    __threadfence();  // gpu-scope fence: invalidates this SM's L1 for the next phase's loads
    p_stamp(trace, 2 * idx + 1);
  }
  __syncthreads();
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ uint4 ld_u4(const void* p) {  // coherent (data written in this kernel)
  return *reinterpret_cast<const uint4*>(p);
}
__device__ __forceinline__ void bf8_to_f(const uint4 raw, float* v) {
  const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __uint_as_float(w[i] << 16);
    v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ uint4 f_to_bf8(const float* v) {
  return make_uint4(pack_bf2(v[0], v[1]), pack_bf2(v[2], v[3]), pack_bf2(v[4], v[5]),
                    pack_bf2(v[6], v[7]));
}

// Role state carried across GEMM phases (each role thread keeps its own copy).
struct PRole {
  int uses[4];     // fills (producer) / drains (MMA) of each ring slot so far
  int tiles;       // tiles accumulated (MMA) / drained (epilogue) so far
  int stores;      // TMA store boxes issued by this epilogue warp (lane 0)
};

struct PBars {
  uint64_t full[4], empty[4], acc_full, tmem_empty;
};

// One GEMM phase: the items of GEMMs g0 and (optionally) g1, dealt out
// round-robin over the CTAs.
__device__ void p_gemm_phase(const PArgs& a, int g0, int g1, uint8_t* ring, uint8_t* boxes,
                             uint32_t tmem, PBars& B, PRole& role, float* bias_s) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0items = pg_items(a.g[g0]);
  const int total = n0items + (g1 >= 0 ? pg_items(a.g[g1]) : 0);
  // uniform slot geometry for the phase: the largest stage of its GEMMs
  int stage = 16384 + a.g[g0].bn * 128;
  if (g1 >= 0) stage = max(stage, 16384 + a.g[g1].bn * 128);
  const int n_slots = min(4, kPRing / stage);
  if (warp == 0) {
    if (lane == 0) {
      int pos = 0;
      for (int it = blockIdx.x; it < total; it += gridDim.x) {
        const PGemm& G = it < n0items ? a.g[g0] : a.g[g1];
        PTile t;
        if (!p_tile(G, it < n0items ? it : it - n0items, t)) continue;
        const CUtensorMap* ma = &a.maps[G.ma];
        const CUtensorMap* mb = &a.maps[G.mb];
        const uint32_t bytes = 16384 + G.bn * 128;
        for (int kb = t.kb0; kb < t.kb1; ++kb, ++pos) {
          const int s = pos % n_slots;
          if (role.uses[s] > 0) mbar_wait(&B.empty[s], (role.uses[s] - 1) & 1);
          if (g0 == 0 && pos < 4) p_stamp(a.trace, 20 + pos);
          ++role.uses[s];
          uint8_t* sa = ring + s * stage;
          uint8_t* sb = sa + 16384;
          const int k0 = kb * BK_T;
          mbar_expect_tx(&B.full[s], bytes);
          if (G.a_mn) {
            tma_load_2d(sa, ma, &B.full[s], t.m0, k0);
            tma_load_2d(sa + 8192, ma, &B.full[s], t.m0 + 64, k0);
          } else {
            tma_load_2d(sa, ma, &B.full[s], k0, t.m0);
          }
          if (G.b_mn) {
            for (int b = 0; b < G.bn / 64; ++b) tma_load_2d(sb + b * 8192, mb, &B.full[s], t.n0 + 64 * b, k0);
          } else {
            tma_load_2d(sb, mb, &B.full[s], k0, t.n0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int pos = 0;
      for (int it = blockIdx.x; it < total; it += gridDim.x) {
        const PGemm& G = it < n0items ? a.g[g0] : a.g[g1];
        PTile t;
        if (!p_tile(G, it < n0items ? it : it - n0items, t)) continue;
        if (role.tiles > 0) mbar_wait(&B.tmem_empty, (role.tiles - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t idesc = make_idesc(G.bn, G.a_mn != 0, G.b_mn != 0);
        for (int kb = t.kb0; kb < t.kb1; ++kb, ++pos) {
          const int s = pos % n_slots;
          mbar_wait(&B.full[s], role.uses[s] & 1);
          if (g0 == 0 && pos < 4) p_stamp(a.trace, 24 + pos);
          ++role.uses[s];
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t sa = smem_u32(ring + s * stage);
          const uint32_t sb = sa + 16384;
#pragma unroll
          for (int kk = 0; kk < BK_T / 16; ++kk) {
            const uint64_t ad = G.a_mn ? make_desc(sa + kk * 2048, 64 * 128, 1024)
                                       : make_desc(sa + kk * 32, 16, 1024);
            const uint64_t bd = G.b_mn ? make_desc(sb + kk * 2048, 64 * 128, 1024)
                                       : make_desc(sb + kk * 32, 16, 1024);
            umma_bf16(tmem, ad, bd, idesc, (kb > t.kb0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&B.empty[s]);
        }
        umma_commit(&B.acc_full);
        ++role.tiles;
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    uint8_t* mybox = boxes + q * 2 * kPBox;
    const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16);
    for (int it = blockIdx.x; it < total; it += gridDim.x) {
      const PGemm& G = it < n0items ? a.g[g0] : a.g[g1];
      PTile t;
      if (!p_tile(G, it < n0items ? it : it - n0items, t)) continue;
      mbar_wait(&B.acc_full, role.tiles & 1);
      if (g0 == 0 && warp == 4 && lane == 0) p_stamp(a.trace, 28);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int M = G.M_dev ? *G.M_dev : G.M;
      const int row = t.m0 + q * 32 + lane;
      const bool valid = row < M;
      const CUtensorMap* mc = &a.maps[G.mc];
      const bool bf = G.epi == PE_BIAS_RELU_BF16 || G.epi == PE_MASK_BF16;
      if (G.epi == PE_BIAS_RELU_BF16) {  // this tile's bias columns into smem (epilogue warps)
        asm volatile("bar.sync 1, 128;" ::: "memory");
        for (int cix = (warp - 4) * 32 + lane; cix < G.bn; cix += 128)
          bias_s[cix] = t.n0 + cix < G.N ? G.bias[t.n0 + cix] : 0.f;
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      const int cw = bf ? 64 : 32;  // columns per 128-byte box row
      for (int c = 0; c < G.bn; c += cw) {
        if (t.n0 + c >= G.N) break;
        uint8_t* box = mybox + (role.stores & 1) * kPBox;
        if (role.stores >= 2 && lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
        if (g0 == 0 && warp == 4 && lane == 0 && role.stores < 4) p_stamp(a.trace, 35 + 4 * role.stores);
        uint8_t* myrow = box + lane * 128;
        if (bf) {
          // two 32-column halves per 64-column box (16 TMEM registers x 2 in flight)
#pragma unroll 1
          for (int hf = 0; hf < 2; ++hf) {
            const int cc = c + hf * 32;
            uint32_t r[32];
            tmem_ld16_issue(tq + cc, r);
            tmem_ld16_issue(tq + cc + 16, r + 16);
            uint4 hraw[4];
            if (G.epi == PE_MASK_BF16) {  // h's 32 columns of this row, loads in flight with TMEM's
              const bf16* hp = G.mask + (int64_t)(valid ? row : 0) * G.N + t.n0 + cc;
#pragma unroll
              for (int u = 0; u < 4; ++u) hraw[u] = ld_u4(hp + u * 8);
            }
            tmem_wait16(r);
            tmem_wait16(r + 16);
            if (g0 == 0 && warp == 4 && lane == 0 && role.stores < 4) p_stamp(a.trace, 32 + 4 * role.stores + hf);
            if (G.epi == PE_BIAS_RELU_BF16) {
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                float v[8];
#pragma unroll
                for (int e = 0; e < 8; ++e)
                  v[e] = valid ? fmaxf(__uint_as_float(r[u * 8 + e]) + bias_s[cc + u * 8 + e], 0.f) : 0.f;
                const int uu = hf * 4 + u;
                *reinterpret_cast<uint4*>(myrow + ((uu ^ (lane & 7)) << 4)) = f_to_bf8(v);
              }
            } else {  // PE_MASK_BF16: dz = acc * (h > 0); column sums into the bias gradient
#pragma unroll
              for (int g16 = 0; g16 < 2; ++g16) {
                float v[16];
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                  float hv[8];
                  bf8_to_f(hraw[g16 * 2 + h2], hv);
#pragma unroll
                  for (int e = 0; e < 8; ++e)
                    v[h2 * 8 + e] = valid && hv[e] > 0.f ? __uint_as_float(r[g16 * 16 + h2 * 8 + e]) : 0.f;
                  const int uu = hf * 4 + g16 * 2 + h2;
                  *reinterpret_cast<uint4*>(myrow + ((uu ^ (lane & 7)) << 4)) = f_to_bf8(v + h2 * 8);
                }
                const float cs = colsum16(v, lane);
                const int col = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 +
                                ((lane >> 1) & 1);
                if ((lane & 1) == 0) atomicAdd(G.colsum + t.n0 + cc + g16 * 16 + col, cs);
              }
            }
          }
        } else {
          uint32_t r[32];
          tmem_ld16_issue(tq + c, r);
          tmem_ld16_issue(tq + c + 16, r + 16);
          tmem_wait16(r);
          tmem_wait16(r + 16);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const uint4 v = valid ? make_uint4(r[u * 4], r[u * 4 + 1], r[u * 4 + 2], r[u * 4 + 3])
                                  : make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4*>(myrow + ((u ^ (lane & 7)) << 4)) = v;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          if (G.epi == PE_REDUCE_F32) tma_store_2d<true>(mc, box, t.n0 + c, t.m0 + q * 32);
          else tma_store_2d<false>(mc, box, t.n0 + c, t.m0 + q * 32);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          if (g0 == 0 && warp == 4 && role.stores < 4) p_stamp(a.trace, 34 + 4 * role.stores);
        }
        ++role.stores;
      }
      // TMEM drained: the MMA of this CTA's next tile may overwrite it
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&B.tmem_empty);
      ++role.tiles;
    }
    // every store of the phase complete before the grid barrier
    if (g0 == 0 && warp == 4 && lane == 0) p_stamp(a.trace, 29);
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (g0 == 0 && warp == 4 && lane == 0) p_stamp(a.trace, 48);
    __syncwarp();
  }
}

// P2: layer-2 gather + aggregate (k_aggregate's arithmetic), warp per row;
// rows [N2, roundup64(N2)) zeroed for the weight-gradient reduction.
__device__ void p_gather2(const PArgs& a) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (kPThreads / 32) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (kPThreads / 32);
  const int H = a.H, in2 = a.in2;
  const int n2 = a.tot[2];
  const int pad = min(a.cap2, (n2 + 63) / 64 * 64);
  const int c0 = lane * 8;
  const bool on = c0 < H;
  for (int r = gw; r < pad; r += nw) {
    bf16* o = a.agg2 + (int64_t)r * in2;
    if (r >= n2) {
      for (int c = lane * 8; c < in2; c += 256) *reinterpret_cast<uint4*>(o + c) = make_uint4(0, 0, 0, 0);
      continue;
    }
    const int s = a.self2[r];
    const int j0 = a.noff2[r], deg = a.noff2[r + 1] - j0;
    float self[8], acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    if (on) bf8_to_f(ld_u4(a.h1 + (int64_t)s * H + c0), self);
    for (int t0 = 0; t0 < deg; t0 += 8) {
      uint4 x[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        x[t] = make_uint4(0, 0, 0, 0);
        if (on && t0 + t < deg) x[t] = ld_u4(a.h1 + (int64_t)a.nidx2[j0 + t0 + t] * H + c0);
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        float v[8];
        bf8_to_f(x[t], v);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += v[e];
      }
    }
    if (!on) continue;
    if (a.sage) {
      float nb[8];
      const float inv = deg > 0 ? 1.0f / (float)deg : 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) nb[e] = deg > 0 ? acc[e] * inv : self[e];
      *reinterpret_cast<uint4*>(o + c0) = f_to_bf8(self);
      *reinterpret_cast<uint4*>(o + H + c0) = f_to_bf8(nb);
    } else {
      const float inv = 1.0f / (float)(deg + 1);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = (acc[e] + self[e]) * inv;
      *reinterpret_cast<uint4*>(o + c0) = f_to_bf8(acc);
    }
  }
}

// P5: softmax-CE of the root rows (k_softmax_ce), warp per root.
__device__ void p_softmax(const PArgs& a) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (kPThreads / 32) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (kPThreads / 32);
  const int C = a.C, Cp = a.Cp;
  const int n = a.tot[2];
  for (int r = gw; r < a.R; r += nw) {
    float* x = a.logits + (int64_t)r * C;
    bf16* dlr = a.dl + (int64_t)r * Cp;
    if (r >= n) {
      for (int c = lane; c < C; c += 32) x[c] = 0.f;
      for (int c = lane; c < Cp; c += 32) dlr[c] = __float2bfloat16_rn(0.f);
      if (lane == 0) a.loss[r] = 0.f;
      continue;
    }
    float mx = -INFINITY;
    for (int c = lane; c < C; c += 32) mx = fmaxf(mx, x[c]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float s = 0.f;
    for (int c = lane; c < C; c += 32) s += expf(x[c] - mx);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const int label = a.labels ? a.labels[r] : (int)(mix64(a.label_state ^ (uint64_t)a.roots[r]) % (uint64_t)C);
    const float xl = x[label];
    __syncwarp();
    const float inv = 1.0f / s;
    for (int c = lane; c < C; c += 32) {
      const float g = expf(x[c] - mx) * inv - (c == label ? 1.f : 0.f);
      x[c] = g;
      dlr[c] = __float2bfloat16_rn(g);
    }
    for (int c = C + lane; c < Cp; c += 32) dlr[c] = __float2bfloat16_rn(0.f);
    if (lane == 0) a.loss[r] = logf(s) - (xl - mx);
  }
}

// P8: top-layer backward map (k_scatter_top's arithmetic) -> dz1 bf16, gb1.
__device__ void p_scatter_top(const PArgs& a, float* red /* [8][257] smem */) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = a.H, ld = a.in2;
  const int c0 = lane * 8;
  const bool lane_on = c0 < H;
  float cs[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) cs[j] = 0.f;
  const int n_rows = a.tot[1];
  for (int r = blockIdx.x * 8 + warp; r < a.R; r += gridDim.x * 8) {
    const int q0 = a.need_off1[r], nq = a.need_off1[r + 1] - q0;
    const int rowL = a.need_off2[r];
    if (!lane_on || nq == 0 || a.need_off2[r + 1] - rowL != 1) continue;
    const int srow = a.self2[rowL];
    const int deg = a.noff2[rowL + 1] - a.noff2[rowL];
    const float* g = a.dagg + (int64_t)rowL * ld;
    float gs[8], gn[8];
#pragma unroll
    for (int j = 0; j < 8; j += 4) {
      const float4 x = *reinterpret_cast<const float4*>(g + c0 + j);
      gs[j] = x.x; gs[j + 1] = x.y; gs[j + 2] = x.z; gs[j + 3] = x.w;
      if (a.sage) {
        const float4 y = *reinterpret_cast<const float4*>(g + H + c0 + j);
        gn[j] = y.x; gn[j + 1] = y.y; gn[j + 2] = y.z; gn[j + 3] = y.w;
      } else {
        gn[j] = gn[j + 1] = gn[j + 2] = gn[j + 3] = 0.f;
      }
    }
    for (int i0 = 0; i0 < nq; i0 += 4) {
      uint4 hr[4];
      int8_t inl[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int u = q0 + min(i0 + t, nq - 1);
        hr[t] = ld_u4(a.h1 + (int64_t)u * H + c0);
        inl[t] = a.inl1[u];
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (i0 + t >= nq) break;
        const int u = q0 + i0 + t;
        const bool self = u == srow, nbr = inl[t] != 0;
        float hv[8], v[8];
        bf8_to_f(hr[t], hv);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float x;
          if (a.sage)
            x = (self ? (deg > 0 ? gs[j] : gs[j] + gn[j]) : 0.f) + (nbr ? gn[j] / (float)deg : 0.f);
          else
            x = gs[j] * ((float)((int)self + (int)nbr) / (float)(deg + 1));
          v[j] = hv[j] > 0.f ? x : 0.f;
          cs[j] += v[j];
        }
        *reinterpret_cast<uint4*>(a.dz1 + (int64_t)u * H + c0) = f_to_bf8(v);
      }
    }
  }
  if (lane_on)
#pragma unroll
    for (int j = 0; j < 8; ++j) red[warp * 257 + c0 + j] = cs[j];
  __syncthreads();
  for (int c = threadIdx.x; c < H; c += blockDim.x) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w * 257 + c];
    atomicAdd(a.gb1 + c, t);
  }
  if (blockIdx.x == 0) {  // the dW1 reduction reads up to the next multiple of 64 rows
    const int pad = min(a.cap1, (n_rows + 63) / 64 * 64);
    for (int64_t i = (int64_t)n_rows * H + threadIdx.x; i < (int64_t)pad * H; i += blockDim.x)
      a.dz1[i] = __float2bfloat16_rn(0.f);
  }
}

// P10: SGD + gradient reset + bf16 operand copies (k_sgd_refresh's tiles).
__device__ void p_sgd(const PArgs& a, bf16* tile /* [32][34] smem */) {
  const SgdPlan& P = a.plan;
  float* __restrict__ p = a.params;
  float* __restrict__ g = a.grads;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
    int mi = 0;
    while (mi + 1 < P.n_mats && P.m[mi + 1].tile0 <= t) ++mi;
    const SgdMat& M = P.m[mi];
    const int lt = t - M.tile0, tr = lt / M.tiles_c, tc = lt % M.tiles_c;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = tr * 32 + ty + 8 * j, c = tc * 32 + tx;
      if (r < M.rows && c < M.cols) {
        const int64_t i = M.off + (int64_t)r * M.cols + c;
        float v = p[i];
        v -= a.lr * (g[i] * a.inv_batch);
        p[i] = v;
        g[i] = 0.f;
        const bf16 b = __float2bfloat16_rn(v);
        if (M.sdst) M.sdst[(int64_t)r * M.sld + c] = b;
        tile[(ty + 8 * j) * 34 + tx] = b;
      }
    }
    __syncthreads();
    if (M.tdst) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = tc * 32 + ty + 8 * j, r = tr * 32 + tx;
        if (r < M.rows && c < M.cols) M.tdst[(int64_t)c * M.tld + r] = tile[tx * 34 + ty + 8 * j];
      }
    }
    __syncthreads();
  }
  for (int64_t i = P.plain_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.plain_hi;
       i += (int64_t)gridDim.x * blockDim.x) {
    p[i] -= a.lr * (g[i] * a.inv_batch);
    g[i] = 0.f;
  }
}

__global__ void __maxnreg__(kPMaxRegs)
k_step_persist(const __grid_constant__ PArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = smem;
  uint8_t* boxes = smem + kPRing;
  __shared__ __align__(8) PBars B;
  __shared__ uint32_t tmem_base_sh;
  __shared__ float bias_s[256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) p_stamp(a.trace, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) {
      mbar_init(&B.full[s], 1);
      mbar_init(&B.empty[s], 1);
    }
    mbar_init(&B.acc_full, 1);
    mbar_init(&B.tmem_empty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane < 3 * kPMaxGemm)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.maps[lane])) : "memory");
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;
  PRole role{{0, 0, 0, 0}, 0, 0};
  unsigned bi = 0;
  if (threadIdx.x == 0) p_stamp(a.trace, 1);
  p_gemm_phase(a, 0, -1, ring, boxes, tmem, B, role, bias_s);     // P1  h1
  p_grid_sync(a.bar, ++bi, a.trace);
  p_gather2(a);                                           // P2  agg2
  p_grid_sync(a.bar, ++bi, a.trace);
  p_gemm_phase(a, 1, -1, ring, boxes, tmem, B, role, bias_s);     // P3  h2
  p_grid_sync(a.bar, ++bi, a.trace);
  p_gemm_phase(a, 2, -1, ring, boxes, tmem, B, role, bias_s);     // P4  logits
  p_grid_sync(a.bar, ++bi, a.trace);
  p_softmax(a);                                           // P5  loss, dlogits
  p_grid_sync(a.bar, ++bi, a.trace);
  p_gemm_phase(a, 3, 4, ring, boxes, tmem, B, role, bias_s);      // P6  dz2 + gb2 | gWc
  p_grid_sync(a.bar, ++bi, a.trace);
  p_gemm_phase(a, 5, 6, ring, boxes, tmem, B, role, bias_s);      // P7  dagg2 | gW2
  p_grid_sync(a.bar, ++bi, a.trace);
  p_scatter_top(a, reinterpret_cast<float*>(ring));       // P8  dz1, gb1
  p_grid_sync(a.bar, ++bi, a.trace);
  p_gemm_phase(a, 7, -1, ring, boxes, tmem, B, role, bias_s);     // P9  gW1
  if (a.update) {
    p_grid_sync(a.bar, ++bi, a.trace);
    p_sgd(a, reinterpret_cast<bf16*>(ring));              // P10 SGD + refresh
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  if (threadIdx.x == 0) {
    p_stamp(a.trace, 30);
    // the last CTA out resets the barrier counters for the next launch (every
    // CTA has passed every barrier once it increments the exit count)
    if (atomicAdd(a.bar + 1, 1u) == gridDim.x - 1) {
      atomicExch(a.bar, 0u);
      atomicExch(a.bar + 1, 0u);
    }
  }
}

// ------------------------------------------------------------------ host side

static int g_persist = 0;        // hg_set_persist
static int g_persist_ctas = 0;   // 0: one per SM
static int g_split_w1 = 0;       // 0: heuristic
static int64_t* g_ptrace = nullptr;

// Barrier counters of the current device, allocated by hg_set_persist (outside
// any graph capture) -- a launch only reads the pointer.
static unsigned* g_bar[64] = {};
static std::mutex g_bar_mu;

static unsigned* persist_bar(bool create) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_bar_mu);
  unsigned*& b = g_bar[dev & 63];
  if (!b && create) {
    if (cudaMalloc(&b, 2 * sizeof(unsigned)) != cudaSuccess) { b = nullptr; return nullptr; }
    if (cudaMemset(b, 0, 2 * sizeof(unsigned)) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
      return nullptr;
  }
  return b;
}

static int n_sms() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}

bool persist_eligible(const hg_step_desc* d, int n_roots) {
  if (!g_persist) return false;
  const int H = d->hidden, C = d->n_classes;
  const int Cp = (C + 63) / 64 * 64;
  return d->act_dtype == 1 && d->use_tc && d->n_layers == 2 && H % 64 == 0 && H >= 64 &&
         H <= 256 && d->in_dim[1] % 64 == 0 && d->in_dim[1] <= 1024 &&
         d->in_dim[2] == (d->arch == 1 ? 2 * H : H) && C >= 1 && C % 4 == 0 && Cp <= 256 &&
         d->WcT && d->Wcp &&
         d->dl_lowp && d->Wb[2] && d->Wlp[1] && d->Wlp[2] && d->lowp_scratch && d->dagg &&
         d->agg1_ready && d->lowp_fresh && n_roots <= d->max_rows[2] && n_roots == d->max_roots;
}

static bf16* dz_region(const hg_step_desc* d, int k) {
  int64_t rows = 0;
  if (d->lowp_layered)
    for (int j = 1; j < k; ++j) rows += d->max_rows[j];
  return (bf16*)d->lowp_scratch + rows * d->hidden;
}

// A GEMM of the step: operand maps (boxes per major), C map (store box), grid.
static int add_gemm(PArgs& a, int gi, const void* A, int64_t lda, bool a_mn, const void* Bp,
                    int64_t ldb, bool b_mn, void* Cm, int64_t ldc, int M, int N, int K,
                    const int32_t* M_dev, const int32_t* K_dev, int bn, int split, int epi) {
  PGemm& g = a.g[gi];
  g = PGemm{};
  g.ma = 3 * gi; g.mb = 3 * gi + 1; g.mc = 3 * gi + 2;
  g.a_mn = a_mn; g.b_mn = b_mn; g.bn = bn;
  g.M = M; g.N = N; g.K = K; g.M_dev = M_dev; g.K_dev = K_dev;
  g.m_tiles = (M + BM_T - 1) / BM_T;
  g.n_tiles = (N + bn - 1) / bn;
  g.split = std::max(1, split);
  g.epi = epi;
  int st;
  if (a_mn) st = make_map(&a.maps[g.ma], A, (uint64_t)M, (uint64_t)K, lda, 64, BK_T);
  else st = make_map(&a.maps[g.ma], A, (uint64_t)K, (uint64_t)M, lda, BK_T, BM_T);
  if (st) return st;
  if (b_mn) st = make_map(&a.maps[g.mb], Bp, (uint64_t)N, (uint64_t)K, ldb, 64, BK_T);
  else st = make_map(&a.maps[g.mb], Bp, (uint64_t)K, (uint64_t)N, ldb, BK_T, (uint32_t)bn);
  if (st) return st;
  const bool bf = epi == PE_BIAS_RELU_BF16 || epi == PE_MASK_BF16;
  if ((uintptr_t)Cm % 16 || (ldc * (bf ? 2 : 4)) % 16)
    return hg_fail(HG_ECONFIG, "persistent step: output %d rows not 16-byte aligned", gi);
  return make_map(&a.maps[g.mc], Cm, (uint64_t)N, (uint64_t)M, ldc, bf ? 64 : 32, 32, bf ? 2 : 4);
}

int persist_step(const hg_step_desc* d, int n_roots, float* params, float* grads, int64_t n,
                 float lr, float inv_batch, int update, cudaStream_t s) {
  const int H = d->hidden, C = d->n_classes, Cp = (C + 63) / 64 * 64;
  const int in1 = d->in_dim[1], in2 = d->in_dim[2];
  const int cap1 = d->max_rows[1], cap2 = d->max_rows[2], R = n_roots;
  const int32_t* tot = d->mg.totals;
  unsigned* bar = persist_bar(false);
  if (!bar) return hg_fail(HG_ECONFIG, "persistent step: hg_set_persist was not called on this device");
  const int P = g_persist_ctas > 0 ? std::min(g_persist_ctas, n_sms()) : n_sms();
  static PArgs a;  // ~5 KB; built per call (graph capture copies the parameters)
  memset(&a, 0, sizeof(a));
  bf16* dz2 = dz_region(d, 2);
  bf16* dz1 = dz_region(d, 1);
  int st;
  const int r_tiles = (R + BM_T - 1) / BM_T;
  // P1  h1 = relu(agg1 @ W1 + b1): W1ᵀ (Wlp[1]) is the K-major B
  if ((st = add_gemm(a, 0, d->agg[1], in1, false, d->Wlp[1], in1, false, d->h[1], H, cap1, H, in1,
                     tot + 1, nullptr, H, 1, PE_BIAS_RELU_BF16))) return st;
  a.g[0].bias = d->b[1];
  // P3  h2 = relu(agg2 @ W2 + b2): N tiles of 64 spread the 8 root tiles
  if ((st = add_gemm(a, 1, d->agg[2], in2, false, d->Wlp[2], in2, false, d->h[2], H, cap2, H, in2,
                     tot + 2, nullptr, 64, 1, PE_BIAS_RELU_BF16))) return st;
  a.g[1].bias = d->b[2];
  // P4  logits = h2 @ Wc (WcT K-major)
  if ((st = add_gemm(a, 2, d->h[2], H, false, d->WcT, H, false, d->logits, C, R, C, H, tot + 2,
                     nullptr, 64, 1, PE_STORE_F32))) return st;
  // P6a dz2 = (dl @ Wcᵀ) * (h2 > 0), gb2 (Wcp = W_c padded, K-major B)
  if ((st = add_gemm(a, 3, d->dl_lowp, Cp, false, d->Wcp, Cp, false, dz2, H, R, H, Cp, tot + 2,
                     nullptr, 64, 1, PE_MASK_BF16))) return st;
  a.g[3].mask = (const bf16*)d->h[2];
  a.g[3].colsum = d->gb[2];
  // P6b gWc += h2ᵀ dl (MN-major both; reduction over the roots)
  const int bnc = std::min(256, (C + 63) / 64 * 64);
  if ((st = add_gemm(a, 4, d->h[2], H, true, d->dl_lowp, Cp, true, d->gWc, C, H, C, R, nullptr,
                     tot + 2, bnc, std::max(1, std::min(8, r_tiles)), PE_REDUCE_F32))) return st;
  // P7a dagg2 = dz2 @ W2ᵀ (Wb[2] = W2 straight, K-major B)
  if ((st = add_gemm(a, 5, dz2, H, false, d->Wb[2], H, false, d->dagg, in2, R, in2, H, tot + 2,
                     nullptr, 64, 1, PE_STORE_F32))) return st;
  // P7b gW2 += agg2ᵀ dz2
  if ((st = add_gemm(a, 6, d->agg[2], in2, true, dz2, H, true, d->gW[2], H, in2, H, cap2, nullptr,
                     tot + 2, H, std::max(1, std::min(8, (cap2 + 127) / 128)), PE_REDUCE_F32))) return st;
  // P9  gW1 += agg1ᵀ dz1: split-K over the layer-1 rows, about one item per CTA
  const int mt1 = (in1 + BM_T - 1) / BM_T;
  const int split1 = g_split_w1 > 0 ? g_split_w1 : std::max(1, P / mt1);
  if ((st = add_gemm(a, 7, d->agg[1], in1, true, dz1, H, true, d->gW[1], H, in1, H, cap1, nullptr,
                     tot + 1, H, split1, PE_REDUCE_F32))) return st;
  a.sage = d->arch == 1;
  a.H = H; a.C = C; a.Cp = Cp; a.in2 = in2;
  a.R = R; a.cap1 = cap1; a.cap2 = cap2; a.tot = tot;
  a.h1 = (const bf16*)d->h[1];
  a.agg2 = (bf16*)d->agg[2];
  a.self2 = d->mg.self_pos[2];
  a.noff2 = d->mg.nbr_off[2];
  a.nidx2 = d->mg.nbr_idx[2];
  a.logits = d->logits;
  a.roots = d->roots;
  a.label_state = d->label_state;
  a.labels = d->labels;
  a.loss = d->loss;
  a.dl = (bf16*)d->dl_lowp;
  a.dagg = d->dagg;
  a.need_off1 = d->mg.need_off[1];
  a.need_off2 = d->mg.need_off[2];
  a.inl1 = d->mg.in_layer[1];
  a.dz1 = dz1;
  a.gb1 = d->gb[1];
  a.update = update;
  a.bar = bar;
  a.trace = g_ptrace;
  if (update) {
    a.params = params;
    a.grads = grads;
    a.lr = lr;
    a.inv_batch = inv_batch;
    if ((st = make_sgd_plan(d, params, n, &a.plan))) return st;
  }
  static bool attr = false;
  if (!attr) {
    HG_CUDA_TRY(cudaFuncSetAttribute(k_step_persist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kPSmem + 1024));
    attr = true;
  }
  count_launch();
  prof_begin(PROF_STEP, s);
  k_step_persist<<<P, kPThreads, kPSmem + 1024, s>>>(a);
  prof_end(PROF_STEP, s);
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}

}  // namespace hg

using namespace hg;

// Debug: %globaltimer stamps of every CTA of later persistent steps into
// trace[cta * 64 + i] (null = off): [0] entry, [1] after setup, [2i] / [2i+1]
// arrival at / release from grid barrier i, [30] exit.
extern "C" int hg_persist_trace(int64_t* trace) {
  g_ptrace = trace;
  return HG_OK;
}

extern "C" int hg_set_persist(int32_t on, int32_t ctas, int32_t split_w1) {
  if (ctas < 0 || split_w1 < 0) return hg_fail(HG_ECONFIG, "hg_set_persist: negative size");
  if (on && !persist_bar(true)) return hg_fail(HG_ECUDA, "persistent step: barrier allocation failed");
  g_persist = on != 0;
  g_persist_ctas = ctas;
  g_split_w1 = split_w1;
  return HG_OK;
}

extern "C" int hg_train_step(const hg_step_desc* d, int32_t n_roots, void* stream);
extern "C" int hg_sgd_refresh(const hg_step_desc* d, float* params, float* grads, int64_t n,
                              float lr, float inv_batch, int32_t update, void* stream);

extern "C" int hg_train_step_sgd(const hg_step_desc* d, int32_t n_roots, float* params,
                                 float* grads, int64_t n, float lr, float inv_batch,
                                 int32_t update, void* stream) {
  if (persist_eligible(d, n_roots))
    return persist_step(d, n_roots, params, grads, n, lr, inv_batch, update, (cudaStream_t)stream);
  int st = hg_train_step(d, n_roots, stream);
  if (st || !update) return st;
  return hg_sgd_refresh(d, params, grads, n, lr, inv_batch, 1, stream);
}
