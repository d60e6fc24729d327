/*
 * libhopgnn — C ABI of the B200 (sm_100a) HopGNN micrograph training step.
 *
 * Drop-in boundary: the reference's operator layer is the `gnnsim.kernels`
 * module (reference pkg/src/gnnsim/kernels.py:31-34), which its callers bind
 * per call from Python.  The first block below replaces those entry points
 * one for one (same argument meaning; device pointers instead of numpy
 * arrays).  The rest is the batched hot path the reference runs as per-root
 * Python loops (sampler.py:84-106, model.py:183-329, engine.py:413-448).
 *
 * Conventions:
 *   - every function returns hg_status (0 = ok); hg_last_error() describes
 *     the last failure of the calling thread;
 *   - all array arguments are caller-owned DEVICE pointers unless the name
 *     ends in _host; nothing is allocated inside except where a *_ws
 *     workspace size query says so;
 *   - every function takes a cudaStream_t (as void*) and is asynchronous;
 *     kernels that detect a data-dependent error (root out of range,
 *     capacity overflow) set *err_flag (device int) instead of trapping;
 *   - no C++ exception crosses the ABI; no torch types in signatures.
 */
#ifndef HOPGNN_H_
#define HOPGNN_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HG_OK = 0,
  HG_ERANGE = 1,      /* maps to ValueError (sampler.py:86-87, model.py:223-224) */
  HG_ECONFIG = 2,     /* maps to ConfigError (errors.py:4)                       */
  HG_EINVARIANT = 3,  /* maps to InvariantViolation (errors.py:8)                */
  HG_ECUDA = 4,       /* CUDA runtime failure                                    */
  HG_ENCCL = 5,       /* NCCL failure                                            */
  HG_ECAPACITY = 6    /* caller buffer too small                                 */
} hg_status;

#define HG_MAX_LAYERS 6
#define HG_MAX_GROUP 16  /* batches per grouped build / gather launch */

const char* hg_last_error(void);
int hg_version(void);
int hg_device_sync(void* stream); /* cudaStreamSynchronize + error-flag check */
/* Kernel-launch counter (every kernel this library launches) and optional
 * CUDA-event timing of kernel sites: 0 build, 1 layer-1 aggregate,
 * 2 layer-1 GEMM, 3 layer-1 dW, 4 whole step, 5 layer-2 aggregate, 6 SGD. */
int hg_launch_count(long long* out, int reset);
/* per-CTA clock64 phase stamps of hg_mg_build (builds with -DHG_BUILD_PROFILE only) */
int hg_debug_build_phases(long long* out, int n);
int hg_prof_enable(int on);
int hg_prof_read(int site, double* total_ms, int* count);
/* device timestamp (ns, %globaltimer) written to *slot in stream order
   (capturable: times the branches of a replayed graph) */
int hg_stamp(int64_t* slot, void* stream);

/* ------------------------------------------------------------------------
 * 1. Reference kernel boundary (gnnsim.kernels, kernels.py:31-34)
 * --------------------------------------------------------------------- */

/* replaces kernels.sample_frontier (_kernels_nb.py:55-90 / _kernels_np.py:55-84).
 * offsets int64[n+1], targets int32[m], frontier int64[f].  Outputs
 * counts_out int64[f] and flat_out int64[flat_cap]; *flat_len_host receives
 * sum(counts) (this call synchronises `stream` to report it). */
int hg_sample_frontier(const int64_t* offsets, const int32_t* targets, int64_t n_vertices,
                       const int64_t* frontier, int64_t n_frontier, int32_t fanout,
                       uint64_t state, int64_t* counts_out, int64_t* flat_out,
                       int64_t flat_cap, int64_t* flat_len_host, void* stream);

/* replaces kernels.feature_rows (_kernels_nb.py:109-122): out f32[n, dim]. */
int hg_feature_rows(const int64_t* ids, int64_t n, int32_t dim, uint64_t state, float* out,
                    void* stream);

/* replaces kernels.pick_k_smallest (_kernels_nb.py:92-106 / _kernels_np.py:87-98):
 * the k of ids[n] with the smallest keys (mix64(state ^ id) & HI32) | i, written to
 * out[min(k, n)] in index order.  n < 2^32. */
int hg_pick_k_smallest(const int64_t* ids, int64_t n, int64_t k, uint64_t state, int64_t* out,
                       void* stream);

/* replaces kernels.sbm_edges (_kernels_nb.py:22-52 / _kernels_np.py:17-52): every
 * unordered pair u < v of block_of[n] once; same-block pairs accepted by
 * (mode_in, thr_in), the others by (mode_out, thr_out) (mode 0 never, 1 iff
 * mix64(mix64(state ^ u) ^ v) < thr, 2 always).  *count_host receives the edge
 * count (synchronises `stream`); with us/vs non-NULL (capacity cap) the edges are
 * written in (u, v) lexicographic order. */
int hg_sbm_edges(const int64_t* block_of, int64_t n, int32_t mode_in, uint64_t thr_in,
                 int32_t mode_out, uint64_t thr_out, uint64_t state, int64_t* us, int64_t* vs,
                 int64_t cap, int64_t* count_host, void* stream);

/* ------------------------------------------------------------------------
 * 2. Counter RNG products (rng.py, engine.py:268-287, model.py:69-109)
 * --------------------------------------------------------------------- */

/* Feature table init: row i of a shard = feature_rows(v_i) (featstore.py:161-184),
 * v_i = ids[i] (ids != NULL) or first + i.  Row stride `ld` elements (ld >= dim,
 * padding columns zeroed).  dtype 0 = f32, 1 = bf16 (RNE). */
int hg_feature_table(const int64_t* ids, int64_t first, int64_t count, int32_t dim, int32_t ld,
                     uint64_t state, int32_t dtype, void* out, void* stream);

/* Epoch permutation: stable argsort of chain(state, v) for v < n
 * (engine.py:273-275).  perm_out int64[n].  ws_bytes query when ws == NULL. */
int hg_epoch_permutation(int64_t n, uint64_t state, int64_t* perm_out, void* ws,
                         size_t* ws_bytes, void* stream);

/* Device-side iteration cursor for graph-replayed training loops: reads
 * it = *it_dev, stages iteration it + ahead (if < iters) -- roots
 * perm[(it+ahead)*batch ...] into roots_out (skipped when roots_out is NULL)
 * and states[it+ahead] into key_out[0] -- then advances *it_dev by `advance`.
 * Every argument is fixed across steps, so the launch can live in a CUDA graph. */
int hg_iter_stage(const int64_t* perm, const uint64_t* states, int64_t iters, int64_t* it_dev,
                  int32_t batch, int32_t ahead, int32_t advance, int64_t* roots_out,
                  uint64_t* key_out, void* stream);
/* Group variant: iterations it+ahead .. it+ahead+n_batches-1 (those < iters):
 * roots of each (contiguous in perm) into roots_out[b * batch ..], their
 * states into key_out[b]; then advances the cursor by `advance`. */
int hg_iter_stage_group(const int64_t* perm, const uint64_t* states, int64_t iters,
                        int64_t* it_dev, int32_t batch, int32_t n_batches, int32_t ahead,
                        int32_t advance, int64_t* roots_out, uint64_t* key_out, void* stream);
/* Ranged variant (multi-GPU: this rank's roots of iteration it are
 * roots[ranges[2it] .. ranges[2it+1])): copies at most `cap` of them, writes
 * the count to *n_out (device), stages states[it+ahead], advances the cursor. */
int hg_iter_stage_ranged(const int64_t* roots, const int64_t* ranges, const uint64_t* states,
                         int64_t iters, int64_t* it_dev, int32_t cap, int32_t ahead,
                         int32_t advance, int64_t* roots_out, int32_t* n_out, uint64_t* key_out,
                         void* stream);

/* mix64 throughput probe (blocks x 256 threads x per_thread hashes): the
 * measured integer ceiling the sampler's hashes/s are reported against. */
int hg_bench_mix64(int32_t blocks, int64_t per_thread, uint64_t* sink, void* stream);

/* Glorot init (model.py:87-90): out f64 or f32 [rows*cols] row-major. */
int hg_glorot(int32_t rows, int32_t cols, uint64_t state, int32_t dtype, void* out,
              void* stream);

/* ------------------------------------------------------------------------
 * 3. Synthetic graph generator (oracle/graphgen.py twin)
 * --------------------------------------------------------------------- */
typedef struct {
  int64_t n;
  int32_t n_blocks;
  int32_t n_levels;
  uint64_t key;           /* row key base: slot draws use mix64(key ^ v) */
  uint64_t deg_key;       /* chain(key, 0xDE): row-length draw           */
  uint32_t thr_in;        /* in-block acceptance threshold on hi32 (0..2^32-1) */
  int32_t in_always;      /* 1 when p_in >= 1 or n_blocks == 1 */
  int64_t block_start[65];
  uint64_t a[64], c[64], a_inv[64];
  uint64_t cum[64];
  int64_t lvl_size[64], deg_lo[64], deg_span[64];
} hg_graph_tables;

/* Pass 1: raw row lengths (pre-dedup) -> raw_deg int64[n]. */
int hg_graph_raw_degrees(const hg_graph_tables* t, int64_t* raw_deg, void* stream);
/* Pass 2: slots of rows [v0, v1) into raw_targets at raw_off[v]-raw_off[v0]. */
int hg_graph_fill(const hg_graph_tables* t, int64_t v0, int64_t v1, const int64_t* raw_off,
                  int32_t* raw_targets, void* stream);
/* Pass 3: per-row sort + unique + self-loop drop in place; row_len int64[v1-v0]. */
int hg_graph_canonicalize(int64_t v0, int64_t v1, const int64_t* raw_off, int32_t* raw_targets,
                          int64_t* row_len, void* ws, size_t* ws_bytes, void* stream);
/* Pass 4: compact canonical rows into targets at offsets[v]. */
int hg_graph_compact(int64_t v0, int64_t v1, const int64_t* raw_off, const int32_t* raw_targets,
                     const int64_t* offsets, int32_t* targets, void* stream);
/* inclusive/exclusive scans used by the host orchestration */
int hg_exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* ws,
                          size_t* ws_bytes, void* stream);

/* ------------------------------------------------------------------------
 * 4. Micrograph batch: sampling + dedup/relabel + need-chain plan
 *    (sampler.py:84-106, model.py:183-198)
 * --------------------------------------------------------------------- */
typedef struct {
  int32_t n_layers;                    /* L */
  int32_t fanout[HG_MAX_LAYERS];       /* fanout[h-1] for hop h (hop 1 = root's neighbours) */
  int32_t cap_lay[HG_MAX_LAYERS + 1];  /* per-root capacity of layers[k] */
  int32_t cap_need[HG_MAX_LAYERS + 1]; /* per-root capacity of need[k] */
  int32_t cand_cap;                    /* per-task candidate buffer (threshold select) */
  int32_t sort_cap;                    /* power-of-two smem sort buffer */
  int32_t smem_bytes;                  /* dynamic smem of the build kernel */
  int32_t ws_root_ints;                /* padded per-root workspace (int32 words) */
} hg_mg_layout;

typedef struct {
  /* compact outputs, global row numbering; index k = layer 0..L */
  int32_t* need_ids[HG_MAX_LAYERS + 1];  /* vertex ids of need[k] rows                */
  int32_t* need_off[HG_MAX_LAYERS + 1];  /* [R+1] first row of each root in need[k]    */
  int8_t* in_layer[HG_MAX_LAYERS + 1];   /* 1 iff the need[k] row is in layers[k]      */
  int32_t* self_pos[HG_MAX_LAYERS + 1];  /* k>=1: row of the same vertex in need[k-1]  */
  int32_t* nbr_off[HG_MAX_LAYERS + 1];   /* k>=1: [N_k+1] CSR of sampled pairs by dst  */
  int32_t* nbr_idx[HG_MAX_LAYERS + 1];   /* k>=1: need[k-1] row of each pair's source  */
  int32_t* pair_off[HG_MAX_LAYERS + 1];  /* k>=1: [R+1] first pair of each root         */
  int32_t* totals;                       /* [2L+2]: N_0..N_L, P_1..P_L, err             */
  /* layer 1 by vertex id (the feature gather skips the need[0] indirection):
   * nbr_vid1[j] = need_ids[0][nbr_idx[1][j]], self_vid1[a] = need_ids[1][a]
   * row; NULL = not produced */
  int32_t* nbr_vid1;
  int32_t* self_vid1;
} hg_mg_batch;

/* Fill capacities / smem / workspace for a fanout list; returns HG_ECONFIG if
 * the per-root tile does not fit in shared memory. */
int hg_mg_plan_layout(int32_t n_layers, const int32_t* fanout, hg_mg_layout* out);

/* Sample + build micrographs for n_roots roots.  Root i uses stream key
 * mix64(iter_state[i / roots_per_state] ^ roots[i]) where iter_state holds
 * chain(sampler_seed, epoch, iteration) (sampler.py:52-54), or, when
 * roots_per_state == 0, iter_state[i] itself (caller-made keys); ws must hold
 * n_roots * layout.ws_root_ints int32 words.  err_flag: device int. */
int hg_mg_build(const int64_t* offsets, const int32_t* targets, int64_t n_vertices,
                const int64_t* roots, int32_t n_roots, const uint64_t* iter_state,
                int32_t roots_per_state, const hg_mg_layout* layout, int32_t* ws,
                hg_mg_batch* out, int* err_flag, void* stream);
/* Same with a device-resident root count: n_roots is the capacity (grid),
 * *n_roots_dev <= n_roots the roots actually built; the rest are empty
 * micrographs (zero rows).  Keeps launch arguments fixed for CUDA graphs. */
int hg_mg_build_n(const int64_t* offsets, const int32_t* targets, int64_t n_vertices,
                  const int64_t* roots, int32_t n_roots, const int32_t* n_roots_dev,
                  const uint64_t* iter_state, int32_t roots_per_state,
                  const hg_mg_layout* layout, int32_t* ws, hg_mg_batch* out, int* err_flag,
                  void* stream);
/* Run-ahead over several iterations in one launch: n_batches (<= HG_MAX_GROUP)
 * batches of n_roots roots each, roots[b * n_roots + i]; batch b's stream keys
 * follow the hg_mg_build rule over the whole group (roots_per_state = n_roots
 * with iter_state[b] = chain(sampler_seed, epoch, it0 + b)); outs[b] receives
 * a complete batch (own numbering and totals), exactly what hg_mg_build would
 * write for that batch alone.  n_roots_dev: NULL or int32[n_batches] device
 * counts (capacity n_roots each).  ws holds n_batches * n_roots roots.  The
 * gain over n_batches separate builds is occupancy: one 1024-root batch is
 * ~1.4 waves of build CTAs, a group keeps every SM busy through the tail.
 * ctas_per_sm > 0: a persistent grid of that many build CTAs per SM strides
 * over the roots (leaves registers / smem on every SM for kernels running
 * concurrently, e.g. the training branch of the graph loop); 0 = CTA/root. */
int hg_mg_build_group(const int64_t* offsets, const int32_t* targets, int64_t n_vertices,
                      const int64_t* roots, int32_t n_roots, int32_t n_batches,
                      const int32_t* n_roots_dev, const uint64_t* iter_state,
                      int32_t roots_per_state, const hg_mg_layout* layout, int32_t* ws,
                      const hg_mg_batch* outs, int* err_flag, int32_t ctas_per_sm, void* stream);

/* Partitioned topology (north_star: CSR rows sharded by home server): shard h
 * is a local CSR (offsets int64[n_h + 1], targets int32) in HBM of GPU h,
 * passed as device pointers valid on the calling GPU (its own shard, peers'
 * mapped over NVLink with hg_ipc_open).  Vertex v's row: contiguous
 * partitions (home_of == NULL) -- shard h holds [vstart[h], vstart[h+1]),
 * local row v - vstart[h]; arbitrary partitions -- shard home_of[v], local row
 * row_of[v] (int32[n] each, device).  Row degrees must be < 2^26. */
#define HG_MAX_SHARDS 16
typedef struct {
  int32_t n_shards;
  const int64_t* offsets[HG_MAX_SHARDS];
  const int32_t* targets[HG_MAX_SHARDS];
  int64_t vstart[HG_MAX_SHARDS + 1];
  const int32_t* home_of;
  const int32_t* row_of;
} hg_csr_shards;

/* hg_mg_build_group over a sharded CSR (remote rows read over NVLink). */
int hg_mg_build_group_sharded(const hg_csr_shards* shards, int64_t n_vertices,
                              const int64_t* roots, int32_t n_roots, int32_t n_batches,
                              const int32_t* n_roots_dev, const uint64_t* iter_state,
                              int32_t roots_per_state, const hg_mg_layout* layout, int32_t* ws,
                              const hg_mg_batch* outs, int* err_flag, int32_t ctas_per_sm,
                              void* stream);

/* Kernel selection of hg_mg_build / _n / _group (process-wide): 0 (default)
 * builds two-layer micrographs with hop-1 fanout <= 31 and <= 256 hop-2 pairs
 * warp-per-root (8 roots per CTA, dynamic hop-2 task list), everything else
 * CTA-per-root; 1 forces the CTA-per-root kernel.  Both are bit-exact with
 * sampler.py:84-106 + model.py:183-198; the switch exists so the parity tests
 * can compare them. */
int hg_mg_build_mode(int32_t mode);


/* Greedy locality partitioner (graph.py:273-327): BFS region growing into
 * parts of <= cap vertices, seeds in seed_order (degree descending, id
 * ascending), one warp running the reference's sequential order exactly.
 * home int32[n] (-1 = leftover), queue int32[n] scratch. */
int hg_partition_greedy(const int64_t* offsets, const int32_t* targets, int64_t n,
                        int32_t n_servers, int64_t cap, const int64_t* seed_order,
                        int32_t* home, int32_t* queue, void* stream);
/* leftovers (home == -1) round-robin by their rank among leftovers */
int hg_partition_leftovers(int32_t* home, int64_t n, int32_t n_servers, const int64_t* rank,
                           void* stream);

/* ------------------------------------------------------------------------
 * 5. Forward / backward of a micrograph batch (model.py:213-287) and the
 *    synchronous update (model.py:299-324)
 * --------------------------------------------------------------------- */
typedef struct {
  int32_t n_layers;                      /* L                                          */
  int32_t arch;                          /* 0 = gcn, 1 = sage-mean                     */
  int32_t act_dtype;                     /* 0 = f32, 1 = bf16 activations / operands   */
  int32_t feat_dim;                      /* D (reference width)                        */
  int32_t feat_ld;                       /* Dp >= D: padded row stride (multiple of 8) */
  int32_t hidden;                        /* H (multiple of 8)                          */
  int32_t n_classes;                     /* C                                          */
  int32_t max_roots;
  int32_t max_rows[HG_MAX_LAYERS + 1];   /* capacity of need[k] rows                   */
  int32_t in_dim[HG_MAX_LAYERS + 1];     /* k>=1: GEMM K of layer k (padded)           */
  int32_t split_k;                       /* CTAs along the row reduction of dW         */
  int32_t use_tc;                        /* 1: tcgen05 GEMMs where act_dtype == bf16   */
  const void* features;                  /* [rows x feat_ld], act dtype                */
  const int32_t* feat_row;               /* vertex -> feature row; NULL = identity     */
  const int64_t* roots;                  /* [n_roots]                                  */
  uint64_t label_state;                  /* chain(label_seed, 0x1A) (model.py:99-100)  */
  hg_mg_batch mg;                        /* from hg_mg_build                           */
  float* W[HG_MAX_LAYERS + 1];           /* k>=1: [in_dim[k] x H] f32 master            */
  float* b[HG_MAX_LAYERS + 1];           /* k>=1: [H]                                  */
  float* Wc;                             /* [H x C]                                    */
  void* Wlp[HG_MAX_LAYERS + 1];          /* bf16 shadows of W (act_dtype == 1)         */
  void* Wclp;
  float* gW[HG_MAX_LAYERS + 1];          /* gradient accumulators (summed, unscaled)   */
  float* gb[HG_MAX_LAYERS + 1];
  float* gWc;
  void* agg[HG_MAX_LAYERS + 1];          /* [max_rows[k] x in_dim[k]] act dtype        */
  void* h[HG_MAX_LAYERS + 1];            /* [max_rows[k] x H] act dtype                */
  float* dh[HG_MAX_LAYERS + 1];          /* [max_rows[k] x H] f32                       */
  float* dagg;                           /* [max_k>=2 max_rows[k] x in_dim[k]] f32      */
  float* logits;                         /* [max_roots x C] (dlogits after backward)   */
  float* loss;                           /* [max_roots] per-root softmax-CE            */
  void* lowp_scratch;                    /* bf16 [max_rows[1] x H] (tcgen05 dW path)    */
  void* Wb[HG_MAX_LAYERS + 1];           /* bf16 copies of W (tcgen05 dX path)          */
  /* peer addressing (multi-GPU without staging): row of vertex v lives in
   * feat_peers[feat_home[v]] at row feat_row[v]; NULL = local table only */
  const void* feat_peers;                /* device array of S row-table pointers        */
  const int32_t* feat_home;              /* int32[n] home server of each vertex          */
  /* staged mode (device pre-gather): local vertices from `features` at
   * feat_row[v], remote ones from stage_base at stage_row[v] */
  const void* stage_base;
  const int32_t* stage_row;
  int32_t rank;
  int32_t agg1_ready;                    /* 1: hg_step_prologue already built agg[1]    */
  /* tensor-core classifier head (bf16 path): Cp = C rounded up to 64 */
  void* WcT;                             /* bf16 [C x H]  (K-major B of the logits)    */
  void* Wcp;                             /* bf16 [H x Cp] (K-major B of dz_L)          */
  void* dl_lowp;                         /* bf16 [max_roots x Cp] dlogits               */
  /* per-root capacity of need[k] rows (hg_mg_layout.cap_need); 0 = unknown.
   * Enables the per-root fused backward scatter when a root's rows fit smem. */
  int32_t root_rows[HG_MAX_LAYERS + 1];
  /* 1: the bf16 operand copies (Wlp, Wb, WcT, Wcp) already hold the current
   * parameters (hg_sgd_refresh ran last) -- the step skips its transposes */
  int32_t lowp_fresh;
  /* per-layer bound on the sampled neighbours of a need[k] row (the fanout of
   * the hop that produced layer k's pairs; 0 = unknown).  Sizes the shared-
   * memory slots of the TMA-staged layer-1 gather; rows above it take the
   * register path. */
  int32_t max_deg[HG_MAX_LAYERS + 1];
  /* 1: lowp_scratch holds one bf16 dz region per layer (rows max_rows[1] +
   * ... + max_rows[L], layer k after layers 1..k-1), so a layer's weight-
   * gradient GEMM can run on a forked stream while the next layer's scatter
   * writes its own dz; 0: one shared region (serial backward). */
  int32_t lowp_layered;
  /* staged mode: row handle of every need[0] entry of the batch (>= 0: row
   * of the local table, < 0: staging row -1-h), written by hg_resolve_rows
   * after each pre-gather; the layer-1 gather then indexes it through the
   * need-index pair lists (one L2-resident lookup per source row instead of
   * the home / staging-row lookups by vertex id).  NULL = by vertex id. */
  const int32_t* row_handle;
  /* explicit class labels of the roots (int32[max_roots]); NULL = hashed by
   * LabelOracle from label_state (model.py:93-109).  The per-micrograph
   * loss_and_backward(state, label, model) API passes its label here. */
  const int32_t* labels;
} hg_step_desc;

/* Side-branch budget of the run-ahead loop (process-wide): resident CTAs per
 * SM (1..3, default 3) of the grouped layer-1 gather (hg_step_prologue_group),
 * which runs beside the training branch (fewer leave registers for the
 * training kernels); agg_stream != 0 (default) reads the feature rows of
 * every layer-1 gather with an L2 evict-first policy. */
int hg_set_side_budget(int32_t agg_ctas_per_sm, int32_t agg_stream);

/* Step variant (process-wide): 1 = softmax-CE fused into the tcgen05 head
 * GEMM's epilogue (C <= 192), 0 (default) = head GEMM + separate softmax-CE. */
int hg_set_fused_head(int32_t on);

/* Step variant (process-wide): 1 = training steps run the top of the
 * network -- layer-L linear, classifier head, softmax-CE, dz_L with its bias
 * gradient, dagg_L -- as one tcgen05 kernel per 128 roots (k_umma_top,
 * tensor-core path, L >= 2, H <= 256, C <= 192); 0 (default) = the split
 * kernels (measured faster on B200).  Results agree up to
 * summation order. */
int hg_set_fused_top(int32_t on);
/* debug: phase timestamps of CTA 0 of later k_umma_top launches (NULL = off) */
int hg_top_trace(int64_t* trace);

/* Peer memory (one process per GPU): device allocations whose CUDA IPC
 * handles (64 bytes) other ranks map; and the reference pre-gather byte
 * accounting of an iteration's remote vertices without a host sync
 * (featstore.py:226-279): uniq_per_home[h] += #distinct ids homed at h != rank,
 * total_remote += #remote occurrences; bitmap: n/32 words, zero on entry/exit. */
int hg_alloc(size_t bytes, void** out);
int hg_free(void* p);
int hg_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream);
/* Gradient all-reduce over NVLink peer memory (model.py:299-324 across the
 * one-process-per-GPU ranks): each rank owns an IPC-shared exchange region of
 * hg_p2p_region_bytes(n_ranks, n) bytes (zeroed: hg_alloc); regions holds the
 * n_ranks region pointers as mapped on this GPU (own + peers').  grads[n] is
 * replaced by the sum over ranks.  seq (int64), counter (uint32) and err
 * (int32) are zero-initialised device words owned by this rank; a peer that
 * never publishes raises HG_EINVARIANT in *err instead of hanging.  Three
 * kernels: push this rank's accumulator into every peer's region + signal,
 * wait for every peer's signal, add the peers' slots. */
int hg_p2p_region_bytes(int32_t n_ranks, int64_t n, int64_t* bytes);
int hg_p2p_allreduce(float* grads, int64_t n, const uint64_t* regions, int32_t rank,
                     int32_t n_ranks, int64_t* seq, unsigned int* counter, int* err, void* stream);

/* *flag = HG_EINVARIANT if a[0..n) and b[0..n) differ bitwise (replica check of
 * the model hop without a host sync, model.py:311-314) */
int hg_flag_if_differ(const float* a, const float* b, int64_t n, int* flag, void* stream);
int hg_ipc_handle(void* p, void* handle_out);
int hg_ipc_open(const void* handle, void** out);
int hg_ipc_close(void* p);
int hg_remote_account(const int32_t* ids, const int32_t* n_dev, int32_t n_host,
                      const int32_t* home, int32_t rank, uint32_t* bitmap,
                      unsigned long long* uniq_per_home, unsigned long long* total_remote,
                      void* stream);
/* reset the bitmap words touched by ids (after every hg_remote_account of a
 * server-iteration, so one plan dedups across all its cells) */
int hg_remote_clear(const int32_t* ids, const int32_t* n_dev, int32_t n_host, uint32_t* bitmap,
                    void* stream);

/* NCCL (torch's libnccl, same process): communicator from a broadcast unique
 * id (128 bytes); gradient all-reduce fused with the SGD update
 * (model.py:299-324); model-hop ring shift of two buffers by delta servers
 * (engine.py:610-618).  All enqueue on `stream`, no host synchronisation. */
int hg_nccl_unique_id(void* out);
int hg_nccl_init(const void* id, int nranks, int rank, void** comm_out);
int hg_nccl_destroy(void* comm);
int hg_allreduce_sgd(void* comm, float* params, float* grads, int64_t n, float lr,
                     float inv_batch, void* stream);
int hg_shift(void* comm, int rank, int nranks, int delta, const float* send0, const float* send1,
             float* recv0, float* recv1, int64_t n, void* stream);

/* Device pre-gathering over NVLink: dedup the remote vertices of ids[0..*n_dev)
 * (bitmap), list them, map vertex -> staging row, copy their rows from the
 * owners' shards (peers[home[v]] + local_row[v] * row_bytes) into `staging`;
 * per-home distinct counts feed the reference ledger. */
int hg_pregather_peer(const int32_t* ids, const int32_t* n_dev, const int32_t* home, int32_t rank,
                      const int32_t* local_row, const void* peers, int32_t row_bytes,
                      uint32_t* bitmap, int32_t* stage_list, int32_t* stage_row,
                      int32_t* stage_count, int32_t stage_cap, void* staging,
                      unsigned long long* uniq_per_home, unsigned long long* total_remote,
                      int* err, void* stream);
/* Same, with the per-home counts written to row *it_dev of an [iters x S]
 * table (uniq_per_home + *it_dev * row_stride): fixed arguments for graphs. */
int hg_pregather_peer_at(const int32_t* ids, const int32_t* n_dev, const int32_t* home,
                         int32_t rank, const int32_t* local_row, const void* peers,
                         int32_t row_bytes, uint32_t* bitmap, int32_t* stage_list,
                         int32_t* stage_row, int32_t* stage_count, int32_t stage_cap,
                         void* staging, unsigned long long* uniq_per_home, const int64_t* it_dev,
                         int32_t row_stride, unsigned long long* total_remote, int* err,
                         void* stream);
/* Push variant (NVLink, owner-side gather): the requester dedups its remote
 * vertices into its mailbox list (slot i -> staging row i of its mailbox,
 * stage_row[v] = i), signals its peers, and every owner copies the rows
 * homed on it from its local shard into the requesters' staging rows over
 * NVLink; returns (stream order) once every peer has signalled completion.
 * All ranks must call it the same number of times.  boxes: device array of
 * the S mailbox base addresses (own + IPC-mapped peers); layout offsets in
 * bytes; stamp: int32[n] zero-initialised dedup stamps (no clearing pass);
 * seq: device int64 sequence counter (starts at 0). */
int hg_pregather_push(const int32_t* ids, const int32_t* n_dev, const int32_t* home, int32_t rank,
                      int32_t n_ranks, const int32_t* local_row, const void* shard,
                      int32_t row_bytes, int32_t* stamp, int32_t* stage_row, int32_t stage_cap,
                      const void* boxes, void* own_box, int64_t o_flags, int64_t o_done,
                      int64_t o_count, int64_t o_list, int64_t o_staging,
                      unsigned long long* uniq_per_home, const int64_t* it_dev,
                      int32_t row_stride, unsigned long long* total_remote, int64_t* seq,
                      int* err, void* stream);
/* Push pre-gather of several batches at once (a run-ahead group): the
 * remote vertices of all n_seg id lists (ids[g][0..*n_dev[g]), host arrays of
 * device pointers) are deduplicated together and fetched with ONE
 * request/completion handshake; no ledger counting here (per-iteration
 * accounting: hg_remote_account_at).  Same mailbox layout as hg_pregather_push;
 * stage_cap must hold the group's distinct remote rows. */
int hg_pregather_push_multi(const int32_t* const* ids, const int32_t* const* n_dev, int32_t n_seg,
                            const int32_t* home, int32_t rank, int32_t n_ranks,
                            const int32_t* local_row, const void* shard, int32_t row_bytes,
                            int32_t* stamp, int32_t* stage_row, int32_t stage_cap,
                            const void* boxes, void* own_box, int64_t o_flags, int64_t o_done,
                            int64_t o_count, int64_t o_list, int64_t o_staging, int64_t* seq,
                            int* err, void* stream);
/* hg_remote_account charged to row (*it_dev + ahead) of an [iters x row_stride]
 * table (the reference's per-iteration pre-gather ledger, featstore.py:226-279). */
/* Group variants (one launch per kind for a whole run-ahead group of n_seg
 * iterations): ledger rows *it_dev + 1 + j with a per-iteration bitmap j
 * (bitmaps: n_seg x words, zero on entry and exit), and the row handles of
 * every iteration's need[0] entries (see hg_resolve_rows). */
int hg_remote_account_group(const int32_t* const* ids, const int32_t* const* n_dev,
                            int32_t n_seg, const int32_t* home, int32_t rank, uint32_t* bitmaps,
                            int64_t words, unsigned long long* uniq_table, const int64_t* it_dev,
                            int32_t row_stride, unsigned long long* total_remote, void* stream);
int hg_resolve_rows_group(const int32_t* const* ids, const int32_t* const* n_dev, int32_t n_seg,
                          const int32_t* home, int32_t rank, const int32_t* local_row,
                          const int32_t* stage_row, int32_t* const* out, void* stream);
int hg_remote_account_at(const int32_t* ids, const int32_t* n_dev, const int32_t* home,
                         int32_t rank, uint32_t* bitmap, unsigned long long* uniq_table,
                         const int64_t* it_dev, int32_t ahead, int32_t row_stride,
                         unsigned long long* total_remote, void* stream);
/* Row handles of a batch's need[0] entries after a pre-gather:
 * out[i] = home[v] == rank ? local_row[v] : -1 - stage_row[v], v = ids[i],
 * for i < *n_dev (see hg_step_desc.row_handle). */
int hg_resolve_rows(const int32_t* ids, const int32_t* n_dev, const int32_t* home, int32_t rank,
                    const int32_t* local_row, const int32_t* stage_row, int32_t* out,
                    void* stream);
/* Parameter-independent prologue of a step: the layer-1 gather + aggregate
 * (sets up agg[1]; run ahead of the previous iteration's training). */
int hg_step_prologue(const hg_step_desc* d, int32_t n_roots, int32_t backward, void* stream);
/* The same for n (<= HG_MAX_GROUP) steps that share one feature source (same
 * table / staging / peers): ONE gather launch over all their layer-1 rows. */
int hg_step_prologue_group(const hg_step_desc* const* descs, int32_t n, int32_t backward,
                           void* stream);

/* Forward + backward of the batch in d->mg for n_roots roots; gradients are
 * ADDED into gW/gb/gWc (the reference GradAccumulator, model.py:144-164). */
int hg_train_step(const hg_step_desc* d, int32_t n_roots, void* stream);
/* Forward only: fills logits (and agg/h).  Used by parity tests. */
int hg_forward(const hg_step_desc* d, int32_t n_roots, void* stream);

/* One training step followed (update != 0) by the SGD + bf16 operand refresh
 * of hg_sgd_refresh -- the unit the training loops replay.  With the
 * persistent step enabled (hg_set_persist) and an eligible descriptor
 * (bf16 tensor-core path, L = 2, H a multiple of 64 up to 256, C <= 256,
 * agg1_ready, lowp_fresh, n_roots == max_roots) the whole chain runs as ONE
 * kernel launch (k_step_persist: grid-wide barriers between the GEMM, gather,
 * softmax, scatter and SGD phases); otherwise hg_train_step then
 * hg_sgd_refresh.  Same results up to the order of atomic reductions. */
int hg_train_step_sgd(const hg_step_desc* d, int32_t n_roots, float* params, float* grads,
                      int64_t n, float lr, float inv_batch, int32_t update, void* stream);

/* Persistent-step switch (process-wide): on != 0 enables it; ctas = grid size
 * (0 = one CTA per SM); split_w1 = split-K of the layer-1 weight gradient
 * (0 = about one work item per CTA). */
int hg_set_persist(int32_t on, int32_t ctas, int32_t split_w1);
/* bf16 tcgen05 GEMM, fp32 accumulate: C[MxN] = A(m,k) B(k,n).
 * A K-major: [M x K] row-major, MN-major: [K x M];  B K-major: [N x K], MN-major: [K x N].
 * epi 0: C f32 store; 1: C bf16 = relu(acc + bias); 2: C f32 += acc (atomic, split-K).
 * Supported: (K,K) with epi 0/1 and (MN,MN) with epi 0/2; N in {64,128,192,256}. */
int hg_gemm_bf16(const void* A, int64_t lda, int a_mn_major, const void* B, int64_t ldb,
                 int b_mn_major, void* C, int64_t ldc, int32_t M, int32_t N, int32_t K,
                 int32_t epi, const float* bias, int32_t split, void* stream);
/* theta -= lr * (g * inv_batch); g = 0; refresh bf16 shadow (model.py:315-324). */
int hg_sgd_update(float* params, float* grads, void* shadow_bf16, int64_t n, float lr,
                  float inv_batch, void* stream);
/* SGD (as hg_sgd_update) fused with the refresh of the step's bf16 operand
 * copies of the parameters (Wlp = Wᵀ, Wb = W, WcT = W_cᵀ, Wcp = W_c padded),
 * so the next step can run with d->lowp_fresh = 1.  update = 0: refresh only. */
int hg_sgd_refresh(const hg_step_desc* d, float* params, float* grads, int64_t n, float lr,
                   float inv_batch, int32_t update, void* stream);
/* NCCL all-reduce of the gradients + hg_sgd_refresh. */
int hg_allreduce_sgd_refresh(void* comm, const hg_step_desc* d, float* params, float* grads,
                             int64_t n, float lr, float inv_batch, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HOPGNN_H_ */
