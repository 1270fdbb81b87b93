/* fssdp.h — C-ABI of libfssdp, the B200-native FSSDP (Hecate, arXiv 2502.02581) hot path.
 *
 * Two halves live behind this one header:
 *
 *   1. The host placement planner, bit-exact with the reference `moesim` package
 *      (/root/reference/pkg/src/moesim).  Every planner entry point names the
 *      reference function it replaces (file:line).  Placements cross the boundary as
 *      dense chunk-major masks  mask[c * D + d] != 0  <=>  (chunk c, device d) is held.
 *
 *   2. The device data plane (sm_100a kernels): gate top-k/load count, counts
 *      all-gather, SparseAllGather / SparseReduceScatter over peer HBM, token
 *      dispatch/combine by routing index, and the tcgen05 grouped expert GEMM.
 *      The reference has no device code; these implement the paper's
 *      semantics.
 *
 * Conventions:
 *   - plain pointers, sizes and a cudaStream_t (passed as void*); no torch types;
 *   - every function returns an int status: 0 ok, negative = error class below,
 *     mapped onto the reference error taxonomy (errors.py:8-53);
 *   - no allocation inside device entry points: workspaces come from the caller;
 *   - stream-ordered, one host thread per rank, no host callbacks;
 *   - peer-visible buffers live in a per-rank "symmetric heap" allocated with
 *     fssdp_heap_alloc; buffers sit at identical offsets on every rank, so a peer
 *     address is  peer_bases[rank] + offset  (peer_bases is a DEVICE array of
 *     world_size uint64 base addresses, own rank included).
 */
#ifndef FSSDP_H_
#define FSSDP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* ------------------------------------------------------------------ status codes */
#define FSSDP_OK 0
#define FSSDP_ERR_DIMENSION (-1)     /* moesim.errors.DimensionError            errors.py:20 */
#define FSSDP_ERR_INVALID_PAIR (-2)  /* moesim.errors.InvalidPairError          errors.py:28 */
#define FSSDP_ERR_ORPHAN_EXPERT (-3) /* moesim.errors.OrphanExpertError         errors.py:32 */
#define FSSDP_ERR_CUDA (-4)          /* CUDA runtime / launch failure (no reference analogue) */
#define FSSDP_ERR_INTERNAL (-5)      /* moesim.errors.InternalError             errors.py:52 */
#define FSSDP_ERR_INFEASIBLE (-6)    /* moesim.errors.InfeasibleSlotsError      errors.py:48 */
#define FSSDP_ERR_EMPTY_HISTORY (-7) /* moesim.errors.EmptyHistoryError         errors.py:36 */
#define FSSDP_ERR_DIM_MISMATCH (-8)  /* moesim.errors.DimensionMismatchError    errors.py:40 */

/* Verdict reasons (placement.py:26-28) */
#define FSSDP_VERDICT_OK 0
#define FSSDP_VERDICT_MISSING_CHUNK 1
#define FSSDP_VERDICT_DUPLICATE_OWNER 2
#define FSSDP_VERDICT_DROPPED_ENTRY 3

/* Library version string and the message of the last error on this thread. */
const char* fssdp_version(void);
const char* fssdp_last_error(void);

/* ================================================================== planner (host)
 * Topology = ClusterTopology (topology.py:14-49). */
typedef struct fssdp_topology {
  int32_t nodes;
  int32_t devices_per_node;
  double intra_bw; /* bytes/s */
  double inter_bw; /* bytes/s */
  double alpha;    /* s */
} fssdp_topology;

/* make_even_partition (placement.py:155-170): owner_out[c] for c in [0, num_chunks). */
int fssdp_make_even_partition(int32_t num_chunks, int32_t num_devices, int32_t* owner_out);

/* ShardPlan.even (placement.py:260-284): owner_out[l * experts + e]. */
int fssdp_shard_plan_even(int32_t layers, int32_t experts, int32_t devices, int32_t* owner_out);

/* validate_spag_pair / validate_sprs_pair (placement.py:200-211).
 * kind 0 = SpAG (pre partition, pre ⊆ post), 1 = SpRS (post partition, post ⊆ pre).
 * verdict_out[3] = {reason, chunk, device} (chunk/device = -1 when absent). */
int fssdp_validate_pair(int32_t kind, int32_t num_chunks, int32_t num_devices,
                        const uint8_t* pre_mask, const uint8_t* post_mask, int32_t* verdict_out);

/* spag_traffic / sprs_traffic (costmodel.py:87-132).  matrix_out is D*D row-major
 * [src, dst] bytes; report_out[4] = {sparsity, total_interdevice_bytes,
 * bottleneck_device, bottleneck_bytes} (SparsityReport, costmodel.py:60-84).
 * Returns FSSDP_ERR_INVALID_PAIR (with the verdict in fssdp_last_error) on bad pairs. */
int fssdp_spag_traffic(int32_t num_chunks, int32_t num_devices, const uint8_t* pre_mask,
                       const uint8_t* post_mask, double chunk_bytes, double* matrix_out,
                       double* report_out);
int fssdp_sprs_traffic(int32_t num_chunks, int32_t num_devices, const uint8_t* pre_mask,
                       const uint8_t* post_mask, double chunk_bytes, double* matrix_out,
                       double* report_out);

/* collective_latency (costmodel.py:149-182). */
int fssdp_collective_latency(int32_t num_devices, const double* matrix, const fssdp_topology* topo,
                             double* seconds_out);

/* overlap_degree (costmodel.py:185-194). */
int fssdp_overlap_degree(double t_nonmoe, const fssdp_topology* topo, double expert_bytes,
                         int64_t* t_out);

/* build_dispatch (dispatch.py:49-97): counts[D*E] (non-negative integers),
 * placement mask [E*D] -> route_out[D*E*D] (route[s, e, d]). */
int fssdp_build_dispatch(int32_t num_devices, int32_t num_experts, const int64_t* counts,
                         const uint8_t* placement_mask, const fssdp_topology* topo,
                         int64_t* route_out);

/* estimate_moe_latency (planner.py:205-216) on integral tokens[D*E]. */
int fssdp_estimate_moe_latency(int32_t num_devices, int32_t num_experts, const uint8_t* placement_mask,
                               const int64_t* tokens, const fssdp_topology* topo, double token_bytes,
                               double per_token_expert_time, double* seconds_out);

/* sparse_materialization (planner.py:171-197): base (a partition) + per-expert loads[E]
 * -> target mask [E*D] and added_per_device[D]. */
int fssdp_sparse_materialization(int32_t num_experts, int32_t num_devices, const uint8_t* base_mask,
                                 const double* per_expert_loads, int64_t t, int64_t m,
                                 const fssdp_topology* topo, uint8_t* target_out,
                                 int32_t* added_out);

/* calibrate (planner.py:228-276).  plan = (source, target) masks; actual[D*E] (float64).
 * out: accepted_out, new target mask, added_out[D], doubles_out[3] =
 * {extra_seconds, estimate_before, estimate_after}. */
int fssdp_calibrate(int32_t num_experts, int32_t num_devices, const uint8_t* source_mask,
                    const uint8_t* target_mask, const double* actual, int64_t remaining_m,
                    double t_remaining, const fssdp_topology* topo, double chunk_bytes,
                    double token_bytes, double per_token_expert_time, int32_t* accepted_out,
                    uint8_t* target_out, int32_t* added_out, double* doubles_out);

/* heterogeneous_sharding (planner.py:302-385): profile[L*E] -> owner_out[L*E]. */
int fssdp_heterogeneous_sharding(int32_t layers, int32_t experts, const double* profile, int64_t t,
                                 const fssdp_topology* topo, int32_t* owner_out);

/* estimate_loads (planner.py:32-42): mean of the last `window` of `n` stacked D*E
 * matrices (history is n*D*E row-major, oldest first). */
int fssdp_estimate_loads(int32_t n, int32_t rows, int32_t cols, const double* history,
                         int32_t window, double* mean_out);

/* One FSSDP layer-iteration decision, FssdpState.run_iteration per layer
 * (engine.py:491-553): adoption gate, calibration, fallback, then build_dispatch on the
 * actual counts.  Inputs: base partition owner[E], estimate est[D*E] (NULL = empty
 * history), actual counts[D*E] (int64), knobs.  Outputs: final target mask [E*D],
 * added[D], route[D*E*D], doubles_out[4] = {spag_lat, sprs_lat, remat_lat, calib_time},
 * flags_out[2] = {adopted_candidate, calibration_accepted}. */
typedef struct fssdp_layer_knobs {
  int64_t t;                    /* overlap degree (experts) */
  int64_t m;                    /* per-device replica capacity (experts) */
  int32_t calibration;          /* Policy.calibration */
  int32_t rematerialize;        /* Policy.rematerialize */
  double expert_bytes;          /* ModelConfig.expert_bytes */
  double token_bytes;           /* ModelConfig.token_bytes */
  double attn_fwd_time;         /* ModelConfig.attn_fwd_time */
  double per_token_expert_time; /* ModelConfig.per_token_expert_time */
} fssdp_layer_knobs;

int fssdp_plan_layer(int32_t num_experts, const int32_t* base_owner, const double* est,
                     const int64_t* actual, const fssdp_topology* topo,
                     const fssdp_layer_knobs* knobs, uint8_t* target_out, int32_t* added_out,
                     int64_t* route_out, double* doubles_out, int32_t* flags_out);

/* FssdpState._shard_score (engine.py:431-442), numpy summation order included:
 * score_out[2] = {max node load, max device load}. */
int fssdp_shard_score(int32_t layers, int32_t experts, const int32_t* owner, const double* profile,
                      const fssdp_topology* topo, double* score_out);

/* n_mats: expert matrices per slot — 2 = GeLU [W1 | W2], 3 = SwiGLU [W13 | W2] (W13 =
 * block-interleaved W1/W3, see FSSDP_EPI_SWIGLU).  d_model % 256 == 0, d_ff % 128 == 0.
 * Device plan tables of one rank for one layer-iteration, derived from the global plan
 * (base owner[E], target mask [E*D], route[D*E*D]) — every rank derives its own, nothing
 * is exchanged.  Packed into one blob of 16-byte-aligned sections whose offsets
 * fssdp_tables_layout returns; header_out[FSSDP_TAB_HEADER_INTS] = {n_slots, n_owned,
 * recv_rows, n_zero, n_spag, n_sprs_jobs, n_sprs_srcs, then per GEMM (fwd1, fwd2, dgrad2,
 * dgrad1, wgrad1, wgrad2): num_groups, n_tiles, total_tiles, then n_shared,
 * wgrad1_shared_tiles, wgrad2_shared_tiles, n_stage}.  n_stage = staging slots this rank
 * receives partial gradients in (see fssdp_sprs).  The wgrad group arrays list the n_shared
 * slots whose expert has other holders (the SpRS inputs) first, as a separately launchable
 * prefix; the remaining groups restart tile_start at 0, so a wgrad runs as two launches
 * (shared prefix, then the rest) and SpRS can start between them.
 * slot_layout (nullable): where a local slot's PARAMETERS live.  Null: the layer's own
 * contiguous region, slot s at index s.  {owned_base, replica_base}: a model-level region —
 * owned slot i at owned_base + i, replica j at replica_base + j (the SpAG copy list and the
 * GEMM B offsets use these indices; gradients and staging stay per-layer, owned slots only).
 * Layout semantics: plan_tables.py. */
#define FSSDP_TAB_HEADER_INTS 29
#define FSSDP_TAB_ROUTE_CUM 0   /* int32 [E][D+1] */
#define FSSDP_TAB_RECV_BASE 1   /* int32 [E][D]   */
#define FSSDP_TAB_ZERO_ROWS 2   /* int32 [<=E][2] {row, count} */
#define FSSDP_TAB_SPAG 3        /* int32 [<=E][3] {src_rank, src_slot, dst_slot} */
#define FSSDP_TAB_SPRS_JOBS 4   /* int32 [<=E][3] {dst_slot, src_begin, src_count} */
#define FSSDP_TAB_SPRS_SRCS 5   /* int32 [<=E*D][2] {rank, slot} */
#define FSSDP_TAB_GEMM0 6       /* 6 x fssdp_gemm_group [<=E] */
#define FSSDP_TAB_SLOT_EXPERT 12 /* int32 [<=E] expert id of each local slot */
#define FSSDP_TAB_SEG_START 13
#define FSSDP_TAB_SEG_ROWS 14
#define FSSDP_TAB_SEG_PADDED 15
#define FSSDP_TAB_SPRS_PULL 16  /* int32 [<=E*D][2] {rank, grads slot on that rank}, parallel
                                   to SPRS_SRCS (fssdp_sprs_pull) */
#define FSSDP_TAB_NSECTIONS 17
int fssdp_tables_layout(int32_t num_experts, int32_t num_devices, int64_t* offsets_out,
                        int64_t* total_bytes_out);
int fssdp_build_rank_tables(int32_t rank, int32_t num_devices, int32_t num_experts,
                            const int32_t* base_owner, const uint8_t* target_mask,
                            const uint8_t* pre_mask, const int64_t* route, int32_t d_model,
                            int32_t d_ff, int32_t n_mats, const int64_t* slot_layout,
                            uint8_t* blob, int64_t blob_bytes, int32_t* header_out);

/* The planning critical path in one call: fssdp_plan_layer on this rank's all-gathered
 * int32 counts [D*E], then fssdp_build_rank_tables for `rank` into the pinned `blob`, then
 * (if blob_dev) its upload on `stream`.  Outputs as the two calls'.  limits (nullable,
 * 6 entries): {slot capacity, receive-row capacity, staging-slot capacity, owned_base,
 * replica_base, replica-slot capacity} of this rank's buffers; owned_base < 0 = the
 * per-layer parameter region (slot_layout null), else the model-level one (slot_layout =
 * limits + 3; slot capacity then counts owned slots only).  A plan exceeding a capacity
 * returns FSSDP_ERR_INFEASIBLE before anything is uploaded. */
int fssdp_plan_layer_tables(int32_t num_experts, const int32_t* base_owner, const double* est,
                            const int32_t* counts, const fssdp_topology* topo,
                            const fssdp_layer_knobs* knobs, int32_t rank, const uint8_t* pre_mask,
                            int32_t d_model, int32_t d_ff, int32_t n_mats, const int64_t* limits,
                            uint8_t* target_out, int32_t* added_out, int64_t* route_out,
                            double* doubles_out, int32_t* flags_out, uint8_t* blob,
                            int64_t blob_bytes, int32_t* header_out, void* blob_dev, void* stream);

/* A copy-engine transfer (cudaMemcpyAsync, any pair of local / peer-heap addresses): moves
 * bytes over NVLink without occupying SMs, e.g. replica parts that land beside a GEMM. */
int fssdp_copy_async(void* dst, const void* src, int64_t bytes, void* stream);

/* Arguments of the dispatch fssdp_plan_layer_dispatch launches (fssdp_dispatch's, minus the
 * three plan-table pointers, n_zero and the stream, which come from the plan call). */
typedef struct fssdp_dispatch_launch {
  const void* x;
  const int32_t* topk_idx;
  const int32_t* slot_rank;
  const int32_t* tile_prefix;
  int64_t T;
  int32_t d_model, E, k, world;
  int32_t* slot_dest;
  int32_t* slot_pos;
  const uint64_t* peer_bases;
  int64_t recv_off;
  int64_t flags_off;
  int32_t rank, bar_slot;
  uint32_t epoch;
  uint32_t* grid_counter;
} fssdp_dispatch_launch;

/* The whole planning critical path of one layer-iteration with no Python in it: wait for
 * the counts readback flag (fssdp_host_wait), fssdp_plan_layer_tables, then — if disp and
 * blob_dev — fssdp_dispatch on the uploaded tables (route_cum / recv_base / zero_rows
 * sections of blob_dev, n_zero = header_out[3]) on the same stream. */
int fssdp_plan_layer_dispatch(const uint32_t* counts_flag, uint32_t counts_epoch,
                              double timeout_s, int32_t num_experts, const int32_t* base_owner,
                              const double* est, const int32_t* counts,
                              const fssdp_topology* topo, const fssdp_layer_knobs* knobs,
                              int32_t rank, const uint8_t* pre_mask, int32_t d_model,
                              int32_t d_ff, int32_t n_mats, const int64_t* limits,
                              uint8_t* target_out, int32_t* added_out, int64_t* route_out,
                              double* doubles_out, int32_t* flags_out, uint8_t* blob,
                              int64_t blob_bytes, int32_t* header_out, void* blob_dev,
                              void* stream, const fssdp_dispatch_launch* disp);

/* The estimate-based, adoption-gated materialization alone (engine.py:497-501 with
 * _adopt_materialization engine.py:406-429): depends only on the load history, so its
 * SparseAllGather can start before the gate.  fssdp_plan_layer's final target is either
 * a superset (calibration only extends) or the bare base partition (fallback). */
int fssdp_plan_candidate(int32_t num_experts, const int32_t* base_owner, const double* est,
                         const fssdp_topology* topo, const fssdp_layer_knobs* knobs,
                         uint8_t* target_out, int32_t* adopted_out);

/* ================================================================== device data plane */

/* GEMM group descriptor (one local expert = one group); see gemm_sm100.cu. */
typedef struct fssdp_gemm_group {
  int32_t m_tiles;    /* 128-row tiles along M */
  int32_t tile_start; /* exclusive prefix of m_tiles * n_tiles over groups */
  int32_t a_m;        /* A tensor-map coordinate of the group's M origin */
  int32_t a_k;        /* A tensor-map coordinate of the group's K origin */
  int32_t b_n;        /* B tensor-map coordinate of the group's N origin */
  int32_t b_k;        /* B tensor-map coordinate of the group's K origin */
  int32_t k_blocks;   /* number of 64-wide K blocks (0 => C tile written as zeros) */
  int32_t c_dest;     /* 0: C;  r + 1: the tensor c_dest_maps[r] (e.g. a peer's staging) */
  int64_t c_off;      /* element offset of the group's C[0, 0] in its destination */
  int32_t rows;       /* real rows along M (0 = all m_tiles * 128): with
                         FSSDP_GEMM_SWAP_TAIL the last M tile's padding is not computed */
  int32_t reserved;   /* 0 */
} fssdp_gemm_group;

#define FSSDP_EPI_BF16 0  /* C = bf16(acc) */
#define FSSDP_EPI_GELU 1  /* C = bf16(gelu'(acc)) (saved for backward), C2 = bf16(gelu(acc)) */
#define FSSDP_EPI_DGELU 2 /* C = bf16(acc * aux)  (aux = the saved gelu'(pre-activation)) */
#define FSSDP_EPI_F32 3   /* C = acc (fp32) */
/* SwiGLU experts.  W13 = [W1; W3] stored block-interleaved: rows [256b, 256b+128) are
 * W1 rows [128b, 128b+128) and rows [256b+128, 256b+256) are W3's, so a 256-wide output
 * tile of x·W13ᵀ holds a1 and a3 of the same 128 hidden units. */
#define FSSDP_EPI_SWIGLU 4  /* N = 2f, 256-wide tiles: C = bf16([a1|a3]) (saved, ldc = 2f),
                               C2 = bf16(silu(a1)·a3) (width ldc/2 = f) */
#define FSSDP_EPI_DSWIGLU 5 /* N = f (acc = dH): aux = the saved [a1|a3] (ldc = 2f);
                               C = bf16([dH·a3·silu'(a1) | dH·silu(a1)]) (ldc = 2f) */

/* Grouped GEMM  C_g = A_g · B_g  on tcgen05 (K5/K7).  A and B are bf16 2-D tensors
 * described by (inner, outer) element extents (inner contiguous).  a_mn / b_mn select
 * the operand major-ness: 0 = K-major (A: [M][K], B: [N][K]), 1 = MN-major
 * (A: [K][M], B: [K][N]).  N (= n_tiles * 256) is shared by every group.
 * C (and C2 / aux) is a row-major [c_rows][ldc] tensor (bf16, or fp32 for
 * FSSDP_EPI_F32); a group's C origin is element c_off (a multiple of ldc).
 * groups_dev: device array of num_groups descriptors; total_tiles must equal their sum,
 * or -1: read on the device from the last group (tile_start + m_tiles * n_tiles).
 * c_dest_maps (nullable): device array of 128-byte tensor maps made by
 * fssdp_epilogue_tmap, the destinations of groups with c_dest > 0 — a wgrad pushes a
 * replica's partial gradient into its owner's staging slot over NVLink this way.
 * flags: FSSDP_GEMM_N_FASTEST orders a group's tiles N-fastest (A tile shared in L2).
 * tile_sched (nullable): device int32[2], zero before the first launch and left zero after
 * each — the persistent CTAs then take tiles dynamically in list order from this counter
 * (CTAs that start late or share their SM with another kernel take fewer); null = a static
 * snake order.  Not shared by launches that may run concurrently. */
#define FSSDP_GEMM_N_FASTEST 1
/* CTA-pair (tcgen05 cta_group::2) 256 x 256 tiles; requires every group's m_tiles even. */
#define FSSDP_GEMM_CTA_PAIR 2
/* 128-wide N tiles (N % 256 != 0, e.g. d_ff = 1408); not with FSSDP_EPI_SWIGLU. */
#define FSSDP_GEMM_BN128 4
/* With CTA_PAIR and N_FASTEST, 256-wide N tiles, an even n_tiles and no tile_sched:
 * clusters of two CTA pairs on N tiles (2j, 2j+1) of one M tile; the A tile is loaded once
 * and multicast into both pairs (half the A operand's L2 -> SM traffic). */
#define FSSDP_GEMM_MULTICAST 8
/* Static order with CTA pairs and 256-wide N tiles (not the SwiGLU epilogues): when the
 * last round of tiles would leave more than half the CTA pairs idle, its tiles run as two
 * 256 x 128 halves each (same results; the short round takes half a tile's time). */
#define FSSDP_GEMM_SPLIT_TAIL 16
/* Token-side GEMMs (A K-major, CTA pairs, 256-wide N tiles; bf16, GeLU and dGeLU
 * epilogues): a group's last M tile whose real rows (fssdp_gemm_group.rows) end within 192
 * rows is computed with swapped operands (D^T = B^T A^T, N' = rows rounded up to 64), so
 * the segment padding to 256 rows costs at most 63 rows of MMA work; rows past N' are not
 * written. */
#define FSSDP_GEMM_SWAP_TAIL 32
int fssdp_grouped_gemm(int32_t a_mn, int32_t b_mn, int32_t epilogue, const void* a, int64_t a_inner,
                       int64_t a_outer, const void* b, int64_t b_inner, int64_t b_outer,
                       const fssdp_gemm_group* groups_dev, int32_t num_groups, int32_t n_tiles,
                       int32_t total_tiles, void* c, void* c2, const void* aux,
                       const void* c_dest_maps, int64_t ldc, int64_t c_rows, int32_t flags,
                       int32_t* tile_sched, void* stream);
/* The epilogue tensor map fssdp_grouped_gemm builds for C = [rows][ldc] at `base` with
 * this epilogue (128 bytes into map_out, host memory); upload it for c_dest_maps. */
int fssdp_epilogue_tmap(int32_t epilogue, const void* base, int64_t ldc, int64_t rows,
                        void* map_out);

#define FSSDP_GATE_TILE 64 /* tokens per gate CTA (slot ranks are tile-relative) */

/* K1: logits = x · Wgᵀ (+ bias) (fp32), top-k (ties -> lower expert id), renormalised
 * softmax weights, tile-relative slot ranks (token-slot order (t, j) ascending) and
 * per-tile expert histograms.  x [T*d] bf16, wg [E*d] fp32, bias [E] fp32 or NULL.
 * logits may be NULL.  tile_counts[ceil(T/64) * E]. */
int fssdp_gate_topk(const void* x, const float* wg, const float* bias, int64_t T, int32_t d,
                    int32_t E, int32_t k, float* logits, int32_t* topk_idx, float* topk_w,
                    int32_t* slot_rank, int32_t* tile_counts, void* stream);

/* Top-k / weights / ranks only, from given fp32 logits [T*E] (same semantics as K1's
 * tail; used to pin K1's selection bit-exactly against the CPU oracle). */
int fssdp_topk_from_logits(const float* logits, int64_t T, int32_t E, int32_t k, int32_t* topk_idx,
                           float* topk_w, int32_t* slot_rank, int32_t* tile_counts, void* stream);

/* K2: exclusive scan of tile_counts over tiles (tile_prefix, same shape), this rank's
 * per-expert totals, and the counts all-gather: the row is stored into every peer's
 * D x E int32 table at heap offset table_off (row = rank), followed by a device
 * barrier (barrier slot `bar_slot`, value `epoch`; a negative bar_slot skips every
 * barrier of an entry point — single rank, or lockstep emulation of several ranks). */
/* K1 + K2 in one launch (the layer's path): the tensor-core gate, whose last CTA to finish
 * then does fssdp_route_scan_allgather's work (tile_prefix, this rank's totals into every
 * rank's count table, world barrier on bar_slot / epoch).  ws: int32[1 + E] device
 * workspace, zero before the first call (left zero after each).  Shapes the tensor-core
 * gate does not take (d % 64 or E not in {8, 16, 32, 64}) run the two kernels.
 * local_tables (nullable; world must be 1): a device table blob of fssdp_tables_layout(E, 1)
 * whose dispatch sections are filled from the counts — route_cum, recv_base and zero_rows
 * with one {row, count >= 0} entry per expert (pass n_zero = E to fssdp_dispatch) — equal to
 * what fssdp_build_rank_tables derives for a single device, so the dispatch can be
 * launched before the host plan.  local_d_ff > 0 (with local_tables): the six GEMM tables
 * too (fssdp_local_gemm_tables for d_model = d, local_d_ff, local_n_mats,
 * local_param_base), so the forward
 * GEMMs (total_tiles = -1) can be queued before the host plan.  counts_host (nullable):
 * host boundary #1 in the same
 * launch — after the count barrier the whole D x E table (counts_bytes, a multiple of 16)
 * is copied to this mapped pinned buffer and *flag_host := flag_value (system-scope
 * release), what fssdp_push_host would do as a separate kernel. */
int fssdp_gate_route(const void* x, const float* wg, const float* bias, int64_t T, int32_t d,
                     int32_t E, int32_t k, int32_t* topk_idx, float* topk_w, int32_t* slot_rank,
                     int32_t* tile_counts, int32_t* tile_prefix, int32_t* ws,
                     const uint64_t* peer_bases, int64_t table_off, int64_t flags_off,
                     int32_t rank, int32_t world, int32_t bar_slot, uint32_t epoch,
                     int32_t* local_tables, int32_t local_d_ff, int32_t local_n_mats,
                     int32_t local_param_base, void* counts_host, int64_t counts_bytes,
                     uint32_t* flag_host, uint32_t flag_value, void* gemm_ws,
                     int64_t gemm_ws_bytes, void* stream);
/* Workspace bytes of the tensor-core gate path of fssdp_gate_route (gemm_ws, device
 * memory): the logits x . [hi(Wg); lo(Wg)] as one tcgen05 grouped-GEMM launch (fp32 C of
 * T x 128), then the selection / count kernel.  E <= 64, d % 64 == 0. */
int64_t fssdp_gate_gemm_ws_bytes(int64_t T, int32_t d);
int fssdp_route_scan_allgather(const int32_t* tile_counts, int32_t n_tiles, int32_t E,
                               int32_t* tile_prefix, const uint64_t* peer_bases, int64_t table_off,
                               int64_t flags_off, int32_t rank, int32_t world, int32_t bar_slot,
                               uint32_t epoch, void* stream);

/* Dense all-reduce of a small replicated gradient over P2P, to run after a world barrier:
 * out[i] = sum over ranks p = 0..world-1 (in rank order, fp32) of rank p's partial at heap
 * offset src_off (n floats, n % 4 == 0, 16-byte aligned) — the same bits on every rank.
 * Replaces the NCCL all-reduce of the gate's dWg (replicated gate, data-parallel grad). */
int fssdp_sum_peers(const uint64_t* peer_bases, int32_t world, int64_t src_off, int64_t n,
                    float* out, void* stream);

/* Device barrier across the world (system-scope release/acquire on flag pads). */
int fssdp_barrier(const uint64_t* peer_bases, int64_t flags_off, int32_t rank, int32_t world,
                  int32_t bar_slot, uint32_t epoch, void* stream);

/* Barrier-protocol self-test (test infrastructure for the multi-rank path on ONE GPU): world
 * emulated ranks (heaps at peer_bases) as the CTAs of one cooperative launch; `rounds`
 * rounds of peer stores -> world barrier (bar_slot, epochs epoch0 ..) -> check.  Each heap
 * needs FSSDP_SELFTEST_BYTES at data_off.  *errors (device int) += mismatched words.
 * bar_slot < 0 skips the barrier: the negative control (stale words expected); skew_ns > 0
 * delays rank r's stores by r * skew_ns each round (makes a missing barrier visible). */
#define FSSDP_SELFTEST_THREADS 256
#define FSSDP_SELFTEST_BYTES (2 * 32 * FSSDP_SELFTEST_THREADS * 4)
int fssdp_barrier_selftest(const uint64_t* peer_bases, int64_t flags_off, int64_t data_off,
                           int32_t world, int32_t rounds, int32_t bar_slot, uint32_t epoch0,
                           int32_t skew_ns, int32_t* errors, void* stream);

/* K4: dispatch.  For token-slot (t, j) with expert e and global rank r within
 * (this source, e) [tile_prefix + slot_rank], the destination d is the first with
 * route_cum[e*(D+1) + d + 1] > r and the row lands at recv_base[e*D + d] + r - route_cum[..d].
 * x rows (bf16, d_model wide) are pushed into peer d's receive buffer (heap offset
 * recv_off).  slot_dest/slot_pos record the destination for the combine.  zero_rows
 * ([n_zero * 2] {row, count}) lists this rank's own padding rows, zeroed here.
 * Ends with a device barrier. */
int fssdp_dispatch(const void* x, const int32_t* topk_idx, const int32_t* slot_rank,
                   const int32_t* tile_prefix, int64_t T, int32_t d_model, int32_t E, int32_t k,
                   int32_t world, const int32_t* route_cum, const int32_t* recv_base,
                   int32_t* slot_dest, int32_t* slot_pos, const uint64_t* peer_bases,
                   int64_t recv_off, const int32_t* zero_rows, int32_t n_zero,
                   int64_t flags_off, int32_t rank, int32_t bar_slot, uint32_t epoch,
                   uint32_t* grid_counter, void* stream);

/* Single rank (N = 1): the six grouped-GEMM tables of the fssdp_tables_layout(E, 1) blob at
 * local_tables, written on the device from this rank's expert totals (the counts row at
 * heap offset table_off, as fssdp_gate_route wrote it) — identical to what
 * fssdp_build_rank_tables writes for one rank (param_base: the parameter slot of expert 0,
 * the slot_layout owned_base; 0 for a per-layer region), so the forward GEMMs (launched
 * with total_tiles = -1) need not wait for the host plan. */
int fssdp_local_gemm_tables(const uint64_t* peer_bases, int32_t rank, int64_t table_off,
                            int32_t E, int32_t d_model, int32_t d_ff, int32_t n_mats,
                            int32_t param_base, void* local_tables, void* stream);

/* K6: combine.  y[t] = sum_j w[t, j] * Y_{dest}[pos]  (fp32, j ascending) -> bf16.
 * Y rows are pulled from peer heaps (offset y_off).  y_slots (nullable, bf16 [T*k, d_model]):
 * the gathered rows are also stored there in slot order, so the backward's <dy, Y> reads
 * them from local HBM instead of pulling them over NVLink a second time. */
int fssdp_combine(const int32_t* slot_dest, const int32_t* slot_pos, const float* topk_w,
                  int64_t T, int32_t d_model, int32_t k, const uint64_t* peer_bases, int64_t y_off,
                  void* y_out, void* y_slots, void* stream);

/* K7 (token side of backward): for every slot, g[t, j] = <dy_t, Y_slot> (fp32) and
 * bf16(w[t, j] * dy_t) is pushed to the slot's destination dY receive buffer
 * (heap offset dy_recv_off).  Y_slot comes from y_slots (the forward combine's copy) when
 * non-null, else from the peer heaps (offset y_off).  slot_grad may be NULL: the dots are
 * then left to fssdp_combine_dx_dots.  dlogit_out (nullable, needs 4 % k == 0 and
 * slot_grad): the gate's dlogit [T*k] (as fssdp_combine_dx defines it) is written here too,
 * so the gate backward can start before the dX combine.  Zeroes own padding rows, ends with a device
 * barrier. */
int fssdp_dispatch_grad(const void* dy, const int32_t* slot_dest, const int32_t* slot_pos,
                        const float* topk_w, int64_t T, int32_t d_model, int32_t k,
                        const uint64_t* peer_bases, int64_t y_off, const void* y_slots,
                        int64_t dy_recv_off, float* slot_grad, float* dlogit_out,
                        const int32_t* zero_rows, int32_t n_zero, int64_t flags_off,
                        int32_t rank, int32_t world, int32_t bar_slot, uint32_t epoch,
                        uint32_t* grid_counter, void* stream);

/* K7 (gate + combine side of backward):
 *   dlogit[t, j] = w_j (g_j - sum_i w_i g_i)            (renormalised top-k softmax)
 *   dx[t] = sum_j dXe_{dest}[pos] + sum_j dlogit[t, j] * Wg[idx_j]     -> bf16
 * dXe rows are pulled from peer heaps (offset dxe_off).  dlogit_out [T*k] fp32 (nullable:
 * not written, e.g. when fssdp_dispatch_grad already wrote it). */
int fssdp_combine_dx(const int32_t* slot_dest, const int32_t* slot_pos, const int32_t* topk_idx,
                     const float* topk_w, const float* slot_grad, const float* wg, int64_t T,
                     int32_t d_model, int32_t E, int32_t k, const uint64_t* peer_bases,
                     int64_t dxe_off, float* dlogit_out, void* dx_out, void* stream);
/* The same, with the gate's per-slot <dy_t, Y_slot> computed here instead of in
 * fssdp_dispatch_grad (call that with slot_grad = NULL: it then only scatters w * dy, the
 * part on the critical path).  Y rows: y_slots [T*k, d] (combine's token-local copy) or,
 * when NULL, the expert-order rows at peer heap offset y_off.  Bit-identical dots (same
 * per-lane order); slot_grad_out [T*k] fp32 (nullable). */
int fssdp_combine_dx_dots(const int32_t* slot_dest, const int32_t* slot_pos,
                          const int32_t* topk_idx, const float* topk_w, const void* dy,
                          const void* y_slots, int64_t y_off, const float* wg, int64_t T,
                          int32_t d_model, int32_t E, int32_t k, const uint64_t* peer_bases,
                          int64_t dxe_off, float* slot_grad_out, float* dlogit_out, void* dx_out,
                          void* stream);

/* Gate weight gradient dWg[e] = sum_t dlogit[t, e] x[t]  (fixed order; fp32 [E*d]).
 * workspace: fp32 [ceil(T / FSSDP_WG_TILE) * E * d] (per-token-tile partials, reduced in
 * tile order). */
#define FSSDP_WG_TILE 64
int fssdp_gate_wgrad(const void* x, const int32_t* topk_idx, const float* dlogit, int64_t T,
                     int32_t d_model, int32_t E, int32_t k, float* workspace, float* dwg_out,
                     void* stream);
/* The same dWg on the tensor cores: the logit gradient as a dense bf16 [T, hi | lo] matrix
 * (~16 mantissa bits of the fp32 dlogit), one split-T grouped-GEMM launch of x^T times it,
 * and a fixed-order reduction of the splits (deterministic for a given T and SM count).
 * E <= 64, d_model % 256 == 0; ws: fssdp_gate_wgrad_tc_ws_bytes(T, d_model) device bytes. */
int64_t fssdp_gate_wgrad_tc_ws_bytes(int64_t T, int32_t d_model);
int fssdp_gate_wgrad_tc(const void* x, const int32_t* topk_idx, const float* dlogit, int64_t T,
                        int32_t d_model, int32_t E, int32_t k, void* ws, int64_t ws_bytes,
                        float* dwg_out, void* stream);

/* K3: SparseAllGather.  copies[n * 3] = {src_rank, src_slot, dst_slot}: pull
 * slot_bytes from peer src_rank's heap (offset param_off + src_slot * slot_bytes) into
 * this rank's heap (param_off + dst_slot * slot_bytes).  128-bit coalesced loads. */
int fssdp_spag(const uint64_t* peer_bases, int32_t rank, int64_t param_off, int64_t slot_bytes,
               const int32_t* copies, int32_t n_copies, void* stream);
/* The same pull with separate heap offsets for the source slots (on src_rank) and the
 * destination slots (here) — re-sharding moves owned shards through a staging region —
 * copying copy_bytes (0 = slot_bytes) of each slot from its start (callers shift the
 * offsets to copy a later part, e.g. W2 of [W1 | W2]), with an optional bound on its
 * footprint: max_ctas > 0 caps the grid (larger chunks per CTA), for a copy that runs
 * beside other kernels (the early SpAG of the planning gap: small latency-bound transfers
 * stall behind a full-width copy); 0 = full width. */
int fssdp_gather_slots(const uint64_t* peer_bases, int32_t rank, int64_t src_off, int64_t dst_off,
                       int64_t slot_bytes, int64_t copy_bytes, const int32_t* copies,
                       int32_t n_copies, int32_t max_ctas, void* stream);

/* K8: SparseReduceScatter, owner side.  The holders' wgrads already pushed their partial
 * gradients into this rank's staging slots (c_dest groups); here, per job
 * jobs[n * 3] = {dst_slot, src_begin, src_count} with srcs[* 2] = {rank, idx} in ascending
 * rank order (owner included):  grads[dst_slot] = sum over srcs (fp32, listed order) of
 * (rank == this rank ? grads[idx] : stage[idx]).  Local memory only; slot_elems elements
 * of elem_bytes per slot — 4: fp32, 2: bf16 (summed in fp32, rounded once; the reference's
 * grad_bytes = param bytes, engine.py:223) — grads / stage at heap offsets grad_off /
 * stage_off. */
int fssdp_sprs(const uint64_t* peer_bases, int32_t rank, int64_t grad_off, int64_t stage_off,
               int64_t slot_elems, int32_t elem_bytes, const int32_t* jobs, int32_t n_jobs,
               const int32_t* srcs, void* stream);
/* K8, pull variant — the standalone SparseReduceScatter (sprs_traffic's schedule,
 * costmodel.py:111-132): every holder's partial stays in its own grads slot and the owner
 * pulls them over NVLink through a TMA ring, summing in listed (ascending-rank) order:
 * grads[dst_slot] = sum over pull_srcs {r, slot} of rank r's grads[slot] (the
 * FSSDP_TAB_SPRS_PULL section; the owner's own entry is local; elem_bytes as fssdp_sprs).
 * The caller orders it after every holder's partials are complete (device barrier) and
 * keeps the holders' replica grads intact until it has finished. */
int fssdp_sprs_pull(const uint64_t* peer_bases, int32_t rank, int64_t grad_off,
                    int64_t slot_elems, int32_t elem_bytes, const int32_t* jobs, int32_t n_jobs,
                    const int32_t* pull_srcs, void* stream);

/* ================================================================== training step */
/* AdamW over n fp32 elements (n % 4 == 0): exp_avg / exp_avg_sq / master updated in place
 * from grads (fp32, or bf16 when grads_bf16 != 0; bias corrections of `step` >= 1, decoupled
 * weight decay), then params_bf16
 * (nullable: the master IS the parameter) = bf16(master).  The owner's expert shards keep
 * master / moments in the symmetric heap so a re-shard moves them with the parameters
 * (params + 6x state = the 7x expert_bytes of engine.py:233, 444-453).  Replaces nothing in
 * the reference (it prices the optimizer state, it has no optimizer). */
int fssdp_adam_step(void* params_bf16, float* master, float* exp_avg, float* exp_avg_sq,
                    const void* grads, int32_t grads_bf16, int64_t n, float lr, float beta1,
                    float beta2, float eps, float weight_decay, int64_t step, void* stream);

/* Owner-update epochs (flag pad slot `slot`, entry [slot][rank] of each rank's own pad):
 * fssdp_publish_epoch stores `epoch` (system-scope release) after every earlier write of the
 * stream — an owner's optimizer step — so peers may read its shards; fssdp_wait_epochs
 * blocks its stream until every rank < world published >= epoch (the early SpAG's copy
 * engines start reading owners' shards before any barrier of the step). */
int fssdp_publish_epoch(const uint64_t* peer_bases, int64_t flags_off, int32_t slot, int32_t rank,
                        uint32_t epoch, void* stream);
int fssdp_wait_epochs(const uint64_t* peer_bases, int64_t flags_off, int32_t slot, int32_t world,
                      uint32_t epoch, void* stream);

/* ================================================================== symmetric heap */
/* cudaMalloc'd, zero-initialised heap (bytes rounded up to 2 MiB). */
int fssdp_heap_alloc(size_t bytes, void** ptr_out);
int fssdp_heap_free(void* ptr);
/* CUDA IPC: 64-byte handle of a heap, and mapping a peer's handle into this process. */
int fssdp_ipc_handle(void* ptr, uint8_t* handle_out /* 64 bytes */);
int fssdp_ipc_open(const uint8_t* handle /* 64 bytes */, void** ptr_out);
int fssdp_ipc_close(void* ptr);
/* Number of SMs of the current device. */
int fssdp_num_sms(void);

/* Launch timing (measurement only).  fssdp_timing_arm(start, end) arms two CUDA events
 * (cudaEvent_t, timing enabled, e.g. from fssdp_event_create); the next device entry point
 * called on this host thread records `start` right before its first kernel launch — after
 * its host-side setup — and `end` right after its last, on the launching stream.
 * fssdp_timing_done() disarms and returns 1 if both were recorded (0: no kernel ran).
 * Unlike events recorded by the caller around the call, the window holds no host time
 * when the GPU is waiting for the launch. */
int fssdp_event_create(void** event_out);
int fssdp_event_destroy(void* event);
int fssdp_event_record(void* event, void* stream);
int fssdp_event_elapsed(void* start, void* end, float* ms_out);
int fssdp_timing_arm(void* start, void* end);
int fssdp_timing_done(void);
/* Plan-boundary transfers without the copy engines (which may be busy with the caller's
 * bulk input/output copies): fssdp_push_host copies `bytes` (multiple of 16, <= 16 MiB) of
 * device memory into pinned host memory with the SMs, then stores flag_value into
 * *flag_host (pinned, nullable) with system-scope release; fssdp_host_wait spins on the
 * host until *flag_host == value (or timeout_s); fssdp_pull_host copies pinned host memory
 * into device memory with the SMs. */
int fssdp_push_host(const void* src_dev, void* dst_host, int64_t bytes, uint32_t* flag_host,
                    uint32_t flag_value, void* stream);
int fssdp_host_wait(const uint32_t* flag_host, uint32_t value, double timeout_s);
int fssdp_pull_host(void* dst_dev, const void* src_host, int64_t bytes, void* stream);
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* FSSDP_H_ */
