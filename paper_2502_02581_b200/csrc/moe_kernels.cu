// FSSDP token-path and sparse-collective kernels for sm_100a.
//
//   K1  gate_topk_kernel        logits (CUDA-core fp32), top-k, renormalised weights,
//                               tile-relative slot ranks, per-tile expert histograms
//   K2  route_scan_kernel       tile prefix over the histograms + counts all-gather via
//                               peer stores + world barrier
//   K4  dispatch_kernel         push token rows into destination receive segments
//   K6  combine_kernel          pull expert outputs back, weighted sum (fixed fp32 order)
//   K7  dispatch_grad_kernel    <dy, Y> for the gate + push w*dy to the experts
//       combine_dx_kernel       pull dX rows back + gate input gradient
//       gate_wgrad_kernels      dWg (split-T partials, fixed-order reduce)
//   K3  spag_kernel             SparseAllGather: pull replica slots from owners
//   K8  sprs_kernel             SparseReduceScatter: owners pull + reduce replica grads
//
// Semantics follow the paper (PAPER.md:234-237 gate/top-k/combine, 370-386 SpAG/SpRS,
// 615-617 dispatch); the routing counts they execute come from the host planner
// (moesim build_dispatch, dispatch.py:49-97).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <chrono>

#include "fssdp_internal.h"
#include "ptx.cuh"

namespace fssdp {

constexpr int kMaxWorld = 32;
constexpr int kSelftestThreads = FSSDP_SELFTEST_THREADS;
constexpr int kGateTile = FSSDP_GATE_TILE;
constexpr int kGateThreads = 256;
constexpr int kGateChunk = 128;
constexpr int kGateMaxE = 64;
constexpr int kGateMaxK = 8;

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

// ------------------------------------------------------------------ world barrier
// Called by one full warp after the caller made its data writes visible
// (__syncthreads + __threadfence_system).  Epochs only grow, so flags never reset.
__device__ __forceinline__ void world_barrier_warp(const uint64_t* __restrict__ peer_bases,
                                                   int64_t flags_off, int rank, int world,
                                                   int slot, uint32_t epoch) {
  if (slot < 0) return;  // barrier disabled (single rank, or lockstep emulation)
  const int lane = threadIdx.x & 31;
  if (lane < world) {
    uint32_t* remote = reinterpret_cast<uint32_t*>(peer_bases[lane] + flags_off) +
                       slot * kMaxWorld + rank;
    st_release_sys(remote, epoch);
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(peer_bases[rank] + flags_off) +
                           slot * kMaxWorld + lane;
    // bounded spin: a peer that never arrives turns into a loud kernel fault after 30 s
    // instead of a silently hung GPU
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (static_cast<int32_t>(ld_acquire_sys(mine) - epoch) < 0) {
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > 30ull * 1000000000ull) __trap();
    }
  }
  __syncwarp();
}

// The two halves of world_barrier_warp, for a caller with work to overlap in between:
// every lane < world publishes this rank's arrival on that peer; later, the same lanes
// wait for every peer's arrival here (30 s bound, as above).
__device__ __forceinline__ void world_barrier_arrive(const uint64_t* __restrict__ peer_bases,
                                                     int64_t flags_off, int rank, int world,
                                                     int slot, uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  if (slot < 0 || lane >= world) return;
  uint32_t* remote = reinterpret_cast<uint32_t*>(peer_bases[lane] + flags_off) +
                     slot * kMaxWorld + rank;
  st_release_sys(remote, epoch);
}
__device__ __forceinline__ void world_barrier_wait(const uint64_t* __restrict__ peer_bases,
                                                   int64_t flags_off, int rank, int world,
                                                   int slot, uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  if (slot >= 0 && lane < world) {
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(peer_bases[rank] + flags_off) +
                           slot * kMaxWorld + lane;
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (static_cast<int32_t>(ld_acquire_sys(mine) - epoch) < 0) {
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > 30ull * 1000000000ull) __trap();
    }
  }
  __syncwarp();
}

// Grid-wide "all CTAs done" followed by the world barrier, run by the last CTA.
__device__ __forceinline__ void grid_done_then_barrier(uint32_t* grid_counter,
                                                       const uint64_t* __restrict__ peer_bases,
                                                       int64_t flags_off, int rank, int world,
                                                       int slot, uint32_t epoch) {
  if (slot < 0) return;
  __shared__ int is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    uint32_t prev = atomicAdd(grid_counter, 1u);
    is_last = (prev == gridDim.x * gridDim.y - 1) ? 1 : 0;
    if (is_last) {
      __threadfence_system();
      atomicExch(grid_counter, 0u);
    }
  }
  __syncthreads();
  if (is_last && threadIdx.x < 32) world_barrier_warp(peer_bases, flags_off, rank, world, slot, epoch);
}

__global__ void barrier_kernel(const uint64_t* peer_bases, int64_t flags_off, int rank, int world,
                               int slot, uint32_t epoch) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // launched with PDL (launch_pdl)
  __threadfence_system();
  world_barrier_warp(peer_bases, flags_off, rank, world, slot, epoch);
}

// Barrier protocol self-test: `world` emulated ranks in ONE cooperative launch (CTA r is
// rank r, all CTAs co-resident), so ranks that wait on each other never depend on the
// scheduler (separate spinning launches on one GPU are not guaranteed to run together).
// Round k: every rank stores a stamp block into every peer's heap (plain peer stores,
// like the dispatch / SpRS pushes), makes them visible the way the product kernels do
// (__syncthreads + __threadfence_system), joins world_barrier_warp with epoch0 + k, then
// checks every writer's block in its own heap.  Blocks alternate between two buffers, so a
// rank one round ahead never overwrites a block a peer is still checking.
__device__ __forceinline__ uint32_t selftest_stamp(int round, int writer, int i) {
  return (static_cast<uint32_t>(round) * 2654435761u) ^ (static_cast<uint32_t>(writer) << 20) ^
         static_cast<uint32_t>(i);
}

__global__ void barrier_selftest_kernel(const uint64_t* __restrict__ peer_bases,
                                        int64_t flags_off, int64_t data_off, int world,
                                        int rounds, int slot, uint32_t epoch0, int skew_ns,
                                        int* errors) {
  const int rank = blockIdx.x;
  const int n = blockDim.x;
  int bad = 0;
  for (int k = 0; k < rounds; ++k) {
    if (skew_ns > 0) __nanosleep(static_cast<unsigned>(rank) * static_cast<unsigned>(skew_ns));
    const int64_t blk = (static_cast<int64_t>(k & 1) * kMaxWorld + rank) * n + threadIdx.x;
    for (int p = 0; p < world; ++p)
      reinterpret_cast<uint32_t*>(peer_bases[p] + data_off)[blk] =
          selftest_stamp(k, rank, threadIdx.x);
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
    __syncthreads();
    if (threadIdx.x < 32)
      world_barrier_warp(peer_bases, flags_off, rank, world, slot, epoch0 + static_cast<uint32_t>(k));
    __syncthreads();
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(peer_bases[rank] + data_off);
    for (int w = 0; w < world; ++w) {
      const int64_t at = (static_cast<int64_t>(k & 1) * kMaxWorld + w) * n + threadIdx.x;
      if (mine[at] != selftest_stamp(k, w, threadIdx.x)) ++bad;
    }
  }
  if (bad) atomicAdd(errors, bad);
}

// ------------------------------------------------------------------ K1 gate
// Selection + weights + tile-relative ranks for the tile's tokens, logits in smem.
__device__ void gate_select_tile(const float* __restrict__ lg, int lg_stride, int tile, int64_t T,
                                 int E, int k, int32_t* s_idx, int32_t* s_cnt,
                                 int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
                                 int32_t* __restrict__ slot_rank,
                                 int32_t* __restrict__ tile_counts) {
  const int tid = threadIdx.x;
  const int64_t t0 = static_cast<int64_t>(tile) * kGateTile;
  const int valid = static_cast<int>(imin64(kGateTile, T - t0));
  if (tid < valid) {
    const float* row = lg + tid * lg_stride;
    uint64_t taken = 0;
    int sel[kGateMaxK];
    for (int j = 0; j < k; ++j) {
      int bi = -1;
      float best = 0.f;
      for (int e = 0; e < E; ++e) {
        if ((taken >> e) & 1ull) continue;
        float v = row[e];
        if (bi < 0 || v > best) {  // strict '>' keeps the lower expert id on ties
          best = v;
          bi = e;
        }
      }
      taken |= 1ull << bi;
      sel[j] = bi;
    }
    // renormalised softmax over the selected logits (GShard top-k): e_j = exp(l_j - l_0)
    float ex[kGateMaxK];
    float m = row[sel[0]];
    float s = 0.f;
    for (int j = 0; j < k; ++j) {
      ex[j] = expf(__fsub_rn(row[sel[j]], m));
      s = __fadd_rn(s, ex[j]);
    }
    const int64_t t = t0 + tid;
    for (int j = 0; j < k; ++j) {
      topk_idx[t * k + j] = sel[j];
      topk_w[t * k + j] = __fdiv_rn(ex[j], s);
      s_idx[tid * k + j] = sel[j];
    }
  }
  if (tid < E) s_cnt[tid] = 0;
  __syncthreads();
  if (tid < 32) {
    const int nslots = valid * k;
    const int lane = tid;
    for (int base = 0; base < nslots; base += 32) {
      const int slot = base + lane;
      const bool ok = slot < nslots;
      const int e = ok ? s_idx[slot] : -1;
      const uint32_t peers = __match_any_sync(0xffffffffu, e);
      const uint32_t below = peers & ((1u << lane) - 1u);
      int r = 0;
      if (ok) r = s_cnt[e] + __popc(below);
      __syncwarp();
      if (ok && (peers >> lane) == 1u) s_cnt[e] += __popc(peers);  // highest lane of the group
      __syncwarp();
      if (ok) slot_rank[t0 * k + slot] = r;
    }
    for (int e = lane; e < E; e += 32) tile_counts[static_cast<int64_t>(tile) * E + e] = s_cnt[e];
  }
}

// EPT = experts per thread (each thread owns one token and experts grp, grp+4, ...):
// templated so the inner loop carries no dead iterations for small E.
template <int EPT>
__global__ void __launch_bounds__(kGateThreads)
    gate_topk_kernel(const __nv_bfloat16* __restrict__ x, const float* __restrict__ wg,
                     const float* __restrict__ bias, int64_t T, int d, int E, int k,
                     float* __restrict__ logits,
                     int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
                     int32_t* __restrict__ slot_rank, int32_t* __restrict__ tile_counts) {
  // dynamic smem: xs [64][kGateChunk+8] bf16 | ws [E][kGateChunk+4] fp32; the logits
  // tile lg [64][kGateMaxE+1] fp32 reuses the xs/ws region once the d loop is done.
  extern __shared__ __align__(16) uint8_t gate_smem[];
  typedef __nv_bfloat16 XRow[kGateChunk + 8];
  typedef float WRow[kGateChunk + 4];
  typedef float LRow[kGateMaxE + 1];
  XRow* xs = reinterpret_cast<XRow*>(gate_smem);
  WRow* ws = reinterpret_cast<WRow*>(gate_smem + kGateTile * sizeof(XRow));
  LRow* lg = reinterpret_cast<LRow*>(gate_smem);
  __shared__ int32_t s_idx[kGateTile * kGateMaxK];
  __shared__ int32_t s_cnt[kGateMaxE];

  const int tid = threadIdx.x;
  const int tile = blockIdx.x;
  const int64_t t0 = static_cast<int64_t>(tile) * kGateTile;
  const int tok = tid >> 2;
  const int grp = tid & 3;
  float acc[EPT];
#pragma unroll
  for (int i = 0; i < EPT; ++i) acc[i] = 0.f;

  for (int c0 = 0; c0 < d; c0 += kGateChunk) {
    const int cw = min(kGateChunk, d - c0);  // multiple of 8
    // x chunk: 64 rows x cw bf16, 16-byte vectors
    for (int v = tid; v < kGateTile * (kGateChunk / 8); v += kGateThreads) {
      const int r = v / (kGateChunk / 8);
      const int c = (v % (kGateChunk / 8)) * 8;
      int4 val = make_int4(0, 0, 0, 0);
      if (t0 + r < T && c < cw)
        val = *reinterpret_cast<const int4*>(x + (t0 + r) * d + c0 + c);
      *reinterpret_cast<int4*>(&xs[r][c]) = val;
    }
    for (int v = tid; v < E * (kGateChunk / 4); v += kGateThreads) {
      const int e = v / (kGateChunk / 4);
      const int c = (v % (kGateChunk / 4)) * 4;
      float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
      if (c < cw) val = *reinterpret_cast<const float4*>(wg + static_cast<int64_t>(e) * d + c0 + c);
      *reinterpret_cast<float4*>(&ws[e][c]) = val;
    }
    __syncthreads();
#pragma unroll 4
    for (int i = 0; i < cw; i += 2) {
      const float2 xv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xs[tok][i]));
#pragma unroll
      for (int q = 0; q < EPT; ++q) {
        const int e = grp + 4 * q;
        if (e < E) {
          const float2 wv = *reinterpret_cast<const float2*>(&ws[e][i]);
          acc[q] = fmaf(xv.x, wv.x, acc[q]);
          acc[q] = fmaf(xv.y, wv.y, acc[q]);
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < EPT; ++q) {
    const int e = grp + 4 * q;
    if (e < E) lg[tok][e] = bias != nullptr ? __fadd_rn(acc[q], bias[e]) : acc[q];
  }
  __syncthreads();
  if (logits != nullptr) {
    for (int v = tid; v < kGateTile * E; v += kGateThreads) {
      const int r = v / E, e = v % E;
      if (t0 + r < T) logits[(t0 + r) * E + e] = lg[r][e];
    }
  }
  gate_select_tile(&lg[0][0], kGateMaxE + 1, tile, T, E, k, s_idx, s_cnt, topk_idx, topk_w,
                   slot_rank, tile_counts);
}

// ------------------------------------------------------------------ K1 on tensor cores
// Gate logits with mma.sync m16n8k16 (bf16 in, fp32 accumulate): x is exactly bf16 and the
// fp32 gate weights are split on the fly into hi = bf16(w) and lo = bf16(w - hi) (about 16
// mantissa bits), logits = x·hi + x·lo.  One warp = 16 tokens x all experts; a CTA = 4
// warps = one 64-token gate tile, so selection/ranks reuse gate_select_tile.  The HMMA
// path is ~50x fewer instructions than the CUDA-core kernel and leaves the kernel bound by
// reading x from HBM.
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4],
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, "
      "{%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void split_bf16x2(float2 w, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(w.x, w.y);
  const float2 hf = __bfloat1622float2(h);
  const __nv_bfloat162 l = __floats2bfloat162_rn(w.x - hf.x, w.y - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

// Count scan + all-gather tail of the fused gate (fssdp_gate_route), run by the gate's LAST
// CTA to finish (ticket in ws[0]; per-expert totals accumulated in ws[1..E] by atomics):
// tile_prefix[t][e] = sum of tile_counts[t'][e] over t' < t, this rank's totals written into
// every rank's count table, then the world barrier.  The other CTAs' tile counts are read
// through L2 (__ldcg): they were published with a fence before taking their ticket.
//
// local != nullptr (a single-rank layer): the placement cannot change (one device holds every
// expert, the route is the counts), so the dispatch tables are a function of the counts and
// are written here — route_cum [E][2], recv_base [E][1], zero_rows [E][2] (every expert,
// count 0 where the segment has no padding) in the fssdp_build_rank_tables layout — and the
// dispatch can run while the host plans.
struct GateLocalTables {
  int32_t* route_cum;
  int32_t* recv_base;
  int32_t* zero_rows;
  // host boundary #1 folded into the tail (nullable): after the count barrier, the whole
  // all-gathered counts table (n16 x 16 B) to mapped pinned host memory, then the flag
  int4* host_counts;
  int host_n16;
  uint32_t* host_flag;
  uint32_t host_flag_value;
  // (nullable) the six grouped-GEMM tables of the same single-rank blob, also written from
  // the totals, so the forward GEMMs need not wait for the host plan (fssdp_local_gemm_tables)
  fssdp_gemm_group* gemm0;
  int64_t gemm_stride;  // bytes between the six GEMM sections
  int32_t d_model, d_ff, n_mats;
  int32_t param_base;   // parameter slot of expert 0 (a model-level parameter region)
};

__device__ void write_local_tables(const int32_t* totals, int E, GateLocalTables local) {
  int32_t row = 0;
  for (int e = 0; e < E; ++e) {
    const int32_t c = totals[e], pad = (c + 255) / 256 * 256;  // CTA-pair GEMM M tile
    local.route_cum[2 * e] = 0;
    local.route_cum[2 * e + 1] = c;
    local.recv_base[e] = row;
    local.zero_rows[2 * e] = row + c;
    local.zero_rows[2 * e + 1] = pad - c;
    row += pad;
  }
}

// the two-kernel path's version (after fssdp_route_scan_allgather wrote the counts row)
__global__ void gate_local_tables_kernel(const uint64_t* peer_bases, int rank, int64_t table_off,
                                         int E, GateLocalTables local) {
  if (threadIdx.x == 0)
    write_local_tables(reinterpret_cast<const int32_t*>(peer_bases[rank] + table_off) + rank * E,
                       E, local);
}

// Single rank, N = 1: the six grouped-GEMM descriptor tables of fssdp_build_rank_tables
// (planner.cpp), written on the device from the expert totals — every expert is an owned
// slot (ascending), segments padded to 256 rows, no replica, no SpRS push; the wgrads list
// the slots longest-first (stable), as the host builder does.  The forward GEMMs can then be
// queued before the host plan exists (fssdp_grouped_gemm total_tiles = -1).  Thread e < E
// derives expert e's entries in O(E) (prefix of the padded rows, its rank in the wgrad
// order), so one block writes every table in a few hundred cycles.
__device__ void write_local_gemm_groups(const int32_t* __restrict__ tot, int E, int64_t d,
                                        int64_t f, int nm, fssdp_gemm_group* gemm0,
                                        int64_t stride, int param_base) {
  const int e = threadIdx.x;
  if (e >= E) return;
  const int64_t n1 = (nm - 1) * f;
  const int64_t bnf = f % 256 == 0 ? 256 : 128, bn1 = nm == 3 ? 256 : bnf, nf = (f + 255) / 256;
  const int64_t n_tiles[6] = {n1 / bn1, d / 256, nf, d / 256, d / 256, nf};
  const int32_t c = tot[e], pad = (c + 255) / 256 * 256;
  int32_t st = 0, before_tiles = 0, rank_w = 0, before_w = 0;
  for (int q = 0; q < E; ++q) {
    const int32_t pq = (tot[q] + 255) / 256 * 256;
    if (q < e) {
      st += pq;
      before_tiles += pq / 128;
    }
    if (pq > pad || (pq == pad && q < e)) {  // stable, padded rows descending
      ++rank_w;
      before_w += pq / 128;
    }
  }
  const int32_t mt = pad / 128, kt = (c + 63) / 64;
  const int64_t ps = param_base + e;  // expert e's parameter slot (gradients: slot e)
  const int32_t w1r = static_cast<int32_t>(ps * nm * f), w2r = static_cast<int32_t>(ps * nm * d);
  for (int gi = 0; gi < 6; ++gi) {
    fssdp_gemm_group x;
    switch (gi) {
      case 0: x = {mt, 0, st, 0, w1r, 0, static_cast<int32_t>(d / 64), 0, st * n1}; break;
      case 1: x = {mt, 0, st, 0, w2r, 0, static_cast<int32_t>(f / 64), 0, st * d}; break;
      case 2: x = {mt, 0, st, 0, 0, w2r, static_cast<int32_t>(d / 64), 0, st * n1}; break;
      case 3: x = {mt, 0, st, 0, 0, w1r, static_cast<int32_t>(n1 / 64), 0, st * d}; break;
      case 4: x = {static_cast<int32_t>(n1 / 128), 0, 0, st, 0, st, kt, 0, e * nm * f * d}; break;
      default: x = {static_cast<int32_t>(d / 128), 0, 0, st, 0, st, kt, 0, e * nm * f * d + n1 * d}; break;
    }
    const bool wgrad = gi >= 4;
    if (!wgrad) x.rows = c;  // the real rows (the last M tile's padding: FSSDP_GEMM_SWAP_TAIL)
    // m_tiles of a wgrad group = its output rows / 128 (the same for every expert)
    x.tile_start = static_cast<int32_t>((wgrad ? static_cast<int64_t>(rank_w) * x.m_tiles
                                               : before_tiles) * n_tiles[gi]);
    fssdp_gemm_group* g = reinterpret_cast<fssdp_gemm_group*>(
        reinterpret_cast<uint8_t*>(gemm0) + gi * stride);
    g[wgrad ? rank_w : e] = x;
  }
  (void)before_w;
}

__global__ void local_gemm_tables_kernel(const uint64_t* __restrict__ peer_bases, int rank,
                                         int64_t table_off, int E, int64_t d, int64_t f, int nm,
                                         fssdp_gemm_group* __restrict__ gemm0, int64_t stride,
                                         int param_base) {
  __shared__ int32_t s_tot[kGateMaxE];
  const int32_t* tot = reinterpret_cast<const int32_t*>(peer_bases[rank] + table_off) + rank * E;
  if (threadIdx.x < E) s_tot[threadIdx.x] = __ldcg(tot + threadIdx.x);
  __syncthreads();
  write_local_gemm_groups(s_tot, E, d, f, nm, gemm0, stride, param_base);
}

__device__ void gate_route_tail(int n_tiles, int E, const int32_t* __restrict__ tile_counts,
                                int32_t* __restrict__ tile_prefix, int32_t* __restrict__ ws,
                                const uint64_t* __restrict__ peer_bases, int64_t table_off,
                                int64_t flags_off, int rank, int world, int slot, uint32_t epoch,
                                GateLocalTables local, int32_t* s_stage, int stage_ints) {
  __shared__ int32_t csum[512];
  __shared__ int32_t s_tot[kGateMaxE];
  // 1. this rank's totals (accumulated by every CTA's atomics) into every rank's count
  //    table, then the barrier ARRIVAL: peers can proceed while the scan below runs
  if (threadIdx.x < E) {
    const int32_t total = __ldcg(ws + 1 + threadIdx.x);
    for (int p = 0; p < world; ++p)
      reinterpret_cast<int32_t*>(peer_bases[p] + table_off)[rank * E + threadIdx.x] = total;
    ws[1 + threadIdx.x] = 0;  // ready for the next call (stream order)
    s_tot[threadIdx.x] = total;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) __threadfence_system();
    __syncwarp();
    world_barrier_arrive(peer_bases, flags_off, rank, world, slot, epoch);
  }
  if (local.route_cum != nullptr && threadIdx.x == 0) write_local_tables(s_tot, E, local);
  if (local.gemm0 != nullptr)
    write_local_gemm_groups(s_tot, E, local.d_model, local.d_ff, local.n_mats, local.gemm0,
                            local.gemm_stride, local.param_base);
  // 2. the tile counts into shared memory in one coalesced pass (the gate's staged weights
  //    are dead by now), then the exclusive scan over tiles from there
  const int n = n_tiles * E;
  const bool staged = s_stage != nullptr && n <= stage_ints && (n % 4) == 0;
  if (staged) {
    const int4* src = reinterpret_cast<const int4*>(tile_counts);
    for (int i = threadIdx.x; i < n / 4; i += blockDim.x)
      reinterpret_cast<int4*>(s_stage)[i] = __ldcg(src + i);
    __syncthreads();
  }
  auto cnt = [&](int t, int e) {
    return staged ? s_stage[t * E + e] : __ldcg(tile_counts + static_cast<int64_t>(t) * E + e);
  };
  const int nthr = blockDim.x;
  const int chunks = (nthr < 512 ? nthr : 512) / E;
  const int per = (n_tiles + chunks - 1) / chunks;
  const int e = threadIdx.x % E;
  const int c = threadIdx.x / E;
  const bool active = c < chunks;
  const int t0 = c * per, t1 = min(n_tiles, t0 + per);
  if (active) {
    int32_t sum = 0;
#pragma unroll 8
    for (int t = t0; t < t1; ++t) sum += cnt(t, e);
    csum[threadIdx.x] = sum;
  }
  __syncthreads();
  if (threadIdx.x < E) {  // exclusive scan over the chunks of expert threadIdx.x
    int32_t run = 0;
    for (int q = 0; q < chunks; ++q) {
      const int32_t v = csum[q * E + threadIdx.x];
      csum[q * E + threadIdx.x] = run;
      run += v;
    }
  }
  __syncthreads();
  if (active) {
    int32_t run = csum[threadIdx.x];
    for (int t = t0; t < t1; ++t) {
      tile_prefix[static_cast<int64_t>(t) * E + e] = run;
      run += cnt(t, e);
    }
  }
  if (threadIdx.x == 0) ws[0] = 0;
  // 3. every peer's arrival (their rows of the count table are in)
  if (threadIdx.x < 32) world_barrier_wait(peer_bases, flags_off, rank, world, slot, epoch);
  if (local.host_counts != nullptr) {  // every rank's row is in (barrier): push the table
    __syncthreads();
    const int4* src = reinterpret_cast<const int4*>(peer_bases[rank] + table_off);
    for (int i = threadIdx.x; i < local.host_n16; i += blockDim.x)
      local.host_counts[i] = __ldcv(src + i);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      st_release_sys(local.host_flag, local.host_flag_value);
    }
  }
}

// NT = E / 8 expert tiles; KS = warps splitting d (the CTA is 4 x KS warps: 4 groups of 16
// tokens, each group's columns split KS ways, partial logits summed in smem in ks order) —
// more warps per SM for a kernel that is bound by the latency of reading x.  SW: the split
// gate weights are staged once per CTA in shared memory (one 16-byte record {hi, hi, lo,
// lo} per 4 columns, rows padded by 16 B) instead of re-read and re-split from L1/L2 by
// every warp inside the MMA loop.
template <int NT, int KS, bool SW>
__global__ void __launch_bounds__(128 * KS)
    gate_topk_mma_kernel(const __nv_bfloat16* __restrict__ x, const float* __restrict__ wg,
                         const float* __restrict__ bias, int64_t T, int d, int E, int k,
                         float* __restrict__ logits, int32_t* __restrict__ topk_idx,
                         float* __restrict__ topk_w, int32_t* __restrict__ slot_rank,
                         int32_t* __restrict__ tile_counts, int32_t* __restrict__ tile_prefix,
                         int32_t* __restrict__ ws, const uint64_t* __restrict__ peer_bases,
                         int64_t table_off, int64_t flags_off, int rank, int world, int slot,
                         uint32_t epoch, GateLocalTables local) {
  __shared__ float lg[kGateTile][kGateMaxE + 1];
  __shared__ float part[KS > 1 ? KS - 1 : 1][kGateTile][8 * NT + 1];
  __shared__ int32_t s_idx[kGateTile * kGateMaxK];
  __shared__ int32_t s_cnt[kGateMaxE];
  __shared__ int is_last;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tg = warp % 4, ks = warp / 4;
  const int g = lane >> 2, t4 = lane & 3;
  const int tile = blockIdx.x;
  const int64_t t0 = static_cast<int64_t>(tile) * kGateTile + tg * 16;
  const int64_t r0 = t0 + g, r1 = t0 + g + 8;
  const bool v0 = r0 < T, v1 = r1 < T;
  const int4* xr0 = reinterpret_cast<const int4*>(x + (v0 ? r0 : 0) * d);
  const int4* xr1 = reinterpret_cast<const int4*>(x + (v1 ? r1 : 0) * d);
  float c[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i) c[n][i] = 0.f;
  // K in 64-column blocks: lane t4 loads 16-byte vectors at columns 8*t4 and 32 + 8*t4 of
  // rows g and g+8 (each load instruction covers 64 contiguous bytes per row).  The MMA's
  // k index is a fixed permutation of the block's columns, applied to x and Wg alike: the
  // logits are the same dot products, summed in another order.  KB blocks in flight.
  extern __shared__ __align__(16) uint8_t gate_wsm[];
  const int wrow = 4 * d + 16;  // bytes per staged expert row
  if (SW) {
    // eight loads in flight per thread before any split: the staging is bound by L2
    // latency (one dependent load -> split -> store per record was ~40 % of the kernel)
    constexpr int kSU = 8;
    const int per_row = d / 4, n_rec = E * per_row;
    for (int i0 = threadIdx.x; i0 < n_rec; i0 += kSU * blockDim.x) {
      float4 v[kSU];
#pragma unroll
      for (int u = 0; u < kSU; ++u) {
        const int i = i0 + u * blockDim.x;
        v[u] = i < n_rec ? __ldg(reinterpret_cast<const float4*>(wg) + i) : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < kSU; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i >= n_rec) break;
        const int e = i / per_row, c4 = i % per_row;
        uint4 rec;
        split_bf16x2(make_float2(v[u].x, v[u].y), rec.x, rec.z);
        split_bf16x2(make_float2(v[u].z, v[u].w), rec.y, rec.w);
        *reinterpret_cast<uint4*>(gate_wsm + e * wrow + c4 * 16) = rec;
      }
    }
    __syncthreads();
  }
  constexpr int KB = 4;
  const int dk = d / KS, kbeg = ks * dk, kend = kbeg + dk;
  for (int kb = kbeg; kb < kend; kb += 64 * KB) {
    int4 va[KB][2], vb[KB][2];
#pragma unroll
    for (int u = 0; u < KB; ++u) {
      const int col = kb + 64 * u + 8 * t4;
      const bool in = kb + 64 * u < kend;
      va[u][0] = (in && v0) ? __ldg(xr0 + col / 8) : make_int4(0, 0, 0, 0);
      va[u][1] = (in && v0) ? __ldg(xr0 + col / 8 + 4) : make_int4(0, 0, 0, 0);
      vb[u][0] = (in && v1) ? __ldg(xr1 + col / 8) : make_int4(0, 0, 0, 0);
      vb[u][1] = (in && v1) ? __ldg(xr1 + col / 8 + 4) : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < KB; ++u) {
      if (kb + 64 * u >= kend) break;
      const uint32_t* pa = reinterpret_cast<const uint32_t*>(&va[u][0]);  // 8 column pairs
      const uint32_t* pb = reinterpret_cast<const uint32_t*>(&vb[u][0]);
#pragma unroll
      for (int st = 0; st < 4; ++st) {
        const uint32_t a[4] = {pa[2 * st], pb[2 * st], pa[2 * st + 1], pb[2 * st + 1]};
        const int wcol = kb + 64 * u + (st < 2 ? 8 * t4 + 4 * st : 32 + 8 * t4 + 4 * (st - 2));
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          if (SW) {
            const uint4 r =
                *reinterpret_cast<const uint4*>(gate_wsm + (n * 8 + g) * wrow + (wcol / 4) * 16);
            mma_bf16_16816(c[n], a, r.x, r.y);
            mma_bf16_16816(c[n], a, r.z, r.w);
          } else {
            const float4 wv = __ldg(
                reinterpret_cast<const float4*>(wg + static_cast<int64_t>(n * 8 + g) * d + wcol));
            uint32_t h0, l0, h1, l1;
            split_bf16x2(make_float2(wv.x, wv.y), h0, l0);
            split_bf16x2(make_float2(wv.z, wv.w), h1, l1);
            mma_bf16_16816(c[n], a, h0, h1);
            mma_bf16_16816(c[n], a, l0, l1);
          }
        }
      }
    }
  }
  const int lr = tg * 16 + g;
  if (KS > 1) {
    if (ks > 0) {
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int e = n * 8 + 2 * t4;
        part[ks - 1][lr][e] = c[n][0];
        part[ks - 1][lr][e + 1] = c[n][1];
        part[ks - 1][lr + 8][e] = c[n][2];
        part[ks - 1][lr + 8][e + 1] = c[n][3];
      }
    }
    __syncthreads();
    if (ks == 0) {
#pragma unroll
      for (int q = 0; q < KS - 1; ++q)
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const int e = n * 8 + 2 * t4;
          c[n][0] = __fadd_rn(c[n][0], part[q][lr][e]);
          c[n][1] = __fadd_rn(c[n][1], part[q][lr][e + 1]);
          c[n][2] = __fadd_rn(c[n][2], part[q][lr + 8][e]);
          c[n][3] = __fadd_rn(c[n][3], part[q][lr + 8][e + 1]);
        }
    }
  }
  if (ks == 0) {
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int e = n * 8 + 2 * t4;
      const float b0 = bias ? bias[e] : 0.f, b1 = bias ? bias[e + 1] : 0.f;
      lg[lr][e] = bias ? __fadd_rn(c[n][0], b0) : c[n][0];
      lg[lr][e + 1] = bias ? __fadd_rn(c[n][1], b1) : c[n][1];
      lg[lr + 8][e] = bias ? __fadd_rn(c[n][2], b0) : c[n][2];
      lg[lr + 8][e + 1] = bias ? __fadd_rn(c[n][3], b1) : c[n][3];
    }
  }
  __syncthreads();
  const int64_t tt0 = static_cast<int64_t>(tile) * kGateTile;
  if (logits != nullptr) {
    for (int v = threadIdx.x; v < kGateTile * E; v += blockDim.x) {
      const int r = v / E, e = v % E;
      if (tt0 + r < T) logits[(tt0 + r) * E + e] = lg[r][e];
    }
  }
  gate_select_tile(&lg[0][0], kGateMaxE + 1, tile, T, E, k, s_idx, s_cnt, topk_idx, topk_w,
                   slot_rank, tile_counts);
  if (ws == nullptr) return;
  // fused K2: publish this tile's counts, and the last CTA scans / all-gathers them
  __syncthreads();
  if (threadIdx.x < E) atomicAdd(ws + 1 + threadIdx.x, s_cnt[threadIdx.x]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int ticket = atomicAdd(ws, 1);
    is_last = ticket == static_cast<int>(gridDim.x) - 1;
    if (is_last) __threadfence();
  }
  __syncthreads();
  if (!is_last) return;
  gate_route_tail(gridDim.x, E, tile_counts, tile_prefix, ws, peer_bases, table_off, flags_off,
                  rank, world, slot, epoch, local,
                  SW ? reinterpret_cast<int32_t*>(gate_wsm) : nullptr, SW ? E * wrow / 4 : 0);
}

// ------------------------------------------------------------------ gate backward on tcgen05
// dWg^T [d, 2E] = x^T [d, T] . G [T, 2E], G = the gate's logit gradient as a dense bf16
// matrix (row t: hi(dlogit) at column e, lo = bf16(dlogit - hi) at column E + e for each of
// its k experts, zeros elsewhere — ~16 mantissa bits of the fp32 gradient), split along T
// into `splits` groups so one wave of CTA pairs covers it; then
// dWg[e, c] = sum over splits, in order, of (C_s[c, e] + C_s[c, E + e]).  Replaces the
// SIMT gate_wgrad partials (their E x 512-column accumulators cannot co-reside with a GEMM
// CTA, so at E = 64 they stretch over the backward's last GEMMs).
constexpr int kGateN = 128;  // the gate GEMMs' N tile: hi and lo of up to 64 experts
static int gate_wgrad_splits(int64_t T, int d) {
  const int pair_tiles = d / 256;                      // M tiles of one split
  int s = (num_sms() / 2 + pair_tiles - 1) / pair_tiles;  // ~one wave of CTA pairs
  const int64_t kb = (T + 63) / 64;                    // at least 4 K blocks per split
  if (s > kb / 4) s = static_cast<int>(kb / 4);
  return s > 0 ? s : 1;
}

__global__ void __launch_bounds__(256)
    gate_wgrad_prep_kernel(const int32_t* __restrict__ topk_idx, const float* __restrict__ dlogit,
                           int64_t T, int64_t rows, int E, int k, int d, int splits, int64_t ks,
                           __nv_bfloat16* __restrict__ g, GemmGroup* __restrict__ groups) {
  // one thread per 8 columns (16 bytes) of G
  const int64_t n16 = rows * kGateN / 8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n16;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / (kGateN / 8);
    const int c0 = static_cast<int>(i % (kGateN / 8)) * 8;
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (t < T && c0 < 2 * E) {
      for (int j = 0; j < k; ++j) {
        const int e = topk_idx[t * k + j];
        const float w = dlogit[t * k + j];
        const float hi = __bfloat162float(__float2bfloat16_rn(w));
        if (e >= c0 && e < c0 + 8) v[e - c0] = hi;
        if (E + e >= c0 && E + e < c0 + 8) v[E + e - c0] = w - hi;
      }
    }
    __nv_bfloat162 o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = __floats2bfloat162_rn(v[2 * q], v[2 * q + 1]);
    reinterpret_cast<int4*>(g)[i] = *reinterpret_cast<const int4*>(o);
  }
  if (blockIdx.x == 0 && threadIdx.x < splits) {
    const int s = threadIdx.x;
    const int64_t k0 = s * ks;
    const int64_t kn = k0 >= rows ? 0 : (rows - k0 < ks ? rows - k0 : ks);
    const int mt = d / 128;
    groups[s] = GemmGroup{mt, s * mt, 0, static_cast<int>(k0), 0, static_cast<int>(k0),
                          static_cast<int>(kn / 64), 0, static_cast<int64_t>(s) * d * kGateN};
  }
}

__global__ void __launch_bounds__(256)
    gate_wgrad_tc_reduce_kernel(const float* __restrict__ c, int splits, int d, int E,
                                float* __restrict__ dwg) {
  // thread i: expert i % E of column i / E (neighbouring threads read one C row)
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<int64_t>(E) * d) return;
  const int e = static_cast<int>(i % E), col = static_cast<int>(i / E);
  float acc = 0.f;
  int s = 0;
  for (; s + 6 <= splits; s += 6) {  // 12 independent loads in flight, summed in order
    float v[6];
#pragma unroll
    for (int u = 0; u < 6; ++u) {
      const float* row = c + (static_cast<int64_t>(s + u) * d + col) * kGateN;
      v[u] = __fadd_rn(__ldcs(row + e), __ldcs(row + E + e));
    }
#pragma unroll
    for (int u = 0; u < 6; ++u) acc = __fadd_rn(acc, v[u]);
  }
  for (; s < splits; ++s) {
    const float* row = c + (static_cast<int64_t>(s) * d + col) * kGateN;
    acc = __fadd_rn(acc, __fadd_rn(row[e], row[E + e]));
  }
  dwg[static_cast<int64_t>(e) * d + col] = acc;
}

// ------------------------------------------------------------------ K1 on tcgen05
// The gate logits as one grouped-GEMM launch on the 5th-generation tensor cores: x [T, d]
// (K-major) times B = [hi(Wg); lo(Wg); 0] (kGateN x d bf16: the fp32 gate weights split
// into two bf16 halves, ~16 mantissa bits) into fp32 C [T, kGateN]; then
// logits[t, e] = (C[t, e] + C[t, E + e]) + bias[e].  The GEMM streams x through TMA at HBM
// rate (the mma.sync gate kernel above is bound by the latency of its register loads).

__global__ void __launch_bounds__(256)
    gate_gemm_prep_kernel(const float* __restrict__ wg, int E, int d,
                          __nv_bfloat16* __restrict__ b, GemmGroup* __restrict__ group,
                          int m_tiles) {
  const int64_t n = static_cast<int64_t>(kGateN) * d;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(i / d);
    const int64_t c = i % d;
    float v = 0.f;
    if (row < E) {
      v = wg[static_cast<int64_t>(row) * d + c];
    } else if (row < 2 * E) {
      const float w = wg[static_cast<int64_t>(row - E) * d + c];
      v = w - __bfloat162float(__float2bfloat16_rn(w));
    }
    b[i] = __float2bfloat16_rn(v);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    *group = GemmGroup{m_tiles, 0, 0, 0, 0, 0, d / 64, 0, 0};
}

__global__ void __launch_bounds__(kGateThreads)
    gate_select_kernel(const float* __restrict__ c, const float* __restrict__ bias, int64_t T,
                       int E, int k, int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
                       int32_t* __restrict__ slot_rank, int32_t* __restrict__ tile_counts,
                       int32_t* __restrict__ tile_prefix, int32_t* __restrict__ ws,
                       const uint64_t* __restrict__ peer_bases, int64_t table_off,
                       int64_t flags_off, int rank, int world, int slot, uint32_t epoch,
                       GateLocalTables local, int stage_ints) {
  __shared__ float lg[kGateTile][kGateMaxE + 1];
  __shared__ int32_t s_idx[kGateTile * kGateMaxK];
  __shared__ int32_t s_cnt[kGateMaxE];
  __shared__ int is_last;
  const int tile = blockIdx.x;
  const int64_t t0 = static_cast<int64_t>(tile) * kGateTile;
  for (int i = threadIdx.x; i < kGateTile * E; i += blockDim.x) {
    const int r = i / E, e = i % E;
    if (t0 + r < T) {
      const float* row = c + (t0 + r) * kGateN;
      const float v = __fadd_rn(__ldcs(row + e), __ldcs(row + E + e));
      lg[r][e] = bias != nullptr ? __fadd_rn(v, bias[e]) : v;
    }
  }
  __syncthreads();
  gate_select_tile(&lg[0][0], kGateMaxE + 1, tile, T, E, k, s_idx, s_cnt, topk_idx, topk_w,
                   slot_rank, tile_counts);
  if (ws == nullptr) return;
  // fused K2, as in gate_topk_mma_kernel: publish this tile's counts, the last CTA scans /
  // all-gathers them
  __syncthreads();
  if (threadIdx.x < E) atomicAdd(ws + 1 + threadIdx.x, s_cnt[threadIdx.x]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int ticket = atomicAdd(ws, 1);
    is_last = ticket == static_cast<int>(gridDim.x) - 1;
    if (is_last) __threadfence();
  }
  __syncthreads();
  if (!is_last) return;
  extern __shared__ __align__(16) int32_t sel_stage[];  // the tail's tile-count staging
  gate_route_tail(gridDim.x, E, tile_counts, tile_prefix, ws, peer_bases, table_off, flags_off,
                  rank, world, slot, epoch, local, stage_ints > 0 ? sel_stage : nullptr,
                  stage_ints);
}

__global__ void __launch_bounds__(kGateThreads)
    topk_from_logits_kernel(const float* __restrict__ logits, int64_t T, int E, int k,
                            int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
                            int32_t* __restrict__ slot_rank, int32_t* __restrict__ tile_counts) {
  __shared__ float lg[kGateTile][kGateMaxE + 1];
  __shared__ int32_t s_idx[kGateTile * kGateMaxK];
  __shared__ int32_t s_cnt[kGateMaxE];
  const int tile = blockIdx.x;
  const int64_t t0 = static_cast<int64_t>(tile) * kGateTile;
  for (int v = threadIdx.x; v < kGateTile * E; v += blockDim.x) {
    const int r = v / E, e = v % E;
    lg[r][e] = (t0 + r < T) ? logits[(t0 + r) * E + e] : 0.f;
  }
  __syncthreads();
  gate_select_tile(&lg[0][0], kGateMaxE + 1, tile, T, E, k, s_idx, s_cnt, topk_idx, topk_w,
                   slot_rank, tile_counts);
}

// ------------------------------------------------------------------ K2 scan + counts all-gather
// One CTA of 1024 threads: thread (chunk c, expert e) owns a contiguous run of tiles,
// so every load is independent (the old one-thread-per-expert loop was latency bound).
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads)
    route_scan_kernel(const int32_t* __restrict__ tile_counts, int n_tiles, int E,
                      int32_t* __restrict__ tile_prefix, const uint64_t* __restrict__ peer_bases,
                      int64_t table_off, int64_t flags_off, int rank, int world, int slot,
                      uint32_t epoch) {
  __shared__ int32_t chunk_sum[kScanThreads];
  const int chunks = kScanThreads / E;  // E <= 64 -> at least 16 chunks
  const int per = (n_tiles + chunks - 1) / chunks;
  const int e = threadIdx.x % E;
  const int c = threadIdx.x / E;
  const bool active = c < chunks;
  const int t0 = c * per;
  const int t1 = min(n_tiles, t0 + per);
  int32_t s = 0;
  if (active)
    for (int t = t0; t < t1; ++t) s += tile_counts[static_cast<int64_t>(t) * E + e];
  chunk_sum[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x < E) {  // exclusive scan over chunks, expert = threadIdx.x
    int32_t run = 0;
    for (int q = 0; q < chunks; ++q) {
      const int32_t v = chunk_sum[q * E + threadIdx.x];
      chunk_sum[q * E + threadIdx.x] = run;
      run += v;
    }
    for (int p = 0; p < world; ++p)
      reinterpret_cast<int32_t*>(peer_bases[p] + table_off)[rank * E + threadIdx.x] = run;
  }
  __syncthreads();
  if (active) {
    int32_t run = chunk_sum[threadIdx.x];
    for (int t = t0; t < t1; ++t) {
      tile_prefix[static_cast<int64_t>(t) * E + e] = run;
      run += tile_counts[static_cast<int64_t>(t) * E + e];
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) __threadfence_system();
    __syncwarp();
    world_barrier_warp(peer_bases, flags_off, rank, world, slot, epoch);
  }
}

// ------------------------------------------------------------------ row copy helpers
__device__ __forceinline__ void warp_copy_row(int4* __restrict__ dst, const int4* __restrict__ src,
                                              int n16) {
  const int lane = threadIdx.x & 31;
  int i = lane;
  for (; i + 96 < n16; i += 128) {
    int4 a = ld_nc_v4(src + i), b = ld_nc_v4(src + i + 32), c = ld_nc_v4(src + i + 64),
         d = ld_nc_v4(src + i + 96);
    st_v4(dst + i, a);
    st_v4(dst + i + 32, b);
    st_v4(dst + i + 64, c);
    st_v4(dst + i + 96, d);
  }
  for (; i < n16; i += 32) st_v4(dst + i, ld_nc_v4(src + i));
}

// Two rows at once: 8 x 16 B loads in flight per lane before the stores.
__device__ __forceinline__ void warp_copy_rows2(int4* __restrict__ d0, const int4* __restrict__ s0,
                                                int4* __restrict__ d1, const int4* __restrict__ s1,
                                                int n16) {
  const int lane = threadIdx.x & 31;
  int i = lane;
  for (; i + 96 < n16; i += 128) {
    int4 a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = ld_nc_v4(s0 + i + 32 * u);
#pragma unroll
    for (int u = 0; u < 4; ++u) b[u] = ld_nc_v4(s1 + i + 32 * u);
#pragma unroll
    for (int u = 0; u < 4; ++u) st_v4(d0 + i + 32 * u, a[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) st_v4(d1 + i + 32 * u, b[u]);
  }
  for (; i < n16; i += 32) {
    const int4 a = ld_nc_v4(s0 + i), b = ld_nc_v4(s1 + i);
    st_v4(d0 + i, a);
    st_v4(d1 + i, b);
  }
}

// The token-side kernels work in warp batches: the lanes first load / derive the index
// data of a batch of slots (or tokens) in parallel — one latency instead of one per item —
// then the warp streams the batch's rows with that data broadcast by shuffles.
constexpr int kBatch = 4;     // slots per warp batch (dispatch, dispatch_grad)
constexpr int kTokBatch = 4;  // tokens per warp batch (combine, combine_dx): 4 * K <= 32

__device__ __forceinline__ void warp_zero_rows(char* base, const int32_t* __restrict__ zero_rows,
                                               int n_zero, int64_t row_bytes, int warp_global,
                                               int nwarps) {
  const int lane = threadIdx.x & 31;
  const int n16 = static_cast<int>(row_bytes / 16);
  const int4 z = make_int4(0, 0, 0, 0);
  for (int r = 0; r < n_zero; ++r) {
    const int64_t row0 = zero_rows[2 * r];
    const int cnt = zero_rows[2 * r + 1];
    for (int i = warp_global; i < cnt; i += nwarps) {
      int4* dst = reinterpret_cast<int4*>(base + (row0 + i) * row_bytes);
      for (int c = lane; c < n16; c += 32) st_v4(dst + c, z);
    }
  }
}

// ------------------------------------------------------------------ K4 dispatch
__global__ void __launch_bounds__(256)
    dispatch_kernel(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ topk_idx,
                    const int32_t* __restrict__ slot_rank, const int32_t* __restrict__ tile_prefix,
                    int64_t T, int d_model, int E, int k, int world,
                    const int32_t* __restrict__ route_cum, const int32_t* __restrict__ recv_base,
                    int32_t* __restrict__ slot_dest, int32_t* __restrict__ slot_pos,
                    const uint64_t* __restrict__ peer_bases, int64_t recv_off,
                    const int32_t* __restrict__ zero_rows, int n_zero, int64_t flags_off, int rank,
                    int bar_slot, uint32_t epoch, uint32_t* grid_counter) {
  const int lane = threadIdx.x & 31;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int64_t row_bytes = static_cast<int64_t>(d_model) * 2;
  const int n16 = static_cast<int>(row_bytes / 16);
  const int64_t nslots = T * k;
  for (int64_t base = static_cast<int64_t>(warp_global) * kBatch; base < nslots;
       base += static_cast<int64_t>(nwarps) * kBatch) {
    int dst = 0, pos = 0;
    const int64_t sl = base + lane;
    if (lane < kBatch && sl < nslots) {
      const int64_t t = sl / k;
      const int e = topk_idx[sl];
      const int r = tile_prefix[(t / kGateTile) * E + e] + slot_rank[sl];
      const int32_t* cum = route_cum + e * (world + 1);
      int dd = 0;
      while (dd + 1 < world && cum[dd + 1] <= r) ++dd;
      dst = dd;
      pos = recv_base[e * world + dd] + (r - cum[dd]);
      slot_dest[sl] = dst;
      slot_pos[sl] = pos;
    }
    const int cnt = static_cast<int>(imin64(kBatch, nslots - base));
    auto out_row = [&](int i) {
      const int di = __shfl_sync(0xffffffffu, dst, i), pi = __shfl_sync(0xffffffffu, pos, i);
      return reinterpret_cast<int4*>(reinterpret_cast<char*>(peer_bases[di] + recv_off) +
                                     static_cast<int64_t>(pi) * row_bytes);
    };
    auto in_row = [&](int i) {
      return reinterpret_cast<const int4*>(x + ((base + i) / k) * d_model);
    };
    int i = 0;
    for (; i + 1 < cnt; i += 2) {
      int4* o0 = out_row(i);
      int4* o1 = out_row(i + 1);
      warp_copy_rows2(o0, in_row(i), o1, in_row(i + 1), n16);
    }
    if (i < cnt) {
      int4* o0 = out_row(i);
      warp_copy_row(o0, in_row(i), n16);
    }
  }
  warp_zero_rows(reinterpret_cast<char*>(peer_bases[rank] + recv_off), zero_rows, n_zero, row_bytes,
                 warp_global, nwarps);
  grid_done_then_barrier(grid_counter, peer_bases, flags_off, rank, world, bar_slot, epoch);
}

// ------------------------------------------------------------------ K6 combine
__device__ __forceinline__ void bf16x8_to_f32(const int4& v, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 p = __bfloat1622float2(h[i]);
    f[2 * i] = p.x;
    f[2 * i + 1] = p.y;
  }
}
__device__ __forceinline__ int4 f32_to_bf16x8(const float (&f)[8]) {
  int4 v;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return v;
}

// Dense all-reduce of a small replicated gradient over P2P (the gate's dWg): after a world
// barrier (every rank's partial is final), out = sum over ranks p = 0..world-1, in rank
// order, of rank p's fp32 partial at heap offset src_off — bit-identical on every rank.
// The loads go through L2 (__ldcg): the partials were released before the barrier.
__global__ void __launch_bounds__(256)
    sum_peers_kernel(const uint64_t* __restrict__ peer_bases, int world, int64_t src_off,
                     int64_t n4, float4* __restrict__ out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // launched behind the barrier (PDL)
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 a = __ldcg(reinterpret_cast<const float4*>(peer_bases[0] + src_off) + i);
#pragma unroll 4
    for (int p = 1; p < world; ++p) {  // independent loads: the unrolled ones are in flight
      const float4 v = __ldcg(reinterpret_cast<const float4*>(peer_bases[p] + src_off) + i);
      a.x = __fadd_rn(a.x, v.x);
      a.y = __fadd_rn(a.y, v.y);
      a.z = __fadd_rn(a.z, v.z);
      a.w = __fadd_rn(a.w, v.w);
    }
    out[i] = a;
  }
}

// Row chunks: a warp walks a row in blocks of 128 x 16 B; a lane holds 4 of them, and the
// loads of all K rows of a token are issued before any use (one memory latency per token).
constexpr int kRowBlk = 128;

template <int K>
__global__ void __launch_bounds__(256)
    combine_kernel(const int32_t* __restrict__ slot_dest, const int32_t* __restrict__ slot_pos,
                   const float* __restrict__ topk_w, int64_t T, int d_model,
                   const uint64_t* __restrict__ peer_bases, int64_t y_off,
                   __nv_bfloat16* __restrict__ y_out, __nv_bfloat16* __restrict__ y_slots) {
  // launched with PDL (launch_pdl): scheduled during the producing GEMM tail
  asm volatile("griddepcontrol.wait;" ::: "memory");
  constexpr int TB = kTokBatch;  // tokens per warp batch (TB * K <= 32)
  const int lane = threadIdx.x & 31;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int64_t row_bytes = static_cast<int64_t>(d_model) * 2;
  const int n16 = static_cast<int>(row_bytes / 16);
  for (int64_t base = static_cast<int64_t>(warp_global) * TB; base < T;
       base += static_cast<int64_t>(nwarps) * TB) {
    const int64_t sl = base * K + lane;
    int sd = 0, sp = 0;
    float sw = 0.f;
    if (lane < TB * K && sl < T * K) {
      sd = slot_dest[sl];
      sp = slot_pos[sl];
      sw = topk_w[sl];
    }
    const int cnt = static_cast<int>(imin64(TB, T - base));
    for (int i = 0; i < cnt; ++i) {
      const int4* rows[K];
      float w[K];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const int src = i * K + j;
        rows[j] = reinterpret_cast<const int4*>(
            reinterpret_cast<const char*>(peer_bases[__shfl_sync(0xffffffffu, sd, src)] + y_off) +
            static_cast<int64_t>(__shfl_sync(0xffffffffu, sp, src)) * row_bytes);
        w[j] = __shfl_sync(0xffffffffu, sw, src);
      }
      int4* out = reinterpret_cast<int4*>(y_out + (base + i) * d_model);
      // the K gathered rows, kept token-local for dispatch_grad's <dy, Y> (slot order)
      int4* keep = y_slots == nullptr ? nullptr
                                      : reinterpret_cast<int4*>(y_slots + (base + i) * K * d_model);
      for (int c0 = 0; c0 < n16; c0 += kRowBlk) {
        int4 v[K][4];
#pragma unroll
        for (int j = 0; j < K; ++j)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = c0 + lane + 32 * u;
            v[j][u] = c < n16 ? ld_nc_v4(rows[j] + c) : make_int4(0, 0, 0, 0);
          }
        if (keep != nullptr) {
#pragma unroll
          for (int j = 0; j < K; ++j)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int c = c0 + lane + 32 * u;
              if (c < n16) st_v4(keep + j * n16 + c, v[j][u]);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + lane + 32 * u;
          if (c >= n16) break;
          float acc[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = 0.f;
#pragma unroll
          for (int j = 0; j < K; ++j) {
            float f[8];
            bf16x8_to_f32(v[j][u], f);
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], __fmul_rn(w[j], f[q]));
          }
          out[c] = f32_to_bf16x8(acc);
        }
      }
    }
  }
}

// ------------------------------------------------------------------ K7 token-side backward
__global__ void __launch_bounds__(256)
    dispatch_grad_kernel(const __nv_bfloat16* __restrict__ dy, const int32_t* __restrict__ slot_dest,
                         const int32_t* __restrict__ slot_pos, const float* __restrict__ topk_w,
                         int64_t T, int d_model, int k, const uint64_t* __restrict__ peer_bases,
                         int64_t y_off, const __nv_bfloat16* __restrict__ y_slots,
                         int64_t dy_recv_off, float* __restrict__ slot_grad,
                         float* __restrict__ dlogit_out, const int32_t* __restrict__ zero_rows, int n_zero, int64_t flags_off,
                         int rank, int world, int bar_slot, uint32_t epoch,
                         uint32_t* grid_counter) {
  const int lane = threadIdx.x & 31;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int64_t row_bytes = static_cast<int64_t>(d_model) * 2;
  const int n16 = static_cast<int>(row_bytes / 16);
  const int64_t nslots = T * k;
  for (int64_t base = static_cast<int64_t>(warp_global) * kBatch; base < nslots;
       base += static_cast<int64_t>(nwarps) * kBatch) {
    const int64_t sl = base + lane;
    int sd = 0, sp = 0;
    float sw = 0.f;
    if (lane < kBatch && sl < nslots) {
      sd = slot_dest[sl];
      sp = slot_pos[sl];
      sw = topk_w[sl];
    }
    float my_dot = 0.f;  // lane i keeps item i's <dy, Y>
    const int cnt = static_cast<int>(imin64(kBatch, nslots - base));
    for (int i = 0; i < cnt; ++i) {
      const int64_t t = (base + i) / k;
      const int dst = __shfl_sync(0xffffffffu, sd, i);
      const int64_t pos = __shfl_sync(0xffffffffu, sp, i);
      const float w = __shfl_sync(0xffffffffu, sw, i);
      const int4* yrow =
          y_slots != nullptr
              ? reinterpret_cast<const int4*>(y_slots + (base + i) * d_model)
              : reinterpret_cast<const int4*>(
                    reinterpret_cast<const char*>(peer_bases[dst] + y_off) + pos * row_bytes);
      const int4* grow = reinterpret_cast<const int4*>(dy + t * d_model);
      int4* out = reinterpret_cast<int4*>(reinterpret_cast<char*>(peer_bases[dst] + dy_recv_off) +
                                          pos * row_bytes);
      float dot = 0.f;
      for (int c0 = 0; c0 < n16; c0 += kRowBlk) {
        int4 vy[4], vg[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + lane + 32 * u;
          // slot_grad null: the dots are left to combine_dx (off the critical path)
          vy[u] = c < n16 && slot_grad != nullptr ? ld_nc_v4(yrow + c) : make_int4(0, 0, 0, 0);
          vg[u] = c < n16 ? ld_nc_v4(grow + c) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + lane + 32 * u;
          if (c >= n16) break;
          float fy[8], fg[8], o[8];
          bf16x8_to_f32(vy[u], fy);
          bf16x8_to_f32(vg[u], fg);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            dot = fmaf(fg[q], fy[q], dot);
            o[q] = __fmul_rn(w, fg[q]);
          }
          st_v4(out + c, f32_to_bf16x8(o));
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
      if (lane == i) my_dot = dot;
    }
    if (lane < cnt && slot_grad != nullptr) slot_grad[sl] = my_dot;
    if (dlogit_out != nullptr) {
      // whole tokens per batch (host guarantees kBatch % k == 0): the gate's dlogit here,
      // in combine_dx's arithmetic, so the gate backward need not wait for the dX combine
      const int first = (lane / k) * k;
      float sg = 0.f;
      for (int j = 0; j < k; ++j)
        sg = fmaf(__shfl_sync(0xffffffffu, sw, (first + j) & 31),
                  __shfl_sync(0xffffffffu, my_dot, (first + j) & 31), sg);
      if (lane < cnt) dlogit_out[sl] = sw * (my_dot - sg);
    }
  }
  warp_zero_rows(reinterpret_cast<char*>(peer_bases[rank] + dy_recv_off), zero_rows, n_zero,
                 row_bytes, warp_global, nwarps);
  grid_done_then_barrier(grid_counter, peer_bases, flags_off, rank, world, bar_slot, epoch);
}

template <int K>
__global__ void __launch_bounds__(256)
    combine_dx_kernel(const int32_t* __restrict__ slot_dest, const int32_t* __restrict__ slot_pos,
                      const int32_t* __restrict__ topk_idx, const float* __restrict__ topk_w,
                      const float* __restrict__ slot_grad, const float* __restrict__ wg, int64_t T,
                      int d_model, const uint64_t* __restrict__ peer_bases, int64_t dxe_off,
                      float* __restrict__ dlogit_out, __nv_bfloat16* __restrict__ dx_out,
                      const __nv_bfloat16* __restrict__ dy, int64_t y_off,
                      const __nv_bfloat16* __restrict__ y_slots, float* __restrict__ slot_grad_out) {
  // launched with PDL (launch_pdl): scheduled during the producing GEMM tail
  asm volatile("griddepcontrol.wait;" ::: "memory");
  constexpr int TB = kTokBatch;
  const int lane = threadIdx.x & 31;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int64_t row_bytes = static_cast<int64_t>(d_model) * 2;
  const int n16 = static_cast<int>(row_bytes / 16);
  for (int64_t base = static_cast<int64_t>(warp_global) * TB; base < T;
       base += static_cast<int64_t>(nwarps) * TB) {
    const int64_t sl = base * K + lane;
    const bool own = lane < TB * K && sl < T * K;
    int sd = 0, sp = 0, se = 0;
    float sw = 0.f, sgr = 0.f;
    if (own) {
      sd = slot_dest[sl];
      sp = slot_pos[sl];
      se = topk_idx[sl];
      sw = topk_w[sl];
      if (dy == nullptr) sgr = slot_grad[sl];
    }
    if (dy != nullptr) {
      // <dy, Y> of every slot of the batch, here instead of in dispatch_grad (which then
      // only scatters w * dy on the critical path): the same per-lane fma order and
      // butterfly as dispatch_grad, so the values are bit-identical
      const int nsl = static_cast<int>(imin64(TB, T - base)) * K;
      for (int i = 0; i < nsl; ++i) {
        const int dst = __shfl_sync(0xffffffffu, sd, i);
        const int64_t pos = __shfl_sync(0xffffffffu, sp, i);
        const int4* yrow =
            y_slots != nullptr
                ? reinterpret_cast<const int4*>(y_slots + (base * K + i) * d_model)
                : reinterpret_cast<const int4*>(
                      reinterpret_cast<const char*>(peer_bases[dst] + y_off) + pos * row_bytes);
        const int4* grow = reinterpret_cast<const int4*>(dy + (base + i / K) * d_model);
        float dot = 0.f;
        for (int c0 = 0; c0 < n16; c0 += kRowBlk) {
          int4 vy[4], vg[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = c0 + lane + 32 * u;
            vy[u] = c < n16 ? ld_nc_v4(yrow + c) : make_int4(0, 0, 0, 0);
            vg[u] = c < n16 ? ld_nc_v4(grow + c) : make_int4(0, 0, 0, 0);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = c0 + lane + 32 * u;
            if (c >= n16) break;
            float fy[8], fg[8];
            bf16x8_to_f32(vy[u], fy);
            bf16x8_to_f32(vg[u], fg);
#pragma unroll
            for (int q = 0; q < 8; ++q) dot = fmaf(fg[q], fy[q], dot);
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
        if (lane == i) sgr = dot;
      }
      if (own && slot_grad_out != nullptr) slot_grad_out[sl] = sgr;
    }
    // dlogit of this lane's slot: w_j (g_j - sum_i w_i g_i), the sum over its token's slots
    const int first = (lane / K) * K;
    float sg = 0.f;
#pragma unroll
    for (int j = 0; j < K; ++j)
      sg = fmaf(__shfl_sync(0xffffffffu, sw, (first + j) & 31),
                __shfl_sync(0xffffffffu, sgr, (first + j) & 31), sg);
    const float dlv = sw * (sgr - sg);
    if (own && dlogit_out != nullptr) dlogit_out[sl] = dlv;
    const int cnt = static_cast<int>(imin64(TB, T - base));
    for (int i = 0; i < cnt; ++i) {
      const int4* rows[K];
      const float* wrow[K];
      float dl[K];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const int src = i * K + j;
        dl[j] = __shfl_sync(0xffffffffu, dlv, src);
        rows[j] = reinterpret_cast<const int4*>(
            reinterpret_cast<const char*>(peer_bases[__shfl_sync(0xffffffffu, sd, src)] +
                                          dxe_off) +
            static_cast<int64_t>(__shfl_sync(0xffffffffu, sp, src)) * row_bytes);
        wrow[j] = wg + static_cast<int64_t>(__shfl_sync(0xffffffffu, se, src)) * d_model;
      }
      int4* out = reinterpret_cast<int4*>(dx_out + (base + i) * d_model);
      for (int c0 = 0; c0 < n16; c0 += kRowBlk) {
        int4 v[K][4];
#pragma unroll
        for (int j = 0; j < K; ++j)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = c0 + lane + 32 * u;
            v[j][u] = c < n16 ? ld_nc_v4(rows[j] + c) : make_int4(0, 0, 0, 0);
          }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + lane + 32 * u;
          if (c >= n16) break;
          float acc[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = 0.f;
#pragma unroll
          for (int j = 0; j < K; ++j) {
            float f[8];
            bf16x8_to_f32(v[j][u], f);
            const float4 w0 = __ldg(reinterpret_cast<const float4*>(wrow[j] + c * 8));
            const float4 w1 = __ldg(reinterpret_cast<const float4*>(wrow[j] + c * 8 + 4));
            const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] += f[q] + dl[j] * wv[q];
          }
          out[c] = f32_to_bf16x8(acc);
        }
      }
    }
  }
}

// Streaming partials: a CTA owns kWgCols columns of dWg for a contiguous run of tokens;
// each thread owns 4 columns and keeps their E accumulators in shared memory (only it
// touches them: no synchronisation, conflict-free float4 accesses).  x is read once,
// kWgU tokens of 8-byte loads in flight per thread; the expert of a slot is uniform
// across the CTA, so the update is one smem read-modify-write per slot and thread.
constexpr int kWgCols = 512;
constexpr int kWgThreads = kWgCols / 4;
constexpr int kWgU = 8;
__global__ void __launch_bounds__(kWgThreads)
    gate_wgrad_partial_kernel(const __nv_bfloat16* __restrict__ x,
                              const int32_t* __restrict__ topk_idx,
                              const float* __restrict__ dlogit, int64_t T, int d_model, int E,
                              int k, int64_t tok_per_cta, float* __restrict__ workspace) {
  extern __shared__ __align__(16) float4 s_acc[];  // [E][kWgThreads]
  __shared__ int32_t s_e[FSSDP_WG_TILE * kGateMaxK];
  __shared__ float s_w[FSSDP_WG_TILE * kGateMaxK];
  const int c = blockIdx.x * kWgCols + threadIdx.x * 4;
  const bool col_ok = c < d_model;
  const int64_t t_begin = static_cast<int64_t>(blockIdx.y) * tok_per_cta;
  const int ntok = static_cast<int>(imin64(T, t_begin + tok_per_cta) - t_begin);
  // the run's slots (expert, dlogit) once into smem: broadcast reads in the loop below
  for (int i = threadIdx.x; i < ntok * k; i += blockDim.x) {
    s_e[i] = topk_idx[t_begin * k + i];
    s_w[i] = dlogit[t_begin * k + i];
  }
  float4* my = s_acc + threadIdx.x;
  for (int e = 0; e < E; ++e) my[e * kWgThreads] = make_float4(0.f, 0.f, 0.f, 0.f);
  const __nv_bfloat16* xc = x + t_begin * d_model + c;
  auto load = [&](int t0, uint2 (&v)[kWgU]) {
#pragma unroll
    for (int u = 0; u < kWgU; ++u)
      v[u] = (col_ok && t0 + u < ntok)
                 ? __ldg(reinterpret_cast<const uint2*>(xc + static_cast<int64_t>(t0 + u) * d_model))
                 : make_uint2(0u, 0u);
  };
  uint2 cur[kWgU], nxt[kWgU];
  load(0, cur);
  __syncthreads();
  for (int t0 = 0; t0 < ntok; t0 += kWgU) {
    load(t0 + kWgU, nxt);  // next group in flight while this one is accumulated
#pragma unroll
    for (int u = 0; u < kWgU; ++u) {
      if (t0 + u >= ntok) break;
      const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&cur[u].x));
      const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&cur[u].y));
      for (int j = 0; j < k; ++j) {
        const int sl = (t0 + u) * k + j;
        const int e = s_e[sl];
        const float w = s_w[sl];
        float4 a = my[e * kWgThreads];
        a.x = fmaf(w, lo.x, a.x);
        a.y = fmaf(w, lo.y, a.y);
        a.z = fmaf(w, hi.x, a.z);
        a.w = fmaf(w, hi.y, a.w);
        my[e * kWgThreads] = a;
      }
    }
#pragma unroll
    for (int u = 0; u < kWgU; ++u) cur[u] = nxt[u];
  }
  if (!col_ok) return;
  for (int e = 0; e < E; ++e)
    *reinterpret_cast<float4*>(workspace + (static_cast<int64_t>(blockIdx.y) * E + e) * d_model +
                               c) = my[e * kWgThreads];
}

// dWg = sum over runs in run order: a CTA owns 32 consecutive outputs (one per lane); its
// 8 warps sum contiguous eighths of the runs (8 loads in flight each), then warp 0 adds the
// eight partial sums in warp order.  Deterministic for a given T.
__global__ void __launch_bounds__(256)
    gate_wgrad_reduce_kernel(const float* __restrict__ workspace, int n_tiles, int d_model, int E,
                             float* __restrict__ dwg) {
  __shared__ float part[8][32];
  const int64_t n = static_cast<int64_t>(E) * d_model;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * 32 + lane;
  const int per = (n_tiles + 7) / 8;
  const int p0 = warp * per, p1 = min(n_tiles, p0 + per);
  float s = 0.f;
  if (i < n) {
    int p = p0;
    for (; p + 8 <= p1; p += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = workspace[(p + u) * n + i];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; p < p1; ++p) s += workspace[p * n + i];
  }
  part[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && i < n) {
    float t = part[0][lane];
#pragma unroll
    for (int w = 1; w < 8; ++w) t += part[w][lane];
    dwg[i] = t;
  }
}

// ------------------------------------------------------------------ K3 SpAG / K8 SpRS
// Chunk size per CTA is chosen by the launcher so every launch spreads over ~4 CTAs per
// SM whatever the expert size (small experts are otherwise latency/parallelism bound).
static int64_t coll_chunk_bytes(int64_t total_bytes, int sms) {
  int64_t c = total_bytes / (4 * static_cast<int64_t>(sms));
  c = (c + 4095) / 4096 * 4096;
  if (c < 8192) c = 8192;
  if (c > 256 * 1024) c = 256 * 1024;
  return c;
}

__global__ void __launch_bounds__(256)
    spag_kernel(const uint64_t* __restrict__ peer_bases, int rank, int64_t param_off,
                int64_t slot_bytes, const int32_t* __restrict__ copies, int64_t chunk) {
  const int job = blockIdx.y;
  const int src_rank = copies[3 * job];
  const int64_t src_slot = copies[3 * job + 1];
  const int64_t dst_slot = copies[3 * job + 2];
  const int64_t begin = static_cast<int64_t>(blockIdx.x) * chunk;
  if (begin >= slot_bytes) return;
  const int64_t bytes = imin64(chunk, slot_bytes - begin);
  const int4* src = reinterpret_cast<const int4*>(
      reinterpret_cast<const char*>(peer_bases[src_rank] + param_off) + src_slot * slot_bytes +
      begin);
  int4* dst = reinterpret_cast<int4*>(reinterpret_cast<char*>(peer_bases[rank] + param_off) +
                                      dst_slot * slot_bytes + begin);
  const int n16 = static_cast<int>(bytes / 16);
  constexpr int U = 8;
  int i = threadIdx.x;
  for (; i + (U - 1) * 256 < n16; i += U * 256) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_nc_v4(src + i + u * 256);
#pragma unroll
    for (int u = 0; u < U; ++u) st_v4(dst + i + u * 256, v[u]);
  }
  for (; i < n16; i += 256) st_v4(dst + i, ld_nc_v4(src + i));
}

// TMA-staged SpAG: one warp per CTA, its elected lane streams the CTA's chunk of a replica
// copy through a kTmaRing-deep ring of kTmaSub-byte smem buffers: bulk load from the owner's
// (peer) HBM, bulk store to the local replica slot.  Few SM resources per byte in flight.
constexpr int kTmaSub = 8 * 1024;
constexpr int kTmaRing = 4;  // 32 KB of static smem per CTA -> several CTAs per SM
__global__ void __launch_bounds__(32)
    spag_tma_kernel(const uint64_t* __restrict__ peer_bases, int rank, int64_t src_off,
                    int64_t dst_off, int64_t slot_bytes, int64_t copy_bytes,
                    const int32_t* __restrict__ copies, int64_t chunk) {
  __shared__ __align__(128) uint8_t ring[kTmaRing][kTmaSub];
  __shared__ __align__(8) uint64_t bar[kTmaRing];
  const int job = blockIdx.y;
  const int64_t begin = static_cast<int64_t>(blockIdx.x) * chunk;
  if (begin >= copy_bytes || threadIdx.x != 0) return;
  const int src_rank = copies[3 * job];
  const int64_t src_slot = copies[3 * job + 1];
  const int64_t dst_slot = copies[3 * job + 2];
  const int64_t bytes = imin64(chunk, copy_bytes - begin);
  const char* src = reinterpret_cast<const char*>(peer_bases[src_rank] + src_off) +
                    src_slot * slot_bytes + begin;
  char* dst = reinterpret_cast<char*>(peer_bases[rank] + dst_off) + dst_slot * slot_bytes + begin;
  for (int i = 0; i < kTmaRing; ++i) mbar_init(&bar[i], 1);
  fence_barrier_init();
  const int nsub = static_cast<int>((bytes + kTmaSub - 1) / kTmaSub);
  auto issue = [&](int s) {
    const int slot = s % kTmaRing;
    const uint32_t n = static_cast<uint32_t>(imin64(kTmaSub, bytes - int64_t(s) * kTmaSub));
    mbar_arrive_expect_tx(&bar[slot], n);
    bulk_load_g2s(ring[slot], src + int64_t(s) * kTmaSub, n, &bar[slot]);
  };
  for (int s = 0; s < kTmaRing && s < nsub; ++s) issue(s);
  uint32_t phase = 0;  // bit per ring slot
  for (int s = 0; s < nsub; ++s) {
    const int slot = s % kTmaRing;
    mbar_wait(&bar[slot], (phase >> slot) & 1u);
    phase ^= 1u << slot;
    const uint32_t n = static_cast<uint32_t>(imin64(kTmaSub, bytes - int64_t(s) * kTmaSub));
    bulk_store_s2g(dst + int64_t(s) * kTmaSub, ring[slot], n);
    bulk_commit();
    if (s + kTmaRing < nsub) {
      bulk_wait_read<0>();  // this slot's store has read the buffer: reuse it
      issue(s + kTmaRing);
    }
  }
  bulk_wait<0>();
}

// Gradient elements in 16-byte vectors: 4 fp32, or 8 bf16 summed in fp32 (one rounding
// after the last holder) — grad_dtype of the layer.
template <bool BF16>
struct GradVec {
  static constexpr int kElems = BF16 ? 8 : 4;
  float v[kElems];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < kElems; ++i) v[i] = 0.f;
  }
  __device__ __forceinline__ void add(const int4 raw) {  // v += raw, element by element
    const uint32_t w[4] = {static_cast<uint32_t>(raw.x), static_cast<uint32_t>(raw.y),
                           static_cast<uint32_t>(raw.z), static_cast<uint32_t>(raw.w)};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (BF16) {
        v[2 * i] = __fadd_rn(v[2 * i], __uint_as_float(w[i] << 16));
        v[2 * i + 1] = __fadd_rn(v[2 * i + 1], __uint_as_float(w[i] & 0xffff0000u));
      } else {
        v[i] = __fadd_rn(v[i], __uint_as_float(w[i]));
      }
    }
  }
  __device__ __forceinline__ int4 pack() const {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (BF16) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
        w[i] = *reinterpret_cast<const uint32_t*>(&h);
      } else {
        w[i] = __float_as_uint(v[i]);
      }
    }
    return make_int4(static_cast<int>(w[0]), static_cast<int>(w[1]), static_cast<int>(w[2]),
                     static_cast<int>(w[3]));
  }
};

// Owner-side SpRS reduction (the holders' partials were pushed into the local staging
// slots by their wgrad epilogues): local HBM reads only.  Persistent over (chunk, job)
// units so the launcher can bound the SMs it occupies beside the backward GEMMs.
// slot_bytes / chunk in bytes; BF16: bf16 gradient slots (GradVec).
template <bool BF16>
__global__ void __launch_bounds__(256)
    sprs_kernel(const uint64_t* __restrict__ peer_bases, int rank, int64_t grad_off,
                int64_t stage_off, int64_t slot_bytes, const int32_t* __restrict__ jobs,
                const int32_t* __restrict__ srcs, int64_t chunk, int n_chunks, int n_units) {
  __shared__ const int4* s_src[kMaxWorld];
  const int64_t slot_vecs = slot_bytes / 16;
  const int64_t chunk_vecs = chunk / 16;
  for (int unit = blockIdx.x; unit < n_units; unit += gridDim.x) {
    const int job = unit / n_chunks;
    const int64_t dst_slot = jobs[3 * job];
    const int src_begin = jobs[3 * job + 1];
    const int src_count = jobs[3 * job + 2];
    const int64_t begin = static_cast<int64_t>(unit % n_chunks) * chunk_vecs;
    __syncthreads();  // previous unit's readers of s_src are done
    if (threadIdx.x < src_count) {  // own grads slot, or the staging slot a holder pushed
      const int r = srcs[2 * (src_begin + threadIdx.x)];
      const int64_t idx = srcs[2 * (src_begin + threadIdx.x) + 1];
      const int64_t off = r == rank ? grad_off : stage_off;
      s_src[threadIdx.x] =
          reinterpret_cast<const int4*>(peer_bases[rank] + off) + idx * slot_vecs + begin;
    }
    __syncthreads();
    const int n4 = static_cast<int>(imin64(chunk_vecs, slot_vecs - begin));
    int4* dst = reinterpret_cast<int4*>(peer_bases[rank] + grad_off) + dst_slot * slot_vecs + begin;
    // U vectors per thread per pass: U * src_count 128-bit loads in flight; each element is
    // still summed over the holders in ascending-rank order (bit-exact vs the oracle).
    constexpr int U = 4;
    for (int i0 = threadIdx.x; i0 < n4; i0 += U * 256) {
      GradVec<BF16> acc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u].zero();
      for (int q = 0; q < src_count; ++q) {
        int4 raw[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          raw[u] = (i0 + u * 256 < n4) ? ld_nc_v4(s_src[q] + i0 + u * 256) : make_int4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u].add(raw[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u * 256 < n4) dst[i0 + u * 256] = acc[u].pack();
    }
  }
}

// SpRS by pull (the standalone SparseReduceScatter): each holder's partial stays in its
// own grads slot; the owner streams every source of a chunk through a TMA ring — remote
// partials straight from the holders' HBM over NVLink, its own from local HBM — and sums
// them in listed (ascending-rank) order into its grads slot.  One pass, no staging round
// trip.  Warp 0 (one lane) produces, kPullWarps warps consume: each consumer thread owns 4
// float4 of every kPullSub-byte sub-chunk, so a sub-chunk's sum stays in registers while
// its sources arrive one ring stage each.
constexpr int kPullSub = 8 * 1024;
constexpr int kPullRing = 8;   // 64 KB of dynamic smem per CTA: 3 CTAs per SM
constexpr int kPullWarps = 4;  // 128 consumer threads x 4 vectors = one sub-chunk
template <bool BF16>
__global__ void __launch_bounds__(32 * (kPullWarps + 1))
    sprs_pull_kernel(const uint64_t* __restrict__ peer_bases, int rank, int64_t grad_off,
                     int64_t slot_bytes, const int32_t* __restrict__ jobs,
                     const int32_t* __restrict__ srcs, int64_t chunk, int n_chunks, int n_units) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[kPullRing], empty[kPullRing];
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPullRing; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kPullWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    if (threadIdx.x != 0) return;
    uint32_t it = 0;
    for (int unit = blockIdx.x; unit < n_units; unit += gridDim.x) {
      const int job = unit / n_chunks;
      const int src_begin = jobs[3 * job + 1], src_count = jobs[3 * job + 2];
      const int64_t begin = static_cast<int64_t>(unit % n_chunks) * chunk;
      const int64_t bytes = imin64(chunk, slot_bytes - begin);
      for (int64_t c = 0; c < bytes; c += kPullSub) {
        const uint32_t n = static_cast<uint32_t>(imin64(kPullSub, bytes - c));
        for (int q = 0; q < src_count; ++q, ++it) {
          const int r = srcs[2 * (src_begin + q)];
          const int64_t idx = srcs[2 * (src_begin + q) + 1];
          const char* src = reinterpret_cast<const char*>(peer_bases[r] + grad_off) +
                            idx * slot_bytes + begin + c;
          const uint32_t st = it % kPullRing;
          if (it >= kPullRing) mbar_wait(&empty[st], ((it / kPullRing) - 1) & 1u);
          mbar_arrive_expect_tx(&full[st], n);
          bulk_load_g2s(ring + st * kPullSub, src, n, &full[st]);
        }
      }
    }
    return;
  }
  const int t = threadIdx.x - 32;
  const int lane = threadIdx.x & 31;
  uint32_t it = 0;
  for (int unit = blockIdx.x; unit < n_units; unit += gridDim.x) {
    const int job = unit / n_chunks;
    const int64_t dst_slot = jobs[3 * job];
    const int src_count = jobs[3 * job + 2];
    const int64_t begin = static_cast<int64_t>(unit % n_chunks) * chunk;
    const int64_t bytes = imin64(chunk, slot_bytes - begin);
    char* dst = reinterpret_cast<char*>(peer_bases[rank] + grad_off) + dst_slot * slot_bytes + begin;
    for (int64_t c = 0; c < bytes; c += kPullSub) {
      const int n16 = static_cast<int>(imin64(kPullSub, bytes - c) / 16);
      GradVec<BF16> acc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u].zero();
      for (int q = 0; q < src_count; ++q, ++it) {
        const uint32_t st = it % kPullRing;
        mbar_wait(&full[st], (it / kPullRing) & 1u);
        const int4* buf = reinterpret_cast<const int4*>(ring + st * kPullSub);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = t + u * 32 * kPullWarps;
          if (i < n16) acc[u].add(buf[i]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
      int4* out = reinterpret_cast<int4*>(dst + c);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = t + u * 32 * kPullWarps;
        if (i < n16) out[i] = acc[u].pack();
      }
    }
  }
}

// ------------------------------------------------------------------ plan-boundary transfers
// Small host<->device transfers on the planning critical path done by the SMs through
// mapped pinned memory: a copy-engine transfer would queue behind bulk H2D/D2H traffic of
// the caller (e.g. the next step's inputs, the previous step's outputs).
__global__ void __launch_bounds__(256)
    push_host_kernel(const int4* __restrict__ src, int4* dst_host, int n16, uint32_t* flag_host,
                     uint32_t flag_value) {
  for (int i = threadIdx.x; i < n16; i += blockDim.x) dst_host[i] = src[i];
  __syncthreads();
  if (threadIdx.x == 0 && flag_host != nullptr) {
    __threadfence_system();
    st_release_sys(flag_host, flag_value);
  }
}

// the two-kernel gate path's counts push (the fused gate does it in its tail)
__global__ void __launch_bounds__(256)
    push_counts_kernel(const uint64_t* __restrict__ peer_bases, int rank, int64_t table_off,
                       GateLocalTables local) {
  const int4* src = reinterpret_cast<const int4*>(peer_bases[rank] + table_off);
  for (int i = threadIdx.x; i < local.host_n16; i += blockDim.x) local.host_counts[i] = src[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(local.host_flag, local.host_flag_value);
  }
}

__global__ void __launch_bounds__(256)
    pull_host_kernel(const int4* src_host, int4* __restrict__ dst, int n16) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x)
    dst[i] = src_host[i];
}

// ------------------------------------------------------------------ launchers
static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static int launch_check() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return kErrCuda;
  }
  return kOk;
}

// end of an entry point's launches: closes an armed timing window (fssdp_timing_arm)
static int launch_status() {
  timing_end();
  return launch_check();
}

// K-templated launch for the token gathers (K = top-k <= kGateMaxK = 8)
// Programmatic dependent launch (FSSDP_TOKEN_PDL, default on; "0" disables): the kernel may
// be scheduled while the previous kernel in the stream drains (the grouped GEMM triggers
// launch_dependents after its mainloop); every kernel launched this way executes
// griddepcontrol.wait before its first global-memory access, so ordering is unchanged.
template <typename... P, typename... A>
static void launch_pdl(void (*kern)(P...), unsigned grid, unsigned block, cudaStream_t stream,
                       A&&... args) {
  static const bool pdl = [] {
    const char* v = getenv("FSSDP_TOKEN_PDL");
    return v == nullptr || v[0] != '0';
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<P>(args)...);
}

#define FSSDP_DISPATCH_K(k, KERNEL, GRID, STREAM, ...)                    \
  switch (k) {                                                             \
    case 1: launch_pdl(KERNEL<1>, GRID, 256, STREAM, __VA_ARGS__); break;  \
    case 2: launch_pdl(KERNEL<2>, GRID, 256, STREAM, __VA_ARGS__); break;  \
    case 3: launch_pdl(KERNEL<3>, GRID, 256, STREAM, __VA_ARGS__); break;  \
    case 4: launch_pdl(KERNEL<4>, GRID, 256, STREAM, __VA_ARGS__); break;  \
    case 5: launch_pdl(KERNEL<5>, GRID, 256, STREAM, __VA_ARGS__); break;  \
    case 6: launch_pdl(KERNEL<6>, GRID, 256, STREAM, __VA_ARGS__); break;  \
    case 7: launch_pdl(KERNEL<7>, GRID, 256, STREAM, __VA_ARGS__); break;  \
    default: launch_pdl(KERNEL<8>, GRID, 256, STREAM, __VA_ARGS__); break; \
  }

static int grid_for_warps(int64_t work_items) {
  // persistent grid-stride: up to 4 CTAs of 8 warps per SM
  int64_t blocks = (work_items + 7) / 8;
  int64_t cap = static_cast<int64_t>(num_sms()) * 4;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return static_cast<int>(blocks);
}

static bool gate_mma_ok(int d, int E) {
  return E % 8 == 0 && d % 64 == 0 && (E == 8 || E == 16 || E == 32 || E == 64);
}

// The tensor-core gate, K split over 2 warps per token group when d allows it.
static int gate_mma_launch(const __nv_bfloat16* x, const float* wg, const float* bias, int64_t T,
                           int d, int E, int k, float* logits, int32_t* topk_idx, float* topk_w,
                           int32_t* slot_rank, int32_t* tile_counts, int32_t* tile_prefix,
                           int32_t* ws, const uint64_t* peer_bases, int64_t table_off,
                           int64_t flags_off, int rank, int world, int slot, uint32_t epoch,
                           cudaStream_t stream, GateLocalTables local = {}) {
  const int tiles = static_cast<int>((T + kGateTile - 1) / kGateTile);
  const bool split = d % 128 == 0;
  // staged split weights when they fit beside two CTAs per SM
  const size_t wsm = static_cast<size_t>(E) * (4 * static_cast<size_t>(d) + 16);
  const bool sw = wsm <= 80 * 1024;
  auto go = [&](auto kern, int threads) {
    const size_t dyn = sw ? wsm : 0;
    // static + dynamic above 48 KB needs the opt-in; raised once per kernel (all the
    if (ensure_dynamic_smem(reinterpret_cast<const void*>(kern), static_cast<int>(dyn)) !=
        cudaSuccess)
      return;  // reported by launch_status()
    timing_begin(stream);
    kern<<<tiles, threads, dyn, stream>>>(x, wg, bias, T, d, E, k, logits, topk_idx, topk_w,
                                          slot_rank, tile_counts, tile_prefix, ws, peer_bases,
                                          table_off, flags_off, rank, world, slot, epoch, local);
  };
#define FSSDP_GATE_GO(KS, SW, THREADS)                              \
  do {                                                              \
    if (E == 8) go(gate_topk_mma_kernel<1, KS, SW>, THREADS);       \
    else if (E == 16) go(gate_topk_mma_kernel<2, KS, SW>, THREADS); \
    else if (E == 32) go(gate_topk_mma_kernel<4, KS, SW>, THREADS); \
    else go(gate_topk_mma_kernel<8, KS, SW>, THREADS);              \
  } while (0)
  if (split && sw) FSSDP_GATE_GO(2, true, 256);
  else if (split) FSSDP_GATE_GO(2, false, 256);
  else if (sw) FSSDP_GATE_GO(1, true, 128);
  else FSSDP_GATE_GO(1, false, 128);
#undef FSSDP_GATE_GO
  return kOk;
}

}  // namespace fssdp

using namespace fssdp;

extern "C" {

int fssdp_gate_topk(const void* x, const float* wg, const float* bias, int64_t T, int32_t d,
                    int32_t E, int32_t k, float* logits, int32_t* topk_idx, float* topk_w, int32_t* slot_rank,
                    int32_t* tile_counts, void* stream) {
  if (T < 0 || d <= 0 || d % 8 != 0 || E <= 0 || E > kGateMaxE || k <= 0 || k > kGateMaxK ||
      k > E) {
    set_error("gate: unsupported shape");
    return kErrDimension;
  }
  if (T == 0) return kOk;
  const int tiles = static_cast<int>((T + kGateTile - 1) / kGateTile);
  if (gate_mma_ok(d, E)) {
    const int rc = gate_mma_launch(static_cast<const __nv_bfloat16*>(x), wg, bias, T, d, E, k,
                                   logits, topk_idx, topk_w, slot_rank, tile_counts, nullptr,
                                   nullptr, nullptr, 0, 0, 0, 1, -1, 0, as_stream(stream));
    if (rc != kOk) return rc;
    return launch_status();
  }
  size_t smem = kGateTile * sizeof(__nv_bfloat16) * (kGateChunk + 8) +
                static_cast<size_t>(E) * sizeof(float) * (kGateChunk + 4);
  const size_t lg_bytes = kGateTile * sizeof(float) * (kGateMaxE + 1);
  if (smem < lg_bytes) smem = lg_bytes;
  const int ept = (E + 3) / 4;
  auto launch = [&](auto kern) -> int {
    const size_t max_smem = kGateTile * sizeof(__nv_bfloat16) * (kGateChunk + 8) +
                            kGateMaxE * sizeof(float) * (kGateChunk + 4);
    if (ensure_dynamic_smem(reinterpret_cast<const void*>(kern), static_cast<int>(max_smem)) !=
        cudaSuccess)
      return launch_status();
    timing_begin(as_stream(stream));
    kern<<<tiles, kGateThreads, smem, as_stream(stream)>>>(
        static_cast<const __nv_bfloat16*>(x), wg, bias, T, d, E, k, logits, topk_idx, topk_w,
        slot_rank, tile_counts);
    return kOk;
  };
  int rc;
  if (ept <= 1) rc = launch(gate_topk_kernel<1>);
  else if (ept <= 2) rc = launch(gate_topk_kernel<2>);
  else if (ept <= 4) rc = launch(gate_topk_kernel<4>);
  else if (ept <= 8) rc = launch(gate_topk_kernel<8>);
  else rc = launch(gate_topk_kernel<16>);
  if (rc != kOk) return rc;
  return launch_status();
}

int fssdp_topk_from_logits(const float* logits, int64_t T, int32_t E, int32_t k, int32_t* topk_idx,
                           float* topk_w, int32_t* slot_rank, int32_t* tile_counts, void* stream) {
  if (T < 0 || E <= 0 || E > kGateMaxE || k <= 0 || k > kGateMaxK || k > E) {
    set_error("topk: unsupported shape");
    return kErrDimension;
  }
  if (T == 0) return kOk;
  const int tiles = static_cast<int>((T + kGateTile - 1) / kGateTile);
  timing_begin(as_stream(stream));
  topk_from_logits_kernel<<<tiles, kGateThreads, 0, as_stream(stream)>>>(
      logits, T, E, k, topk_idx, topk_w, slot_rank, tile_counts);
  return launch_status();
}

int64_t fssdp_gate_gemm_ws_bytes(int64_t T, int32_t d) {
  const int64_t rows = (T + 255) / 256 * 256;
  return 1024 + (static_cast<int64_t>(kGateN) * d * 2 + 1023) / 1024 * 1024 + rows * kGateN * 4;
}

int fssdp_gate_route(const void* x, const float* wg, const float* bias, int64_t T, int32_t d,
                     int32_t E, int32_t k, int32_t* topk_idx, float* topk_w, int32_t* slot_rank,
                     int32_t* tile_counts, int32_t* tile_prefix, int32_t* ws,
                     const uint64_t* peer_bases, int64_t table_off, int64_t flags_off,
                     int32_t rank, int32_t world, int32_t bar_slot, uint32_t epoch,
                     int32_t* local_tables, int32_t local_d_ff, int32_t local_n_mats,
                     int32_t local_param_base, void* counts_host, int64_t counts_bytes,
                     uint32_t* flag_host, uint32_t flag_value, void* gemm_ws,
                     int64_t gemm_ws_bytes, void* stream) {
  if (T < 0 || d <= 0 || d % 8 != 0 || E <= 0 || E > kGateMaxE || k <= 0 || k > kGateMaxK ||
      k > E || world <= 0 || world > kMaxWorld || rank < 0 || rank >= world ||
      (local_tables != nullptr && world != 1) ||
      (counts_host != nullptr && (counts_bytes % 16 != 0 || flag_host == nullptr))) {
    set_error("gate_route: unsupported shape (local tables need world == 1; counts push "
              "needs 16-byte multiples and a flag)");
    return kErrDimension;
  }
  const int tiles = static_cast<int>((T + kGateTile - 1) / kGateTile);
  GateLocalTables local = {};
  if (local_tables != nullptr) {  // the fssdp_tables_layout sections of a (E, 1) blob
    int64_t off[FSSDP_TAB_NSECTIONS], total = 0;
    fssdp_tables_layout(E, 1, off, &total);
    auto sec = [&](int i) {
      return reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(local_tables) + off[i]);
    };
    local.route_cum = sec(FSSDP_TAB_ROUTE_CUM);
    local.recv_base = sec(FSSDP_TAB_RECV_BASE);
    local.zero_rows = sec(FSSDP_TAB_ZERO_ROWS);
    if (local_d_ff > 0) {  // + the six GEMM tables (fssdp_local_gemm_tables' work)
      if (d % 256 != 0 || local_d_ff % 128 != 0 || local_n_mats < 2 || local_n_mats > 3) {
        set_error("gate_route: local GEMM tables need d % 256, d_ff % 128, n_mats 2 or 3");
        return kErrDimension;
      }
      local.gemm0 = reinterpret_cast<fssdp_gemm_group*>(sec(FSSDP_TAB_GEMM0));
      local.gemm_stride = off[FSSDP_TAB_GEMM0 + 1] - off[FSSDP_TAB_GEMM0];
      local.d_model = d;
      local.d_ff = local_d_ff;
      local.n_mats = local_n_mats;
      local.param_base = local_param_base;
    }
  }
  if (counts_host != nullptr) {
    local.host_counts = static_cast<int4*>(counts_host);
    local.host_n16 = static_cast<int>(counts_bytes / 16);
    local.host_flag = flag_host;
    local.host_flag_value = flag_value;
  }
  if (gemm_ws != nullptr && tiles > 0) {  // the logits on tcgen05 (gate_gemm_prep_kernel)
    if (E > kGateN / 2 || d % 64 != 0 || gemm_ws_bytes < fssdp_gate_gemm_ws_bytes(T, d)) {
      set_error("gate_route: tensor-core gate needs E <= 64, d % 64 == 0 and "
                "fssdp_gate_gemm_ws_bytes of workspace");
      return kErrDimension;
    }
    uint8_t* w8 = static_cast<uint8_t*>(gemm_ws);
    GemmGroup* group = reinterpret_cast<GemmGroup*>(w8);
    __nv_bfloat16* bmat = reinterpret_cast<__nv_bfloat16*>(w8 + 1024);
    float* cmat = reinterpret_cast<float*>(w8 + 1024 + (static_cast<int64_t>(kGateN) * d * 2 + 1023) /
                                                          1024 * 1024);
    const int m_tiles = static_cast<int>(2 * ((T + 255) / 256));  // 128-row units, pairs
    const int64_t nb = static_cast<int64_t>(kGateN) * d;
    const int pb = static_cast<int>((nb + 255) / 256 < 2 * num_sms() ? (nb + 255) / 256 : 2 * num_sms());
    timing_begin(as_stream(stream));
    gate_gemm_prep_kernel<<<pb, 256, 0, as_stream(stream)>>>(wg, E, d, bmat, group, m_tiles);
    int rc = launch_check();
    if (rc != kOk) return rc;
    GemmLaunch args = {};
    args.groups = group;
    args.num_groups = 1;
    args.n_tiles = 1;
    args.total_tiles = m_tiles;
    args.n_fast = 0;
    args.cta_group = 2;
    args.bn = kGateN;
    args.ldc = kGateN;
    args.c = cmat;
    rc = grouped_gemm_launch(0, 0, kEpiF32, x, d, T, bmat, d, kGateN,
                             static_cast<int64_t>(m_tiles) * 128, args, as_stream(stream));
    if (rc != kOk) return rc;
    // dynamic smem for the last CTA's tile-count staging (the tail's scan)
    const int stage_bytes = tiles * E * 4 <= 96 * 1024 ? tiles * E * 4 : 0;
    if (stage_bytes > 48 * 1024 &&
        ensure_dynamic_smem(reinterpret_cast<const void*>(gate_select_kernel), stage_bytes) !=
            cudaSuccess)
      return launch_status();
    gate_select_kernel<<<tiles, kGateThreads, stage_bytes, as_stream(stream)>>>(
        cmat, bias, T, E, k, topk_idx, topk_w, slot_rank, tile_counts, tile_prefix, ws,
        peer_bases, table_off, flags_off, rank, world, bar_slot, epoch, local, stage_bytes / 4);
    return launch_status();
  }
  if (!gate_mma_ok(d, E) || tiles == 0) {  // the two-kernel path (+ the local tables)
    int rc = fssdp_gate_topk(x, wg, bias, T, d, E, k, nullptr, topk_idx, topk_w, slot_rank,
                             tile_counts, stream);
    if (rc != kOk) return rc;
    rc = fssdp_route_scan_allgather(tile_counts, tiles, E, tile_prefix, peer_bases, table_off,
                                    flags_off, rank, world, bar_slot, epoch, stream);
    if (rc != kOk) return rc;
    if (local_tables != nullptr) {
      gate_local_tables_kernel<<<1, 32, 0, as_stream(stream)>>>(peer_bases, rank, table_off, E,
                                                               local);
      rc = launch_status();
      if (rc != kOk) return rc;
      if (local.gemm0 != nullptr) {
        local_gemm_tables_kernel<<<1, kGateMaxE, 0, as_stream(stream)>>>(
            peer_bases, rank, table_off, E, local.d_model, local.d_ff, local.n_mats, local.gemm0,
            local.gemm_stride, local.param_base);
        rc = launch_status();
        if (rc != kOk) return rc;
      }
    }
    if (counts_host == nullptr) return kOk;
    push_counts_kernel<<<1, 256, 0, as_stream(stream)>>>(peer_bases, rank, table_off, local);
    return launch_status();
  }
  const int rc = gate_mma_launch(static_cast<const __nv_bfloat16*>(x), wg, bias, T, d, E, k,
                                 nullptr, topk_idx, topk_w, slot_rank, tile_counts, tile_prefix,
                                 ws, peer_bases, table_off, flags_off, rank, world, bar_slot,
                                 epoch, as_stream(stream), local);
  if (rc != kOk) return rc;
  return launch_status();
}

int fssdp_route_scan_allgather(const int32_t* tile_counts, int32_t n_tiles, int32_t E,
                               int32_t* tile_prefix, const uint64_t* peer_bases, int64_t table_off,
                               int64_t flags_off, int32_t rank, int32_t world, int32_t bar_slot,
                               uint32_t epoch, void* stream) {
  if (world <= 0 || world > kMaxWorld || rank < 0 || rank >= world || E <= 0 || E > kGateMaxE) {
    set_error("route_scan: bad world/rank/E");
    return kErrDimension;
  }
  timing_begin(as_stream(stream));
  route_scan_kernel<<<1, kScanThreads, 0, as_stream(stream)>>>(tile_counts, n_tiles, E, tile_prefix,
                                                       peer_bases, table_off, flags_off, rank,
                                                       world, bar_slot, epoch);
  return launch_status();
}

int fssdp_barrier(const uint64_t* peer_bases, int64_t flags_off, int32_t rank, int32_t world,
                  int32_t bar_slot, uint32_t epoch, void* stream) {
  if (world <= 0 || world > kMaxWorld || rank < 0 || rank >= world) {
    set_error("barrier: bad world/rank");
    return kErrDimension;
  }
  timing_begin(as_stream(stream));
  launch_pdl(barrier_kernel, 1, 32, as_stream(stream), peer_bases, flags_off, rank, world,
             bar_slot, epoch);
  return launch_status();
}

int fssdp_sum_peers(const uint64_t* peer_bases, int32_t world, int64_t src_off, int64_t n,
                    float* out, void* stream) {
  if (world <= 0 || world > kMaxWorld || n < 0 || (n % 4) != 0 || (src_off % 16) != 0 ||
      (reinterpret_cast<uintptr_t>(out) & 15) != 0) {
    set_error("sum_peers: bad world / n (multiple of 4) / alignment");
    return kErrDimension;
  }
  if (n == 0) return kOk;
  const int64_t n4 = n / 4;
  int64_t blocks = (n4 + 255) / 256;
  if (blocks > 2 * num_sms()) blocks = 2 * num_sms();
  timing_begin(as_stream(stream));
  launch_pdl(sum_peers_kernel, static_cast<int>(blocks), 256, as_stream(stream), peer_bases,
             world, src_off, n4, reinterpret_cast<float4*>(out));
  return launch_status();
}

int fssdp_barrier_selftest(const uint64_t* peer_bases, int64_t flags_off, int64_t data_off,
                           int32_t world, int32_t rounds, int32_t bar_slot, uint32_t epoch0,
                           int32_t skew_ns, int32_t* errors, void* stream) {
  if (world <= 0 || world > kMaxWorld || rounds <= 0) {
    set_error("barrier_selftest: bad world/rounds");
    return kErrDimension;
  }
  int coop = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) {
    set_error("barrier_selftest: device cannot launch cooperative kernels");
    return kErrCuda;
  }
  int threads = kSelftestThreads;
  void* args[] = {&peer_bases, &flags_off, &data_off, &world,   &rounds,
                  &bar_slot,   &epoch0,    &skew_ns,  &errors};
  timing_begin(as_stream(stream));
  const cudaError_t err = cudaLaunchCooperativeKernel(
      reinterpret_cast<const void*>(barrier_selftest_kernel), dim3(world), dim3(threads), args,
      0, as_stream(stream));
  timing_end();
  if (err != cudaSuccess) {
    set_error(cudaGetErrorString(err));
    return kErrCuda;
  }
  return launch_status();
}

int fssdp_dispatch(const void* x, const int32_t* topk_idx, const int32_t* slot_rank,
                   const int32_t* tile_prefix, int64_t T, int32_t d_model, int32_t E, int32_t k,
                   int32_t world, const int32_t* route_cum, const int32_t* recv_base,
                   int32_t* slot_dest, int32_t* slot_pos, const uint64_t* peer_bases,
                   int64_t recv_off, const int32_t* zero_rows, int32_t n_zero, int64_t flags_off,
                   int32_t rank, int32_t bar_slot, uint32_t epoch, uint32_t* grid_counter,
                   void* stream) {
  if (d_model % 8 != 0 || world <= 0 || world > kMaxWorld || k > kGateMaxK) {
    set_error("dispatch: bad shape");
    return kErrDimension;
  }
  const int grid = grid_for_warps((T * k + kBatch - 1) / kBatch);  // one warp per batch
  timing_begin(as_stream(stream));
  dispatch_kernel<<<grid, 256, 0, as_stream(stream)>>>(
      static_cast<const __nv_bfloat16*>(x), topk_idx, slot_rank, tile_prefix, T, d_model, E, k,
      world, route_cum, recv_base, slot_dest, slot_pos, peer_bases, recv_off, zero_rows, n_zero,
      flags_off, rank, bar_slot, epoch, grid_counter);
  return launch_status();
}

int fssdp_local_gemm_tables(const uint64_t* peer_bases, int32_t rank, int64_t table_off,
                            int32_t E, int32_t d_model, int32_t d_ff, int32_t n_mats,
                            int32_t param_base, void* local_tables, void* stream) {
  if (E <= 0 || E > kGateMaxE || d_model % 256 != 0 || d_ff % 128 != 0 || n_mats < 2 ||
      n_mats > 3 || local_tables == nullptr) {
    set_error("local_gemm_tables: unsupported shape");
    return kErrDimension;
  }
  int64_t off[FSSDP_TAB_NSECTIONS], total = 0;
  fssdp_tables_layout(E, 1, off, &total);
  uint8_t* blob = static_cast<uint8_t*>(local_tables);
  local_gemm_tables_kernel<<<1, kGateMaxE, 0, as_stream(stream)>>>(
      peer_bases, rank, table_off, E, d_model, d_ff, n_mats,
      reinterpret_cast<fssdp_gemm_group*>(blob + off[FSSDP_TAB_GEMM0]),
      off[FSSDP_TAB_GEMM0 + 1] - off[FSSDP_TAB_GEMM0], param_base);
  return launch_status();
}

int fssdp_combine(const int32_t* slot_dest, const int32_t* slot_pos, const float* topk_w, int64_t T,
                  int32_t d_model, int32_t k, const uint64_t* peer_bases, int64_t y_off,
                  void* y_out, void* y_slots, void* stream) {
  if (d_model % 8 != 0 || k <= 0 || k > kGateMaxK) {
    set_error("combine: bad shape");
    return kErrDimension;
  }
  if (T == 0) return kOk;
  const int grid = grid_for_warps((T + kTokBatch - 1) / kTokBatch);
  timing_begin(as_stream(stream));
  FSSDP_DISPATCH_K(k, combine_kernel, grid, as_stream(stream), slot_dest, slot_pos, topk_w, T,
                   d_model, peer_bases, y_off, static_cast<__nv_bfloat16*>(y_out),
                   static_cast<__nv_bfloat16*>(y_slots));
  return launch_status();
}

int fssdp_dispatch_grad(const void* dy, const int32_t* slot_dest, const int32_t* slot_pos,
                        const float* topk_w, int64_t T, int32_t d_model, int32_t k,
                        const uint64_t* peer_bases, int64_t y_off, const void* y_slots,
                        int64_t dy_recv_off, float* slot_grad, float* dlogit_out,
                        const int32_t* zero_rows, int32_t n_zero, int64_t flags_off, int32_t rank,
                        int32_t world, int32_t bar_slot, uint32_t epoch, uint32_t* grid_counter,
                        void* stream) {
  if (d_model % 8 != 0 || world <= 0 || world > kMaxWorld || k <= 0 || k > kGateMaxK ||
      (dlogit_out != nullptr && (kBatch % k != 0 || slot_grad == nullptr))) {
    set_error("dispatch_grad: bad shape");
    return kErrDimension;
  }
  timing_begin(as_stream(stream));
  dispatch_grad_kernel<<<grid_for_warps((T * k + kBatch - 1) / kBatch), 256, 0, as_stream(stream)>>>(
      static_cast<const __nv_bfloat16*>(dy), slot_dest, slot_pos, topk_w, T, d_model, k,
      peer_bases, y_off, static_cast<const __nv_bfloat16*>(y_slots), dy_recv_off, slot_grad,
      dlogit_out, zero_rows, n_zero, flags_off, rank, world,
      bar_slot, epoch, grid_counter);
  return launch_status();
}

static int combine_dx_launch(const int32_t* slot_dest, const int32_t* slot_pos,
                             const int32_t* topk_idx, const float* topk_w, const float* slot_grad,
                             const float* wg, int64_t T, int32_t d_model, int32_t E, int32_t k,
                             const uint64_t* peer_bases, int64_t dxe_off, float* dlogit_out,
                             void* dx_out, const void* dy, int64_t y_off, const void* y_slots,
                             float* slot_grad_out, void* stream);

int fssdp_combine_dx(const int32_t* slot_dest, const int32_t* slot_pos, const int32_t* topk_idx,
                     const float* topk_w, const float* slot_grad, const float* wg, int64_t T,
                     int32_t d_model, int32_t E, int32_t k, const uint64_t* peer_bases,
                     int64_t dxe_off, float* dlogit_out, void* dx_out, void* stream) {
  if (slot_grad == nullptr && T > 0) {
    set_error("combine_dx: slot_grad is required (fssdp_combine_dx_dots computes it)");
    return kErrDimension;
  }
  return combine_dx_launch(slot_dest, slot_pos, topk_idx, topk_w, slot_grad, wg, T, d_model, E, k,
                           peer_bases, dxe_off, dlogit_out, dx_out, nullptr, 0, nullptr, nullptr,
                           stream);
}

int fssdp_combine_dx_dots(const int32_t* slot_dest, const int32_t* slot_pos,
                          const int32_t* topk_idx, const float* topk_w, const void* dy,
                          const void* y_slots, int64_t y_off, const float* wg, int64_t T,
                          int32_t d_model, int32_t E, int32_t k, const uint64_t* peer_bases,
                          int64_t dxe_off, float* slot_grad_out, float* dlogit_out, void* dx_out,
                          void* stream) {
  if (dy == nullptr && T > 0) {
    set_error("combine_dx_dots: dy is required");
    return kErrDimension;
  }
  return combine_dx_launch(slot_dest, slot_pos, topk_idx, topk_w, nullptr, wg, T, d_model, E, k,
                           peer_bases, dxe_off, dlogit_out, dx_out, dy, y_off, y_slots,
                           slot_grad_out, stream);
}

static int combine_dx_launch(const int32_t* slot_dest, const int32_t* slot_pos,
                             const int32_t* topk_idx, const float* topk_w, const float* slot_grad,
                             const float* wg, int64_t T, int32_t d_model, int32_t E, int32_t k,
                             const uint64_t* peer_bases, int64_t dxe_off, float* dlogit_out,
                             void* dx_out, const void* dy, int64_t y_off, const void* y_slots,
                             float* slot_grad_out, void* stream) {
  if (d_model % 8 != 0 || k <= 0 || k > kGateMaxK || E > kGateMaxE) {
    set_error("combine_dx: bad shape");
    return kErrDimension;
  }
  if (T == 0) return kOk;
  // CTA cap (FSSDP_COMBINE_DX_CTAS, experiments): it runs beside the weight-gradient GEMMs
  static const int cap = [] {
    const char* v = getenv("FSSDP_COMBINE_DX_CTAS");
    return v ? atoi(v) : 0;
  }();
  int grid = grid_for_warps((T + kTokBatch - 1) / kTokBatch);
  if (cap > 0 && grid > cap) grid = cap;
  timing_begin(as_stream(stream));
  FSSDP_DISPATCH_K(k, combine_dx_kernel, grid, as_stream(stream), slot_dest, slot_pos, topk_idx,
                   topk_w, slot_grad, wg, T, d_model, peer_bases, dxe_off, dlogit_out,
                   static_cast<__nv_bfloat16*>(dx_out), static_cast<const __nv_bfloat16*>(dy),
                   y_off, static_cast<const __nv_bfloat16*>(y_slots), slot_grad_out);
  return launch_status();
}

int fssdp_gate_wgrad(const void* x, const int32_t* topk_idx, const float* dlogit, int64_t T,
                     int32_t d_model, int32_t E, int32_t k, float* workspace, float* dwg_out,
                     void* stream) {
  if (E > kGateMaxE || d_model <= 0 || d_model % 4 != 0 || k > kGateMaxK) {
    set_error("gate_wgrad: bad shape");
    return kErrDimension;
  }
  // fixed FSSDP_WG_TILE-token runs (the partition, hence the fp32 grouping, depends only on
  // the token index), reduced in run order
  const int col_blocks = (d_model + kWgCols - 1) / kWgCols;
  const int64_t tok_per_cta = FSSDP_WG_TILE;
  const int n_tiles = static_cast<int>((T + tok_per_cta - 1) / tok_per_cta);
  if (n_tiles > 0) {
    const int smem = E * kWgThreads * static_cast<int>(sizeof(float4));
    if (smem > 48 * 1024 &&
        ensure_dynamic_smem(reinterpret_cast<const void*>(gate_wgrad_partial_kernel), smem) !=
            cudaSuccess)
      return launch_status();
    dim3 grid(col_blocks, n_tiles);
    timing_begin(as_stream(stream));
    gate_wgrad_partial_kernel<<<grid, kWgThreads, smem, as_stream(stream)>>>(
        static_cast<const __nv_bfloat16*>(x), topk_idx, dlogit, T, d_model, E, k, tok_per_cta,
        workspace);
    int rc = launch_check();
    if (rc != kOk) return rc;
  }
  const int64_t n_out = static_cast<int64_t>(E) * d_model;
  timing_begin(as_stream(stream));
  gate_wgrad_reduce_kernel<<<static_cast<unsigned>((n_out + 31) / 32), 256, 0, as_stream(stream)>>>(
      workspace, n_tiles, d_model, E, dwg_out);
  return launch_status();
}

int64_t fssdp_gate_wgrad_tc_ws_bytes(int64_t T, int32_t d) {
  const int64_t rows = (T + 63) / 64 * 64;
  const int splits = gate_wgrad_splits(T, d);
  return 4096 + rows * kGateN * 2 + static_cast<int64_t>(splits) * d * kGateN * 4;
}

int fssdp_gate_wgrad_tc(const void* x, const int32_t* topk_idx, const float* dlogit, int64_t T,
                        int32_t d_model, int32_t E, int32_t k, void* ws, int64_t ws_bytes,
                        float* dwg_out, void* stream) {
  if (E <= 0 || E > kGateN / 2 || k <= 0 || k > kGateMaxK || k > E || d_model <= 0 ||
      d_model % 256 != 0 || T < 0 || ws_bytes < fssdp_gate_wgrad_tc_ws_bytes(T, d_model)) {
    set_error("gate_wgrad_tc: needs E <= 64, d_model % 256 == 0 and "
              "fssdp_gate_wgrad_tc_ws_bytes of workspace");
    return kErrDimension;
  }
  const int64_t rows = (T + 63) / 64 * 64;
  const int splits = gate_wgrad_splits(T, d_model);
  const int64_t ks = (rows / 64 + splits - 1) / splits * 64;  // K rows per split
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  GemmGroup* groups = reinterpret_cast<GemmGroup*>(w8);
  __nv_bfloat16* g = reinterpret_cast<__nv_bfloat16*>(w8 + 4096);
  float* c = reinterpret_cast<float*>(w8 + 4096 + rows * kGateN * 2);
  cudaStream_t s = as_stream(stream);
  const int64_t n16 = rows * kGateN / 8;
  // one 16-byte vector per thread: every thread's two dependent loads in flight at once
  const int pb = static_cast<int>((n16 + 255) / 256 < 16 * num_sms() ? (n16 + 255) / 256
                                                                      : 16 * num_sms());
  timing_begin(s);
  gate_wgrad_prep_kernel<<<pb > 0 ? pb : 1, 256, 0, s>>>(topk_idx, dlogit, T, rows, E, k,
                                                       d_model, splits, ks, g, groups);
  int rc = launch_check();
  if (rc != kOk) return rc;
  if (T > 0) {
    GemmLaunch args = {};
    args.groups = groups;
    args.num_groups = splits;
    args.n_tiles = 1;
    args.total_tiles = splits * (d_model / 128);
    args.n_fast = 0;
    args.cta_group = 2;
    args.bn = kGateN;
    args.ldc = kGateN;
    args.c = c;
    // A = x [T][d] read M-contiguous (MN-major), B = G [rows][kGateN] (MN-major)
    rc = grouped_gemm_launch(1, 1, kEpiF32, x, d_model, T, g, kGateN, rows,
                             static_cast<int64_t>(splits) * d_model, args, s);
    if (rc != kOk) return rc;
  }
  const int64_t n_out = static_cast<int64_t>(E) * d_model;
  timing_begin(s);
  gate_wgrad_tc_reduce_kernel<<<static_cast<unsigned>((n_out + 255) / 256), 256, 0, s>>>(
      c, T > 0 ? splits : 0, d_model, E, dwg_out);
  return launch_status();
}

int fssdp_gather_slots(const uint64_t* peer_bases, int32_t rank, int64_t src_off, int64_t dst_off,
                       int64_t slot_bytes, int64_t copy_bytes, const int32_t* copies,
                       int32_t n_copies, int32_t max_ctas, void* stream) {
  if (copy_bytes == 0) copy_bytes = slot_bytes;
  if (slot_bytes % 16 != 0 || copy_bytes % 16 != 0 || copy_bytes < 0 || copy_bytes > slot_bytes) {
    set_error("gather_slots: slot_bytes / copy_bytes must be multiples of 16, copy <= slot");
    return kErrDimension;
  }
  if (n_copies <= 0) return kOk;
  static const int impl = [] {
    const char* v = getenv("FSSDP_SPAG_IMPL");
    return (v && strcmp(v, "ldg") == 0) ? 0 : 1;  // default: TMA-staged bulk copies
  }();
  if (impl == 1 || src_off != dst_off || copy_bytes != slot_bytes) {
    int64_t chunk = copy_bytes * n_copies / (2 * static_cast<int64_t>(num_sms()));
    chunk = (chunk + kTmaSub - 1) / kTmaSub * kTmaSub;
    if (chunk < 4 * kTmaSub) chunk = 4 * kTmaSub;
    if (chunk > (1 << 20)) chunk = 1 << 20;
    // a bounded footprint (max_ctas > 0): a copy running beside other kernels must leave
    // them SM slots — small latency-bound transfers stall behind a full-width copy
    while (max_ctas > 0 && chunk < copy_bytes &&
           ((copy_bytes + chunk - 1) / chunk) * n_copies > max_ctas)
      chunk *= 2;
    dim3 grid(static_cast<unsigned>((copy_bytes + chunk - 1) / chunk), n_copies);
    timing_begin(as_stream(stream));
    spag_tma_kernel<<<grid, 32, 0, as_stream(stream)>>>(peer_bases, rank, src_off, dst_off,
                                                        slot_bytes, copy_bytes, copies, chunk);
    return launch_status();
  }
  const int64_t chunk = coll_chunk_bytes(slot_bytes * n_copies, num_sms());
  dim3 grid(static_cast<unsigned>((slot_bytes + chunk - 1) / chunk), n_copies);
  timing_begin(as_stream(stream));
  spag_kernel<<<grid, 256, 0, as_stream(stream)>>>(peer_bases, rank, src_off, slot_bytes, copies,
                                                   chunk);
  return launch_status();
}

int fssdp_spag(const uint64_t* peer_bases, int32_t rank, int64_t param_off, int64_t slot_bytes,
               const int32_t* copies, int32_t n_copies, void* stream) {
  return fssdp_gather_slots(peer_bases, rank, param_off, param_off, slot_bytes, 0, copies,
                            n_copies, 0, stream);
}

int fssdp_sprs(const uint64_t* peer_bases, int32_t rank, int64_t grad_off, int64_t stage_off,
               int64_t slot_elems, int32_t elem_bytes, const int32_t* jobs, int32_t n_jobs,
               const int32_t* srcs, void* stream) {
  if ((elem_bytes != 2 && elem_bytes != 4) || (slot_elems * elem_bytes) % 16 != 0) {
    set_error("sprs: elem_bytes must be 2 (bf16) or 4 (fp32) and a slot whole 16-byte vectors");
    return kErrDimension;
  }
  const int64_t slot_bytes = slot_elems * elem_bytes;
  if (n_jobs <= 0) return kOk;
  // CTA budget (FSSDP_SPRS_CTAS, default one per SM): SpRS runs beside the backward GEMMs
  // and a full 4-per-SM grid slows them more than it speeds the reduction (measured, N=4)
  static const int budget = [] {
    const char* v = getenv("FSSDP_SPRS_CTAS");
    return v ? atoi(v) : num_sms();
  }();
  const int64_t chunk = coll_chunk_bytes(slot_bytes * n_jobs, num_sms());
  const int n_chunks = static_cast<int>((slot_bytes + chunk - 1) / chunk);
  const int n_units = n_chunks * n_jobs;
  const int ctas = budget > 0 ? (budget < n_units ? budget : n_units) : n_units;
  timing_begin(as_stream(stream));
  if (elem_bytes == 2)
    sprs_kernel<true><<<ctas, 256, 0, as_stream(stream)>>>(peer_bases, rank, grad_off, stage_off,
                                                           slot_bytes, jobs, srcs, chunk, n_chunks,
                                                           n_units);
  else
    sprs_kernel<false><<<ctas, 256, 0, as_stream(stream)>>>(peer_bases, rank, grad_off,
                                                            stage_off, slot_bytes, jobs, srcs,
                                                            chunk, n_chunks, n_units);
  return launch_status();
}

int fssdp_sprs_pull(const uint64_t* peer_bases, int32_t rank, int64_t grad_off,
                    int64_t slot_elems, int32_t elem_bytes, const int32_t* jobs, int32_t n_jobs,
                    const int32_t* pull_srcs, void* stream) {
  if ((elem_bytes != 2 && elem_bytes != 4) || (slot_elems * elem_bytes) % 16 != 0) {
    set_error("sprs_pull: elem_bytes must be 2 (bf16) or 4 (fp32) and a slot whole 16-byte "
              "vectors");
    return kErrDimension;
  }
  if (n_jobs <= 0) return kOk;
  const int64_t slot_bytes = slot_elems * elem_bytes;
  constexpr int kSmem = kPullRing * kPullSub;
  auto kern = elem_bytes == 2 ? sprs_pull_kernel<true> : sprs_pull_kernel<false>;
  if (ensure_dynamic_smem(reinterpret_cast<const void*>(kern), kSmem) != cudaSuccess) {
    set_error("sprs_pull: cannot reserve the TMA ring");
    return kErrCuda;
  }
  // CTA budget (FSSDP_SPRS_PULL_CTAS, default 3 per SM): beside the backward GEMMs the
  // caller may want fewer
  static const int budget = [] {
    const char* v = getenv("FSSDP_SPRS_PULL_CTAS");
    return v ? atoi(v) : 3 * num_sms();
  }();
  int64_t chunk = slot_bytes * n_jobs / (3 * static_cast<int64_t>(num_sms()));
  chunk = (chunk + kPullSub - 1) / kPullSub * kPullSub;
  if (chunk < 4 * kPullSub) chunk = 4 * kPullSub;
  if (chunk > (1 << 20)) chunk = 1 << 20;
  const int n_chunks = static_cast<int>((slot_bytes + chunk - 1) / chunk);
  const int n_units = n_chunks * n_jobs;
  const int ctas = budget > 0 ? (budget < n_units ? budget : n_units) : n_units;
  timing_begin(as_stream(stream));
  kern<<<ctas, 32 * (kPullWarps + 1), kSmem, as_stream(stream)>>>(
      peer_bases, rank, grad_off, slot_bytes, jobs, pull_srcs, chunk, n_chunks, n_units);
  return launch_status();
}

int fssdp_push_host(const void* src_dev, void* dst_host, int64_t bytes, uint32_t* flag_host,
                    uint32_t flag_value, void* stream) {
  if (bytes < 0 || bytes % 16 != 0 || bytes > (int64_t(1) << 24)) {
    set_error("push_host: bytes must be a multiple of 16 and at most 16 MiB");
    return kErrDimension;
  }
  timing_begin(as_stream(stream));
  push_host_kernel<<<1, 256, 0, as_stream(stream)>>>(static_cast<const int4*>(src_dev),
                                                    static_cast<int4*>(dst_host),
                                                    static_cast<int>(bytes / 16), flag_host,
                                                    flag_value);
  return launch_status();
}

int fssdp_pull_host(void* dst_dev, const void* src_host, int64_t bytes, void* stream) {
  if (bytes < 0 || bytes % 16 != 0 || bytes > (int64_t(1) << 24)) {
    set_error("pull_host: bytes must be a multiple of 16 and at most 16 MiB");
    return kErrDimension;
  }
  if (bytes == 0) return kOk;
  const int n16 = static_cast<int>(bytes / 16);
  const int grid = (n16 + 255) / 256 < 16 ? (n16 + 255) / 256 : 16;
  timing_begin(as_stream(stream));
  pull_host_kernel<<<grid, 256, 0, as_stream(stream)>>>(static_cast<const int4*>(src_host),
                                                       static_cast<int4*>(dst_dev), n16);
  return launch_status();
}

int fssdp_host_wait(const uint32_t* flag_host, uint32_t value, double timeout_s) {
  const volatile uint32_t* f = flag_host;
  const auto t0 = std::chrono::steady_clock::now();
  for (uint64_t spins = 0;; ++spins) {
    if (*f == value) {
      std::atomic_thread_fence(std::memory_order_acquire);
      return kOk;
    }
    if ((spins & 1023) == 0 &&
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
      set_error("host_wait: timed out waiting for the device");
      return kErrCuda;
    }
  }
}

}  // extern "C"
