// Grouped expert-FFN GEMM for sm_100a (K5 forward, K7 dgrad/wgrad).
//
// One persistent, warp-specialised kernel serves all six GEMMs of an FSSDP MoE layer
// (fwd1, fwd2, dgrad2, dgrad1, wgrad1, wgrad2).  Operands are staged by TMA
// (cp.async.bulk.tensor, SWIZZLE_128B) into a shared-memory ring, multiplied by
// tcgen05.mma (kind::f16, bf16 in / fp32 accumulate) into a double-buffered TMEM
// accumulator, and drained by four epilogue warps that fuse the activation (GeLU fwd,
// GeLU' in dgrad) and the output cast, then hand 32x32 tiles to TMA bulk stores through
// double-buffered, bank-conflict-free swizzled staging buffers.
//
// CG = 2 (default): a CTA pair (cluster of 2) computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 issued by the leader; each CTA stages only its 128-row half of
// A and its 128-column half of B (32 KB per k-block instead of 48 KB for a 128 x 256
// single-CTA tile), TMA bytes of both CTAs complete on the leader's mbarrier, MMA
// completion is multicast to both CTAs, and each CTA drains its own 128 TMEM lanes.
// CG = 1: the single-CTA 128 x 256 variant (used when a GEMM has an odd number of 128-row
// tiles in some group).
//
// Grouping: every local expert (owned shard or SpAG replica) is one group.  A group's
// tokens are a 256-row-aligned segment of the receive buffer, so an M tile never
// straddles two experts; for wgrad the token axis is K and the segment padding rows are
// zero, so K blocks never mix experts either.
//
// Warp roles (192 threads): w0 = TMA producer, w1 = MMA issuer (leader) + TMEM owner,
// w2..w5 = epilogue (warp w reads TMEM lanes 32*(w%4) .. +31).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fssdp_internal.h"
#include "ptx.cuh"

namespace fssdp {

// Diagnostic build only (build.py --gemm-profile): per-CTA cycle counters of the roles'
// waits — producer waiting for a free stage, MMA waiting for data / for the epilogue,
// epilogue waiting for the accumulator — read back with fssdp_gemm_profile_read.
#ifdef FSSDP_GEMM_PROFILE
__device__ unsigned long long g_gemm_prof[1024][8];
#define PROF_T0(v) const long long v = clock64()
#define PROF_ADD(slot, v) atomicAdd(&g_gemm_prof[blockIdx.x][slot], (unsigned long long)(clock64() - (v)))
#define PROF_INC(slot) atomicAdd(&g_gemm_prof[blockIdx.x][slot], 1ull)
#else
#define PROF_T0(v)
#define PROF_ADD(slot, v)
#define PROF_INC(slot)
#endif

constexpr int kBM = 128;  // rows per CTA
// K per pipeline stage: 64 (one 128-byte swizzle atom of bf16) or 128 — two atoms staged by
// ONE 3-D TMA load per operand (half the load instructions per byte; fewer, larger stages).
// FSSDP_GEMM_BK: 0 = per GEMM (below), 64 / 128 = every CTA-pair GEMM (experiments).
// 128 pays where B is MN-major and the epilogue leaves three 64 KB stages — dgrad1 (bf16)
// and dgrad2 (dGeLU): cfg2 step -1.7 % (dgrad1 -10 %, dgrad2 -4 %), while the K-major and
// the MN/MN GEMMs lose 1-3 % with half as many stages, and cfg4's SwiGLU epilogues (two
// stages) 1 % per step (interleaved A/B).  Single-CTA tiles keep 64 (shared memory).
#ifndef FSSDP_GEMM_BK
#define FSSDP_GEMM_BK 0
#endif
// MN/MN GEMMs (the wgrads): 64 (96 measured neutral: wgrad1 -2 %, wgrad2 +0.5 %; 128 — three
// stages — slightly slower); FSSDP_GEMM_BK_MNMN overrides (any multiple of 16, MN-major
// boxes take kBK K rows)
#ifndef FSSDP_GEMM_BK_MNMN
#define FSSDP_GEMM_BK_MNMN 64
#endif
constexpr int k_block(bool a_mn, bool b_mn, int epi, int cg) {
  return cg < 2 ? 64
         : FSSDP_GEMM_BK != 0 ? FSSDP_GEMM_BK
         : (!a_mn && b_mn && (epi == FSSDP_EPI_BF16 || epi == FSSDP_EPI_DGELU)) ? 128
         : (a_mn && b_mn) ? FSSDP_GEMM_BK_MNMN
                          : 64;
}
// Epilogue warps: 4 (one per TMEM lane quarter), or 8 (two per quarter, column halves)
// for the GeLU epilogue, whose per-element math otherwise outlasts a K = d_model mainloop
// (the extra staging smem costs one mainloop stage).
#ifndef FSSDP_GELU_EPI_WARPS
#define FSSDP_GELU_EPI_WARPS 4
#endif
#ifndef FSSDP_F32_SETS
#define FSSDP_F32_SETS 2
#endif
#ifndef FSSDP_GELU_SETS
#define FSSDP_GELU_SETS 2
#endif
// The bf16-output MN/MN GEMMs (the weight gradients): 8 epilogue warps, two per TMEM lane
// quarter on column halves — with K = one expert's token rows, short-K tiles outrun a
// 4-warp epilogue (cfg4's 64 fine-grained experts), and their 2 KB staging tiles leave room
// for 8 warps at 6 stages.  cfg4 step -5.3 % (wgrad1 517 -> 446 us, wgrad2 252 -> 215 us),
// cfg2 -0.5 % (interleaved A/B).  FSSDP_WGRAD_EPI_WARPS=4 restores one warp per quarter
#ifndef FSSDP_WGRAD_EPI_WARPS
#define FSSDP_WGRAD_EPI_WARPS 8
#endif
template <int EPI, bool MNMN = false>
constexpr int epi_warps() {
  return EPI == FSSDP_EPI_GELU ? FSSDP_GELU_EPI_WARPS
         : (EPI == FSSDP_EPI_BF16 && MNMN) ? FSSDP_WGRAD_EPI_WARPS
                                           : 4;
}
template <int EPI, bool MNMN = false>
constexpr int gemm_threads() {
  return 64 + 32 * epi_warps<EPI, MNMN>();
}
constexpr int kEpiCols = 32;  // columns per epilogue chunk (one 32x32 TMA store box)
// Dynamic tile scheduling (GemmLaunch.sched != null): the (leader) producer takes the next
// tile from a global counter and hands its id to the MMA issuer, the epilogue warps and
// the peer CTA through a ring of kSched entries — CTA (pairs) that start late, or whose
// SMs are shared with a co-running kernel, simply take fewer tiles.
constexpr int kSched = 8;

template <int BN, int EPI, int CG, int BK = 64, int EW = epi_warps<EPI>()>
struct GemmSmem {
  static constexpr int kEpiWarps = EW;
  static constexpr int kBK = BK;             // K per stage
  static constexpr int kKC = kBK / 64;       // 64-wide K chunks per stage
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = (BN / CG) * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kOutBytes = (EPI == kEpiF32) ? 4 : 2;
  static constexpr int kBufBytes = 32 * kEpiCols * kOutBytes;  // one 32x32 staging tile
  // output staging tiles per warp (two sets, so a store can drain while the next chunk is
  // staged): C; C + C2 (GeLU); a1 + a3 + h (SwiGLU); da1 + da3 (SwiGLU backward)
  static constexpr int kOutTiles = EPI == kEpiGelu ? 2 : EPI == kEpiSwiglu ? 3
                                   : EPI == kEpiDSwiglu ? 2 : 1;
  // staging sets per epilogue warp: chunk c uses set c % kSets and may reuse it once the
  // TMA store issued kSets chunks earlier has read it (fp32 outputs: FSSDP_F32_SETS)
  static constexpr int kSets = EPI == kEpiF32 ? FSSDP_F32_SETS : EPI == kEpiGelu ? FSSDP_GELU_SETS : 2;
  static constexpr int kCBufs = kSets * kOutTiles;
  // aux-tile prefetch ring (dgrad2): entries of one tile (GeLU') or two (a1, a3)
  static constexpr int kAuxBufs =
      EPI == kEpiDGelu ? (CG == 2 && BK == 64 ? 4 : 2) : EPI == kEpiDSwiglu ? 2 : 0;
  static constexpr int kAuxTiles = EPI == kEpiDSwiglu ? 2 : 1;
  static constexpr int kEpiWarpBytes = (kCBufs + kAuxBufs * kAuxTiles) * kBufBytes;
  // as many mainloop stages (up to 6) as the 227 KB budget leaves
  static constexpr int kEpiBytes = kEpiWarps * kEpiWarpBytes;
  // dynamic tile scheduler ring (kSched entries): full / empty mbarriers + the tile ids
  static constexpr int kSchedBytes = 2 * kSched * 8 + kSched * 8;
  static constexpr int kBarBytes = (2 * 6 + 4 + 4 * kEpiWarps) * 8 + 16 + kSchedBytes;
  static constexpr int kFit = (232448 - 1024 - kBarBytes - kEpiBytes) / kStageBytes;
  static constexpr int kStages = kFit < 6 ? kFit : 6;
  static_assert(kStages >= 2, "shared memory budget exceeded");
  static constexpr int kEpiOffset = kStages * kStageBytes;
  static constexpr int kBarOffset = kEpiOffset + kEpiBytes;
  // full[S], empty[S], tmem_full[2], tmem_empty[2], aux[kEpiWarps][4], tmem base slot
  static constexpr int kTotal =
      kBarOffset + (2 * kStages + 4 + 4 * kEpiWarps) * 8 + 16 + kSchedBytes;
  static constexpr int kDynamic = kTotal + 1024;  // slack for 1024-B alignment
  static_assert(kDynamic <= 232448, "shared memory budget exceeded");
};

// tanh.approx (MUFU) is below bf16 output resolution; parity is tolerance-based.

// Work order of a persistent CTA (pair): round r takes tile r*units + unit, in reverse
// CTA order on odd rounds ("snake").  With groups listed by descending cost (wgrad: K =
// segment rows), this deals the tiles out close to longest-processing-time-first.
__device__ __forceinline__ int snake_tile(int round, int unit, int units) {
  return round * units + ((round & 1) ? units - 1 - unit : unit);
}

// Packed fp32x2 (FFMA2 / FMUL2 on sm_100): the GeLU epilogue works on element pairs, which
// halves its FP instruction count — it is the limiter of the fwd1 tile loop.
__device__ __forceinline__ uint64_t f2_pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 f2_unpack(uint64_t r) {
  float2 f;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(f.x), "=f"(f.y) : "l"(r));
  return f;
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// gelu and gelu' of an element pair from one tanh each:
//   t = tanh(k0 (x + k1 x^3)),  gelu = hx (1 + t),
//   gelu' = 0.5 (1 + t) + hx (1 - t^2) (k0 + 3 k0 k1 x^2)
__device__ __forceinline__ void gelu_and_grad2(uint64_t x, uint64_t& g, uint64_t& dg) {
  constexpr float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const uint64_t one = f2_pack(1.f, 1.f), half = f2_pack(0.5f, 0.5f);
  const uint64_t x2 = f2_mul(x, x);
  const uint64_t v = f2_fma(f2_mul(f2_pack(k1, k1), x2), x, x);
  const float2 a = f2_unpack(f2_mul(f2_pack(k0, k0), v));
  const uint64_t t = f2_pack(tanh_approx(a.x), tanh_approx(a.y));
  const uint64_t hx = f2_mul(half, x);
  g = f2_fma(hx, t, hx);
  const uint64_t q = f2_fma(f2_mul(t, f2_pack(-1.f, -1.f)), t, one);  // 1 - t^2
  const uint64_t w = f2_fma(f2_pack(3.f * k1 * k0, 3.f * k1 * k0), x2, f2_pack(k0, k0));
  dg = f2_fma(half, f2_add(one, t), f2_mul(f2_mul(hx, q), w));
}

// SwiGLU backward of one element from the fp32 dh and the saved bf16 a1, a3 (both the
// normal and the swapped-tail epilogue use this one expression: bit-identical results):
//   s = sigmoid(a1), d1 = dh a3 s (1 + a1 (1 - s)), d3 = dh silu(a1)
__device__ __forceinline__ void dswiglu1(float dh, float a1, float a3, float& d1, float& d3) {
  const float sg = __frcp_rn(1.f + __expf(-a1));
  const float ds = sg * (1.f + a1 * (1.f - sg));
  d1 = dh * a3 * ds;
  d3 = dh * a1 * sg;
}

struct TileCoord {
  int group, m_tile, n_tile;  // m_tile in units of CG * 128 rows
};

// Tiles are enumerated in units of (CG*128 rows) x BN columns; groups carry m_tiles and
// tile_start in 128-row units (both even when CG == 2).
// CL = 2: a cluster of two CTA pairs takes N tiles (2 n2, 2 n2 + 1) of the same M tile
// (N-fastest order only); `pair` selects this pair's one.
template <int CG, int CL = 1>
__device__ __forceinline__ TileCoord locate_tile(const GemmGroup* __restrict__ groups,
                                                 int num_groups, int n_tiles, int n_fast,
                                                 int tile, int& cursor, int pair = 0) {
  // A role's tiles come in increasing order (snake rounds, or the scheduler's counter), so
  // the group search resumes from the previous tile's group: a scan from group 0 is a chain
  // of dependent loads as long as the group index (64+ groups at cfg4), at every tile.
  constexpr int U = CG * CL;
  int g = groups[cursor].tile_start / U <= tile ? cursor : 0;
  while (g + 1 < num_groups && groups[g + 1].tile_start / U <= tile) ++g;
  cursor = g;
  const int local = tile - groups[g].tile_start / U;
  const int mt = groups[g].m_tiles / CG;
  const int nt = n_tiles / CL;
  TileCoord tc;
  tc.group = g;
  if (n_fast) {  // neighbouring CTAs share the A tile (activation rows) in L2
    tc.n_tile = (local % nt) * CL + pair;
    tc.m_tile = local / nt;
  } else {  // neighbouring CTAs share the B tile (weights) in L2
    tc.m_tile = local % mt;
    tc.n_tile = local / mt;
  }
  return tc;
}

// Swizzled staging addresses: row r of a 32-row tile, 16-byte chunk j.
__device__ __forceinline__ uint32_t sw64(int r, int j) {  // 64-byte rows, SWIZZLE_64B
  return static_cast<uint32_t>(r * 64 + ((j ^ ((r >> 1) & 3)) << 4));
}
__device__ __forceinline__ uint32_t sw128(int r, int j) {  // 128-byte rows, SWIZZLE_128B
  return static_cast<uint32_t>(r * 128 + ((j ^ (r & 7)) << 4));
}

// CGX: 1 = one CTA per 128x256 tile, 2 = a CTA pair per 256x256 tile (cta_group::2),
// 4 = clusters of two pairs on neighbouring N tiles of one M tile: the A tile is loaded
// once per cluster and multicast into both pairs (TMA .multicast::cluster), halving the
// A operand's L2 -> SM traffic.
template <bool A_MN, bool B_MN, int BN, int EPI, int CGX>
__global__ void __launch_bounds__(gemm_threads<EPI, A_MN && B_MN>(), 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                        const __grid_constant__ CUtensorMap map_b,
                        const __grid_constant__ CUtensorMap map_c,
                        const __grid_constant__ CUtensorMap map_x,
                        const __grid_constant__ GemmLaunch args) {
  constexpr int CG = CGX == 4 ? 2 : CGX;  // CTAs per tile
  constexpr int CL = CGX == 4 ? 2 : 1;    // tiles (pairs) per cluster
  using S = GemmSmem<BN, EPI, CG, k_block(A_MN, B_MN, EPI, CG), epi_warps<EPI, A_MN && B_MN>()>;
  constexpr int kStages = S::kStages;
  constexpr int kBK = S::kBK;
  constexpr int kKC = S::kKC;
  constexpr int kBNc = BN / CG;  // B columns staged by this CTA
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S::kBarOffset);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* aux_bar = tempty_bar + 2;
  constexpr int kEpiWarps = S::kEpiWarps;
  uint64_t* sched_full = aux_bar + 4 * kEpiWarps;
  uint64_t* sched_empty = sched_full + kSched;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sched_empty + kSched);
  int32_t* sched_tile = reinterpret_cast<int32_t*>(tmem_slot + 4);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t crank = CG == 2 ? cluster_ctarank() : 0u;
  const uint32_t rank = crank & 1u;  // position in the pair
  const int pair = static_cast<int>(crank >> 1);  // pair in the cluster (CL = 2)
  const bool leader = rank == 0;
  const int unit = static_cast<int>(blockIdx.x) / (CG * CL);
  const int units = static_cast<int>(gridDim.x) / (CG * CL);
  // tfull commits go to this pair's two CTAs; a stage is free once every pair consumed it
  const uint16_t pair_mask = static_cast<uint16_t>(3u << (2 * pair));
  const uint16_t stage_mask = CL == 2 ? static_cast<uint16_t>(0xF) : static_cast<uint16_t>(3);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    tma_prefetch_desc(&map_c);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], CL);  // one MMA commit per pair sharing the stage
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], kEpiWarps * CG);  // one arrival per epilogue warp of the pair
    }
    for (int a = 0; a < 4 * kEpiWarps; ++a) mbar_init(&aux_bar[a], 1);
    // sched_empty (used on the leader): its MMA issuer, every epilogue warp of the pair
    // and the peer's producer release an entry
    for (int i = 0; i < kSched; ++i) {
      mbar_init(&sched_full[i], 1);
      mbar_init(&sched_empty[i], 1 + CG * kEpiWarps + (CG - 1));
      sched_tile[2 * i] = -1;  // round tag of an entry never published
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if (CG == 2)
      tmem_alloc_pair<2 * BN>(tmem_slot);
    else
      tmem_alloc<2 * BN>(tmem_slot);
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // programmatic dependent launch (FSSDP_GEMM_PDL): the prologue above overlapped the
  // previous kernel's tail; nothing global is read or written before it has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");

  const GemmGroup* __restrict__ groups = args.groups;
  // total_tiles = -1: the tables were written on the device (fssdp_local_gemm_tables)
  const int total =
      (args.total_tiles >= 0
           ? args.total_tiles
           : args.groups[args.num_groups - 1].tile_start +
                 args.groups[args.num_groups - 1].m_tiles * args.n_tiles) / (CG * CL);

  const bool dyn = CL == 1 && args.sched != nullptr;
  // Tail split (args.split_tail): when the static order's last round would leave most CTA
  // pairs idle (0 < total % units <= units / 2 — e.g. cfg2's fwd2: 544 tiles on 74 pairs),
  // each of its tiles runs as two 256 x 128 halves spread over the idle pairs, so the last
  // round takes half a tile's time.  Work item i < split_from is tile i; after it, items
  // come in (half 0, half 1) pairs of one tile.
  constexpr bool kSplitOk =
      CG == 2 && CL == 1 && BN == 256 && EPI != kEpiSwiglu && EPI != kEpiDSwiglu;
  const int rem = units > 0 ? total % units : 0;
  const bool split = kSplitOk && args.split_tail != 0 && !dyn && rem > 0 && 2 * rem <= units;
  const int split_from = split ? total - rem : total;
  const int n_items = split ? total + rem : total;
  auto item_tile = [&](int item, int& half) -> int {
    if (item < split_from) {
      half = -1;
      return item;
    }
    half = (item - split_from) & 1;
    return split_from + ((item - split_from) >> 1);
  };
  // Swapped tail tiles (args.swap_tail, token-side GEMMs: A = the token rows, K-major): the
  // last M tile of a group whose real rows (GemmGroup.rows) end within its first 192 rows
  // is computed as D^T = W . X^T — M' = the tile's 256 weight columns (the pair's B halves,
  // staged in the A slots), N' = the real rows rounded up to 64 (staged in the B slots,
  // N'/2 per CTA) — so the 256-row padding of the segment costs at most 63 rows of MMA
  // work.  The epilogue stores the transposed accumulator through the same 32x32 boxes.
  constexpr bool kSwapOk = CG == 2 && CL == 1 && !A_MN && BN == 256 && kEpiWarps == 4 &&
                           (EPI == kEpiBF16 || EPI == kEpiGelu || EPI == kEpiDGelu ||
                            EPI == kEpiDSwiglu || (EPI == kEpiSwiglu && !B_MN));
  constexpr bool kWideOk = (EPI == kEpiBF16 || EPI == kEpiGelu) && kEpiWarps == 4 &&
                           S::kSets * S::kOutTiles * S::kBufBytes >= 4096 * S::kOutTiles;
  auto tail_rows = [&](const GemmGroup& g) -> int {  // N' of the group's tail, 0: none
    if (!kSwapOk || !args.swap_tail || g.rows <= 0 || g.m_tiles < CG) return 0;
    const int tail = g.rows - (g.m_tiles / CG - 1) * (CG * kBM);
    const int np = (tail + 63) / 64 * 64;
    return tail > 0 && np <= 192 ? np : 0;
  };
  auto swap_rows = [&](const TileCoord& tc, const GemmGroup& g, int half) -> int {
    if (!kSwapOk || half >= 0 || tc.m_tile != g.m_tiles / CG - 1) return 0;
    return tail_rows(g);
  };
  // Tails last (args.tail_last, static order with swapped tails): every group's full tiles
  // first (group order, N-fastest inside a group), then the groups' tail tiles, so the
  // order's last round(s) are the cheap tail tiles.  Measured 0.5 % SLOWER per step at cfg2
  // (each tail re-reads its weight tiles long after the group's other tiles), neutral at
  // cfg4: off by default (FSSDP_GEMM_TAIL_LAST=1).
  const bool tail_order = kSwapOk && args.swap_tail != 0 && args.tail_last != 0 && !dyn && !split;
  int n_tail_tiles = 0;
  if (tail_order) {  // every warp counts (all threads are here)
    int c = 0;
    for (int i = lane; i < args.num_groups; i += 32) c += tail_rows(groups[i]) > 0 ? 1 : 0;
    n_tail_tiles = __reduce_add_sync(0xffffffffu, c) * args.n_tiles;
  }
  const int total_full = total - n_tail_tiles;
  struct TailCursor {
    int g = 0, base = 0, gt = 0, tbase = 0;
  };
  // tile id -> coordinates (and N' of a swapped tile) in either order; ids increase per role
  auto locate = [&](int tl, int half, int& gcur, TailCursor& tcur, int& sw) -> TileCoord {
    if (!tail_order) {
      const TileCoord tc = locate_tile<CG, CL>(groups, args.num_groups, args.n_tiles,
                                               args.n_fast, tl, gcur, pair);
      sw = swap_rows(tc, groups[tc.group], half);
      return tc;
    }
    const int nt = args.n_tiles;
    TileCoord tc;
    if (tl < total_full) {
      for (;;) {
        const GemmGroup& gg = groups[tcur.g];
        const int ft = (gg.m_tiles / CG - (tail_rows(gg) > 0 ? 1 : 0)) * nt;
        if (tl < tcur.base + ft) break;
        tcur.base += ft;
        ++tcur.g;
      }
      const int local = tl - tcur.base;
      tc.group = tcur.g;
      tc.m_tile = local / nt;
      tc.n_tile = local % nt;
      sw = 0;
    } else {
      const int u = tl - total_full;
      for (;;) {
        const int tt = tail_rows(groups[tcur.gt]) > 0 ? nt : 0;
        if (u < tcur.tbase + tt) break;
        tcur.tbase += tt;
        ++tcur.gt;
      }
      tc.group = tcur.gt;
      tc.m_tile = groups[tcur.gt].m_tiles / CG - 1;
      tc.n_tile = u - tcur.tbase;
      sw = tail_rows(groups[tcur.gt]);
    }
    return tc;
  };
  // consumer side of the scheduler ring: entry `it` -> tile id (-1: no more work); the
  // entry is released on the leader (remote arrive from the follower CTA)
  auto sched_take = [&](int it) -> int {
    const int slot = it % kSched;
    // CTA-scope wait (a cluster-scope acquire here, in every consumer warp, cost ~3 % of
    // the step: the epilogue-heavy GEMMs slowed by 15 %), then the entry's round tag is
    // checked, so a value from another CTA is never used before it has landed
    mbar_wait(&sched_full[slot], static_cast<uint32_t>(it / kSched) & 1u);
    int2 v;
    do {
      v = ld_volatile_shared_v2(&sched_tile[2 * slot]);
    } while (v.x != it);
    const int t = v.y;
    if (CG == 2 && !leader)
      mbar_arrive_leader(&sched_empty[slot]);
    else
      mbar_arrive(&sched_empty[slot]);
    return t;
  };
  // the tile of round `it` for a role: static snake order, or the ring
  auto next_tile = [&](int it) -> int {
    if (!dyn) {
      const int t = snake_tile(it, unit, units);
      return t < n_items ? t : -1;
    }
    return sched_take(it);
  };

  if (warp == 0) {
    if (lane == 0) {
      // ===================== TMA producer (both CTAs stage their own halves)
      PROF_T0(tp0);
      int stage = 0;
      uint32_t phase = 0;
      int gcur = 0;  // group cursor (locate_tile)
      TailCursor tcur;
      // The pair's scheduler (leader producer): entry it + 1 is published while tile `it`
      // is being loaded, so the peer CTA's producer never waits for a tile id at a tile
      // boundary, and one atomic is always in flight (its round trip overlaps the loads).
      int cur = -1, pending = 0;
      bool done = !(dyn && leader);
      auto sched_exit = [&]() {  // once per pair, on its first fetch past the end
        // the last pair to run dry resets the counters for the next launch (stream order,
        // or PDL's griddepcontrol.wait, keeps the next grid behind this one)
        if (atomicAdd(args.sched + 1, 1) == units - 1) {
          atomicExch(args.sched, 0);
          atomicExch(args.sched + 1, 0);
        }
      };
      auto publish = [&](int it, int t) {
        const int slot = it % kSched;
        if (it >= kSched)
          mbar_wait(&sched_empty[slot], static_cast<uint32_t>(it / kSched - 1) & 1u);
        // entry = {round, tile}: the round tag lets a consumer verify the value it read
        st_volatile_shared_v2(&sched_tile[2 * slot], it, t);
        mbar_arrive(&sched_full[slot]);
        if (CG == 2) {
          st_cluster_v2(cluster_map(&sched_tile[2 * slot], 1u), static_cast<uint32_t>(it),
                        static_cast<uint32_t>(t));
          mbar_arrive_cluster(cluster_map(&sched_full[slot], 1u));
        }
      };
      if (!done) {
        cur = atomicAdd(args.sched, 1);
        if (cur >= total) {
          cur = -1;
          sched_exit();
        }
        publish(0, cur);
        done = cur < 0;
        if (!done) pending = atomicAdd(args.sched, 1);
      }
      for (int it = 0;; ++it) {
        int tile;
        if (dyn && leader) {
          tile = cur;
          if (!done) {
            int t = pending;
            if (t >= total) {
              t = -1;
              sched_exit();
              done = true;
            } else {
              pending = atomicAdd(args.sched, 1);
            }
            publish(it + 1, t);
            cur = t;
          }
        } else {
          tile = next_tile(it);
        }
        if (tile < 0) break;
        int half;
        const int tl = item_tile(tile, half);
        int sw;
        const TileCoord tc = locate(tl, half, gcur, tcur, sw);
        const GemmGroup& g = groups[tc.group];
        const int m0 = g.a_m + tc.m_tile * (CG * kBM) + static_cast<int>(rank) * kBM;
        // a half tile's MMA reads the first kBNc / 2 staged B rows of each CTA
        const int n0 = g.b_n + tc.n_tile * BN + (half > 0 ? BN / 2 : 0) +
                       static_cast<int>(rank) * (half >= 0 ? kBNc / 2 : kBNc);
        // swapped: this CTA's N'/2 token rows of the tile (into its B slot)
        const int sm0 = g.a_m + tc.m_tile * (CG * kBM) + static_cast<int>(rank) * (sw / 2);
        // K-major operand (rows x kBK): one 2-D load, or kKC chunks by one 3-D load
        auto kmaj = [&](uint8_t* dst, const CUtensorMap* m2, const CUtensorMap* m3, int k, int row) {
          if (kKC == 1) {
            if (CG == 2)
              tma_load_2d_pair(dst, m2, &full_bar[stage], k, row);
            else
              tma_load_2d(dst, m2, &full_bar[stage], k, row);
          } else {
            if (CG == 2)
              tma_load_3d_pair(dst, m3, &full_bar[stage], 0, row, k / 64);
            else
              tma_load_3d(dst, m3, &full_bar[stage], 0, row, k / 64);
          }
        };
        const int nkb = (g.k_blocks * 64 + kBK - 1) / kBK;
        for (int kb = 0; kb < nkb; ++kb) {
          PROF_T0(tw);
          mbar_wait(&empty_bar[stage], phase ^ 1);
          PROF_ADD(1, tw);
          uint8_t* sa = smem + stage * S::kStageBytes;
          uint8_t* sb = sa + S::kABytes;
          // swapped tail: the weights fill the A slots, only N' token rows the B slots
          if (leader)
            mbar_arrive_expect_tx(&full_bar[stage], (kSwapOk && sw > 0)
                                                        ? CG * S::kABytes + sw * kBK * 2
                                                        : CG * S::kStageBytes);
          const int ka = g.a_k + kb * kBK;
          const int kbb = g.b_k + kb * kBK;
          if (kSwapOk && sw > 0) {  // weights -> A slot, token rows -> B slot
            if (EPI == kEpiSwiglu) {
              // a1 units [rank * 64, +64) and the same a3 units: h pairs them in one CTA
              const int nu = g.b_n + tc.n_tile * BN + static_cast<int>(rank) * 64;
#pragma unroll
              for (int c = 0; c < kKC; ++c) {
                uint8_t* d = sa + c * (kBM * 128);
                tma_load_2d_pair(d, &args.map_b64, &full_bar[stage], kbb + 64 * c, nu);
                tma_load_2d_pair(d + 64 * 128, &args.map_b64, &full_bar[stage], kbb + 64 * c,
                                 nu + BN / 2);
              }
            } else if (B_MN) {
              if (args.mn3d_b) {
                tma_load_3d_pair(sa, &args.map_b3, &full_bar[stage], 0, kbb, n0 / 64);
              } else {
#pragma unroll
                for (int j = 0; j < kBNc / 64; ++j)
                  tma_load_2d_pair(sa + j * (kBK * 128), &map_b, &full_bar[stage], n0 + 64 * j, kbb);
              }
            } else {
              kmaj(sa, &map_b, &args.map_bk, kbb, n0);
            }
            for (int c = 0; c < kKC; ++c)
              for (int j = 0; j < sw / 64; ++j)  // this CTA's sw / 2 rows, 32 per box
                tma_load_2d_pair(sb + c * (sw / 2) * 128 + j * 32 * 128, &args.map_a32,
                                 &full_bar[stage], ka + 64 * c, sm0 + 32 * j);
          } else if (CG == 2) {
            if (CL == 2) {  // the first pair loads A for both: CTA r -> CTAs r and r + 2
              if (pair == 0) {
                const uint16_t mc = static_cast<uint16_t>(0x5u << rank);
                if (A_MN) {
#pragma unroll
                  for (int j = 0; j < kBM / 64; ++j)
                    tma_load_2d_pair_mc(sa + j * (kBK * 128), &map_a, &full_bar[stage],
                                        m0 + 64 * j, ka, mc);
                } else {
#pragma unroll
                  for (int c = 0; c < kKC; ++c)
                    tma_load_2d_pair_mc(sa + c * (kBM * 128), &map_a, &full_bar[stage],
                                        ka + 64 * c, m0, mc);
                }
              }
            } else if (A_MN) {
              if (args.mn3d_a) {
                tma_load_3d_pair(sa, &args.map_a3, &full_bar[stage], 0, ka, m0 / 64);
              } else {
#pragma unroll
                for (int j = 0; j < kBM / 64; ++j)
                  tma_load_2d_pair(sa + j * (kBK * 128), &map_a, &full_bar[stage], m0 + 64 * j, ka);
              }
            } else {
              kmaj(sa, &map_a, &args.map_ak, ka, m0);
            }
            if (B_MN) {
              if (args.mn3d_b && half < 0) {
                tma_load_3d_pair(sb, &args.map_b3, &full_bar[stage], 0, kbb, n0 / 64);
              } else {
#pragma unroll
                for (int j = 0; j < kBNc / 64; ++j)
                  tma_load_2d_pair(sb + j * (kBK * 128), &map_b, &full_bar[stage], n0 + 64 * j, kbb);
              }
            } else {
              kmaj(sb, &map_b, &args.map_bk, kbb, n0);
            }
          } else {
            if (A_MN) {
#pragma unroll
              for (int j = 0; j < kBM / 64; ++j)
                tma_load_2d(sa + j * (kBK * 128), &map_a, &full_bar[stage], m0 + 64 * j, ka);
            } else {
              kmaj(sa, &map_a, &args.map_ak, ka, m0);
            }
            if (B_MN) {
#pragma unroll
              for (int j = 0; j < kBNc / 64; ++j)
                tma_load_2d(sb + j * (kBK * 128), &map_b, &full_bar[stage], n0 + 64 * j, kbb);
            } else {
              kmaj(sb, &map_b, &args.map_bk, kbb, n0);
            }
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      PROF_ADD(0, tp0);
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ===================== MMA issuer (single thread of the leader CTA)
      PROF_T0(tm0);
      constexpr uint32_t idesc =
          make_idesc_bf16(CG * kBM, BN, A_MN ? 1u : 0u, B_MN ? 1u : 0u);
      constexpr uint32_t idesc_half =
          make_idesc_bf16(CG * kBM, BN / 2, A_MN ? 1u : 0u, B_MN ? 1u : 0u);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int gcur = 0;
      TailCursor tcur;
      for (int it = 0;; ++it) {
        const int item = next_tile(it);
        if (item < 0) break;
        int half;
        const int tile = item_tile(item, half);
        int sw;
        const TileCoord tc = locate(tile, half, gcur, tcur, sw);
        const int kblocks = groups[tc.group].k_blocks;
        // swapped: A' = the weights (B's majorness), B' = the token rows (K-major), N' = sw
        const uint32_t tdesc = sw > 0 ? make_idesc_bf16(CG * kBM, static_cast<uint32_t>(sw),
                                                        B_MN ? 1u : 0u, 0u)
                               : half >= 0 ? idesc_half : idesc;
        PROF_T0(te);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        PROF_ADD(3, te);
        PROF_INC(7);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
        const int nkb = (kblocks * 64 + kBK - 1) / kBK;
        for (int kb = 0; kb < nkb; ++kb) {
          PROF_T0(tf);
          mbar_wait(&full_bar[stage], phase);
          PROF_ADD(2, tf);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem + stage * S::kStageBytes);
          const uint32_t b_base = a_base + S::kABytes;
          // a K block count that is not a multiple of kKC: the last stage's extra chunk
          // (staged, possibly stale or zero) is not multiplied
          const int kk_end = min(kBK / 16, (kblocks * 64 - kb * kBK) / 16);
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            if (kk >= kk_end) break;
            // K-major: 16 K elements = 32 B inside the 128-B swizzled row, chunk kk / 4 at
            // (staged rows) * 128 B; MN-major: 16 K rows = 2048 B, MN chunks at kBK * 128 B
            const uint32_t kofs = static_cast<uint32_t>((kk & 3) * 32);
            const uint32_t kch = static_cast<uint32_t>(kk >> 2);
            uint64_t adesc, bdesc;
            if (A_MN)
              adesc = make_sdesc_sw128(a_base + kk * 2048, kBK * 128, 1024);
            else
              adesc = make_sdesc_sw128(a_base + kch * (kBM * 128) + kofs, 16, 1024);
            if (B_MN)
              bdesc = make_sdesc_sw128(b_base + kk * 2048, kBK * 128, 1024);
            else
              bdesc = make_sdesc_sw128(b_base + kch * (kBNc * 128) + kofs, 16, 1024);
            if (kSwapOk && sw > 0) {  // the A slot holds B's operand and vice versa
              adesc = B_MN ? make_sdesc_sw128(a_base + kk * 2048, kBK * 128, 1024)
                           : make_sdesc_sw128(a_base + kch * (kBM * 128) + kofs, 16, 1024);
              bdesc = make_sdesc_sw128(b_base + kch * static_cast<uint32_t>(sw / 2 * 128) + kofs,
                                       16, 1024);
            }
            if (CG == 2)
              umma_bf16_pair(d_tmem, adesc, bdesc, tdesc, (kb | kk) ? 1u : 0u);
            else
              umma_bf16(d_tmem, adesc, bdesc, tdesc, (kb | kk) ? 1u : 0u);
          }
          // frees the smem slot (in both CTAs; CL = 2: in all four) when these MMAs finish
          if (CG == 2)
            umma_commit_pair(&empty_bar[stage], stage_mask);
          else
            umma_commit(&empty_bar[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (CG == 2)  // accumulator ready for both CTAs' epilogues
          umma_commit_pair(&tfull_bar[acc], pair_mask);
        else
          umma_commit(&tfull_bar[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      PROF_ADD(4, tm0);
    }
  } else {
    // ===================== epilogue: TMEM -> registers -> fused op -> smem -> TMA store
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int ew = warp - 2;
    uint8_t* wbase = smem + S::kEpiOffset + ew * S::kEpiWarpBytes;
    uint8_t* cbuf0 = wbase;                               // output staging, 2 sets
    uint8_t* abuf0 = wbase + S::kCBufs * S::kBufBytes;    // aux ring (dgrad2)
    constexpr int kAB = S::kAuxBufs > 0 ? S::kAuxBufs : 1;
    constexpr int kAT = S::kAuxTiles;
    constexpr int kOT = S::kOutTiles;
    constexpr bool kAux = EPI == kEpiDGelu || EPI == kEpiDSwiglu;
    uint64_t* abar = aux_bar + 4 * ew;
    uint32_t aux_phase = 0;  // bit i = phase of aux entry i
    // SwiGLU drains column PAIRS (a1 chunk c, a3 chunk c + 4): BN/64 steps of 32 hidden units
    constexpr int kChunks = EPI == kEpiSwiglu ? BN / (2 * kEpiCols) : BN / kEpiCols;
    constexpr int kCW = kChunks / (kEpiWarps / 4);  // chunks drained by this warp
    const int cbase = (ew / 4) * kCW;                // warps 2-5: left half, 6-9: right half
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t gchunk = 0;  // running chunk counter (selects the staging set)
    bool wide_out = false;  // lane 0: a wide store may still be reading the staging sets
    int gcur = 0;
    TailCursor tcur;
    PROF_T0(tep0);
    // aux / output column of f-space column j in the interleaved [a1|a3] layout (SwiGLU)
    auto a13_col = [](int j) { return 256 * (j >> 7) + (j & 127); };
    for (int it = 0;; ++it) {
      int tile = 0;
      if (lane == 0) tile = next_tile(it);
      tile = __shfl_sync(0xffffffffu, tile, 0);
      if (tile < 0) break;
      int half;
      const int tl = item_tile(tile, half);
      int sw;
      const TileCoord tc = locate(tl, half, gcur, tcur, sw);
      const GemmGroup& g = groups[tc.group];
      const int row0 = static_cast<int>(g.c_off / args.ldc) + tc.m_tile * (CG * kBM) +
                       static_cast<int>(rank) * kBM + q * 32;
      const int col0 = tc.n_tile * BN + (half > 0 ? BN / 2 : 0);
      // chunks this warp drains: a half tile has kChunks / 2 (in its first TMEM columns)
      const int cw_end = half < 0 ? kCW : min(kCW, max(0, kChunks / 2 - cbase));
      const bool zero = g.k_blocks == 0;
      // wide stores (args.wide_store): BF16 / GeLU outputs leave through 32 x 64 boxes of
      // 128-byte rows — half the TMA store requests of the 32 x 32 boxes
      const bool wide = kWideOk && args.wide_store != 0 && g.c_dest == 0 && (cw_end & 1) == 0;
      // destination: C, or (c_dest > 0) a tensor map in global memory — e.g. a peer's
      // staging slot, so the store itself is the NVLink transfer
      const CUtensorMap* cmap =
          g.c_dest > 0 ? static_cast<const CUtensorMap*>(args.c_dest_maps) + (g.c_dest - 1) : &map_c;
      auto aux_load = [&](int entry, int c) {  // the aux tile(s) of chunk c into an entry
        uint8_t* dst = abuf0 + entry * kAT * S::kBufBytes;
        mbar_arrive_expect_tx(&abar[entry], kAT * S::kBufBytes);
        if (EPI == kEpiDSwiglu) {
          const int a1 = a13_col(col0 + c * kEpiCols);
          tma_load_2d(dst, &map_x, &abar[entry], a1, row0);
          tma_load_2d(dst + S::kBufBytes, &map_x, &abar[entry], a1 + 128, row0);
        } else {
          tma_load_2d(dst, &map_x, &abar[entry], col0 + c * kEpiCols, row0);
        }
      };
      if (kSwapOk && sw > 0) {
        // swapped tail tile: TMEM lane = output column wcol + lane, TMEM column = token row;
        // each 32-row chunk is staged transposed ([row][col] as the normal path) and stored
        // through the same 32x32 boxes
        const int wcol = tc.n_tile * BN + static_cast<int>(rank) * kBNc + q * 32;
        const int trow = static_cast<int>(g.c_off / args.ldc) + tc.m_tile * (CG * kBM);
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
        const int nch = sw / 32;
        if constexpr (EPI == kEpiSwiglu) {
          // TMEM lanes 0-63: a1 of units u1 + 0..63, lanes 64-127: a3 of the same units
          // (u1 = the tile's first unit + rank * 64); warp q < 2 holds a1 of units
          // u1 + 32 q + lane, warp q + 2 their a3.  Per 32-row chunk the a3 warp hands its
          // fp32 values to the a1 warp through shared memory (double-buffered by chunk
          // parity, one 64-thread named barrier per chunk), which computes h as the normal
          // path does; each warp stores its own a1 / a3 box, the a1 warps the h box.
          const int u = tc.n_tile * (BN / 2) + static_cast<int>(rank) * 64 + (q & 1) * 32;
          const int ocol = a13_col(u) + (q >= 2 ? BN / 2 : 0);
          const int trow = static_cast<int>(g.c_off / args.ldc) + tc.m_tile * (CG * kBM);
          // staging: the a1 warps 2 tiles per set (a1, h), the a3 warps 1 (a3), which leaves
          // 8 KB of the a3 warp's region for the exchange buffers
          static_assert(S::kEpiWarpBytes >= 6 * S::kBufBytes, "SwiGLU swap: staging space");
          float* xch = reinterpret_cast<float*>(smem + S::kEpiOffset + (q & 1) * S::kEpiWarpBytes +
                                                2 * S::kBufBytes);
          const int ot = q < 2 ? 2 : 1;
          // the staging layout differs from the normal path's: no older store may still read
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
#pragma unroll 1
          for (int ci = 0; ci < nch; ++ci, ++gchunk) {
            const int b = static_cast<int>(gchunk % S::kSets);
            uint32_t r[32];
            tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                                   static_cast<uint32_t>(acc * BN + ci * 32),
                               r);
            tmem_ld_wait();
            if (ci == nch - 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) {
                if (!leader)
                  mbar_arrive_leader(&tempty_bar[acc]);
                else
                  mbar_arrive(&tempty_bar[acc]);
              }
            }
            float* xb = xch + (ci & 1) * 1024;  // [32 rows][32 units] fp32
            if (q >= 2) {
#pragma unroll
              for (int j = 0; j < 32; ++j) xb[j * 32 + lane] = __uint_as_float(r[j]);
            }
            asm volatile("bar.sync %0, 64;" ::"r"(1 + (q & 1)) : "memory");
            if (lane == 0) bulk_wait_read<S::kSets - 1>();
            __syncwarp();
            uint8_t* cb = cbuf0 + b * ot * S::kBufBytes;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float a = __uint_as_float(r[j]);
              const uint32_t o = static_cast<uint32_t>(sw64(j, lane >> 3)) + (lane & 7) * 2;
              *reinterpret_cast<__nv_bfloat16*>(cb + o) = __float2bfloat16_rn(a);
              if (q < 2) {  // h = silu(a1) a3 from the fp32 accumulators
                const float a3 = xb[j * 32 + lane];
                *reinterpret_cast<__nv_bfloat16*>(cb + S::kBufBytes + o) =
                    __float2bfloat16_rn(__fdividef(a, 1.f + __expf(-a)) * a3);
              }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(cmap, cb, ocol, trow + ci * 32);
              if (q < 2) tma_store_2d(&map_x, cb + S::kBufBytes, u, trow + ci * 32);
              bulk_commit();
            }
          }
          // back to the normal layout: this tile's stores have read their staging, and the
          // a1 warp is done with the exchange buffers before the a3 warp reuses its region
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
          asm volatile("bar.sync %0, 64;" ::"r"(1 + (q & 1)) : "memory");
          if (++acc == 2) {
            acc = 0;
            acc_phase ^= 1;
          }
          continue;
        }
#pragma unroll 1
        for (int ci = 0; ci < nch; ++ci, ++gchunk) {
          const int b = static_cast<int>(gchunk % S::kSets);
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                                 static_cast<uint32_t>(acc * BN + ci * 32),
                             r);
          tmem_ld_wait();
          if (ci == nch - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if (!leader)
                mbar_arrive_leader(&tempty_bar[acc]);
              else
                mbar_arrive(&tempty_bar[acc]);
            }
          }
          float pre[32], pre3[32];
          if (kAux) {  // the saved gelu' (dSwiGLU: a1 and a3) box of these rows / columns
            const int entry = static_cast<int>(gchunk % kAB);
            uint8_t* ab = abuf0 + entry * kAT * S::kBufBytes;
            if (lane == 0) {
              fence_proxy_async_smem();
              mbar_arrive_expect_tx(&abar[entry], kAT * S::kBufBytes);
              if (EPI == kEpiDSwiglu) {
                const int a1c = a13_col(wcol);
                tma_load_2d(ab, &map_x, &abar[entry], a1c, trow + ci * 32);
                tma_load_2d(ab + S::kBufBytes, &map_x, &abar[entry], a1c + 128, trow + ci * 32);
              } else {
                tma_load_2d(ab, &map_x, &abar[entry], wcol, trow + ci * 32);
              }
            }
            mbar_wait(&abar[entry], (aux_phase >> entry) & 1u);
            aux_phase ^= 1u << entry;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const uint32_t o = static_cast<uint32_t>(sw64(j, lane >> 3)) + (lane & 7) * 2;
              pre[j] = __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(ab + o));
              if (EPI == kEpiDSwiglu)
                pre3[j] = __bfloat162float(
                    *reinterpret_cast<const __nv_bfloat16*>(ab + S::kBufBytes + o));
            }
          }
          if (lane == 0) {
            if (wide_out)
              bulk_wait_read<0>();
            else
              bulk_wait_read<S::kSets - 1>();
          }
          wide_out = false;
          __syncwarp();
          uint8_t* cb = cbuf0 + b * kOT * S::kBufBytes;
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float a0 = __uint_as_float(r[j]), a1 = __uint_as_float(r[j + 1]);
            __nv_bfloat162 o, act;
            if (EPI == kEpiGelu) {
              uint64_t g2, d2;
              gelu_and_grad2(f2_pack(a0, a1), g2, d2);
              const float2 gf = f2_unpack(g2), df = f2_unpack(d2);
              act = __floats2bfloat162_rn(gf.x, gf.y);
              o = __floats2bfloat162_rn(df.x, df.y);
            } else if (EPI == kEpiDGelu) {
              const float2 v = f2_unpack(f2_mul(f2_pack(a0, a1), f2_pack(pre[j], pre[j + 1])));
              o = __floats2bfloat162_rn(v.x, v.y);
            } else if (EPI == kEpiDSwiglu) {  // o = d1, act = d3 of rows j, j + 1
              float d1a, d3a, d1b, d3b;
              dswiglu1(a0, pre[j], pre3[j], d1a, d3a);
              dswiglu1(a1, pre[j + 1], pre3[j + 1], d1b, d3b);
              o = __floats2bfloat162_rn(d1a, d1b);
              act = __floats2bfloat162_rn(d3a, d3b);
            } else {
              o = __floats2bfloat162_rn(a0, a1);
            }
            const uint32_t o0 = static_cast<uint32_t>(sw64(j, lane >> 3)) + (lane & 7) * 2;
            const uint32_t o1 = static_cast<uint32_t>(sw64(j + 1, lane >> 3)) + (lane & 7) * 2;
            *reinterpret_cast<__nv_bfloat16*>(cb + o0) = o.x;
            *reinterpret_cast<__nv_bfloat16*>(cb + o1) = o.y;
            if (EPI == kEpiGelu || EPI == kEpiDSwiglu) {
              *reinterpret_cast<__nv_bfloat16*>(cb + S::kBufBytes + o0) = act.x;
              *reinterpret_cast<__nv_bfloat16*>(cb + S::kBufBytes + o1) = act.y;
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (EPI == kEpiDSwiglu) {  // da1, da3 columns of the interleaved [a1 | a3] layout
              const int a1c = a13_col(wcol);
              tma_store_2d(cmap, cb, a1c, trow + ci * 32);
              tma_store_2d(cmap, cb + S::kBufBytes, a1c + 128, trow + ci * 32);
            } else {
              tma_store_2d(cmap, cb, wcol, trow + ci * 32);
              if (EPI == kEpiGelu) tma_store_2d(&map_x, cb + S::kBufBytes, wcol, trow + ci * 32);
            }
            bulk_commit();
          }
        }
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
        continue;
      }
      if (kAux && lane == 0) {  // prefetch the first aux tiles of this tile
        fence_proxy_async_smem();
        for (int p = 0; p < kAB - 1 && p < cw_end; ++p) aux_load((gchunk + p) % kAB, cbase + p);
      }
      PROF_T0(ta);
      mbar_wait(&tfull_bar[acc], acc_phase);
      if (ew == 0 && lane == 0) PROF_ADD(5, ta);
      tc_fence_after();
      if (cw_end == 0) {  // nothing of this half tile to drain: release TMEM right away
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (CG == 2 && !leader)
            mbar_arrive_leader(&tempty_bar[acc]);
          else
            mbar_arrive(&tempty_bar[acc]);
        }
      }
#pragma unroll 1
      for (int ci = 0; ci < cw_end; ++ci, ++gchunk) {
        const int c = cbase + ci;
        const int b = static_cast<int>(gchunk % S::kSets);
        uint32_t r[32], r3[32];
        const uint32_t tm = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                            static_cast<uint32_t>(acc * BN + c * kEpiCols);
        if (!zero) {
          tmem_ld_32x32b_x32(tm, r);
          if (EPI == kEpiSwiglu) tmem_ld_32x32b_x32(tm + BN / 2, r3);  // the a3 half
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = r3[i] = 0u;
        }
        if (ci == cw_end - 1) {  // this warp's share of the accumulator read: release TMEM
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (CG == 2 && !leader)
              mbar_arrive_leader(&tempty_bar[acc]);
            else
              mbar_arrive(&tempty_bar[acc]);
          }
        }
        __nv_bfloat162 pre[16], pre3[16];
        if (kAux) {
          if (lane == 0 && ci + kAB - 1 < cw_end) {  // keep kAB-1 aux entries in flight
            fence_proxy_async_smem();
            aux_load((gchunk + kAB - 1) % kAB, c + kAB - 1);
          }
          const int cur = gchunk % kAB;
          mbar_wait(&abar[cur], (aux_phase >> cur) & 1u);
          aux_phase ^= 1u << cur;
          const uint8_t* ab = abuf0 + cur * kAT * S::kBufBytes;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            *reinterpret_cast<int4*>(&pre[4 * j]) =
                *reinterpret_cast<const int4*>(ab + sw64(lane, j));
            if (EPI == kEpiDSwiglu)
              *reinterpret_cast<int4*>(&pre3[4 * j]) =
                  *reinterpret_cast<const int4*>(ab + S::kBufBytes + sw64(lane, j));
          }
        }
        // the staging set b was last used kSets chunks ago: its TMA stores must have read it
        // (wide stores: one 32 x 64 buffer per output, waited for below, after the math)
        if (!wide) {
          if (lane == 0) {
            if (wide_out)  // a wide store (spanning both sets) may still be reading
              bulk_wait_read<0>();
            else
              bulk_wait_read<S::kSets - 1>();
          }
          wide_out = false;
          __syncwarp();
        }
        uint8_t* cb = cbuf0 + b * kOT * S::kBufBytes;
        auto stage_bf16 = [&](uint8_t* dst, const __nv_bfloat162 (&v)[16]) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<int4*>(dst + sw64(lane, j)) = *reinterpret_cast<const int4*>(&v[4 * j]);
        };
#ifdef FSSDP_EXP_EPI_NOSTS  // experiment: accumulators read, nothing staged or stored
        if (true) {
          if (r[0] == 0x7fc00001u && lane == 0) cb[0] = 1;  // keep the TMEM load live
          continue;
        }
#endif
        if (EPI == kEpiF32) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<int4*>(cb + sw128(lane, j)) =
                make_int4(static_cast<int>(r[4 * j]), static_cast<int>(r[4 * j + 1]),
                          static_cast<int>(r[4 * j + 2]), static_cast<int>(r[4 * j + 3]));
        } else if (EPI == kEpiSwiglu) {
          __nv_bfloat162 o1[16], o3[16], oh[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 a1 = make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
            const float2 a3 = make_float2(__uint_as_float(r3[2 * i]), __uint_as_float(r3[2 * i + 1]));
            o1[i] = __floats2bfloat162_rn(a1.x, a1.y);
            o3[i] = __floats2bfloat162_rn(a3.x, a3.y);
            // h = silu(a1) a3 from the fp32 accumulators
            oh[i] = __floats2bfloat162_rn(__fdividef(a1.x, 1.f + __expf(-a1.x)) * a3.x,
                                          __fdividef(a1.y, 1.f + __expf(-a1.y)) * a3.y);
          }
          stage_bf16(cb, o1);
          stage_bf16(cb + S::kBufBytes, o3);
          stage_bf16(cb + 2 * S::kBufBytes, oh);
        } else if (EPI == kEpiDSwiglu) {
          __nv_bfloat162 d1[16], d3[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {  // dH (fp32) with the saved bf16 a1, a3
            const float2 a1 = __bfloat1622float2(pre[i]), a3 = __bfloat1622float2(pre3[i]);
            float d1a, d3a, d1b, d3b;
            dswiglu1(__uint_as_float(r[2 * i]), a1.x, a3.x, d1a, d3a);
            dswiglu1(__uint_as_float(r[2 * i + 1]), a1.y, a3.y, d1b, d3b);
            d1[i] = __floats2bfloat162_rn(d1a, d1b);
            d3[i] = __floats2bfloat162_rn(d3a, d3b);
          }
          stage_bf16(cb, d1);
          stage_bf16(cb + S::kBufBytes, d3);
        } else {
          __nv_bfloat162 out[16], act[16];
          if (EPI == kEpiBF16) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              out[i] = __floats2bfloat162_rn(__uint_as_float(r[2 * i]),
                                             __uint_as_float(r[2 * i + 1]));
          } else if (EPI == kEpiGelu) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {  // one tanh feeds both GeLU and GeLU'
              uint64_t g2, d2;
              gelu_and_grad2(f2_pack(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])),
                             g2, d2);
              const float2 gf = f2_unpack(g2), df = f2_unpack(d2);
              act[i] = __floats2bfloat162_rn(gf.x, gf.y);
              out[i] = __floats2bfloat162_rn(df.x, df.y);
            }
          } else {  // kEpiDGelu: out = acc * gelu'(pre-activation), gelu' saved by fwd1
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float2 p = __bfloat1622float2(pre[i]);
              const float2 o = f2_unpack(f2_mul(
                  f2_pack(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])),
                  f2_pack(p.x, p.y)));
              out[i] = __floats2bfloat162_rn(o.x, o.y);
            }
          }
          if (wide) {
            // chunk pair (2 p, 2 p + 1) fills one 128-byte-row box per output: its first
            // chunk waits until the previous pair's stores have read the buffers
            if ((ci & 1) == 0) {
              if (lane == 0) bulk_wait_read<0>();
              __syncwarp();
            }
            const int h = (ci & 1) * 4;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              *reinterpret_cast<int4*>(cbuf0 + sw128(lane, h + j)) =
                  *reinterpret_cast<const int4*>(&out[4 * j]);
              if (EPI == kEpiGelu)
                *reinterpret_cast<int4*>(cbuf0 + 2 * S::kBufBytes + sw128(lane, h + j)) =
                    *reinterpret_cast<const int4*>(&act[4 * j]);
            }
          } else {
            if (EPI == kEpiGelu) stage_bf16(cb + S::kBufBytes, act);
            stage_bf16(cb, out);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
#ifdef FSSDP_EXP_EPI_NOSTORE  // experiment: staged in shared memory, never stored
        if (true) continue;
#endif
        if (lane == 0) {
          if (EPI == kEpiSwiglu) {
            const int j = col0 + c * kEpiCols;  // a1 column in the interleaved 2f layout
            tma_store_2d(cmap, cb, j, row0);
            tma_store_2d(cmap, cb + S::kBufBytes, j + BN / 2, row0);
            tma_store_2d(&map_x, cb + 2 * S::kBufBytes, col0 / 2 + c * kEpiCols, row0);
          } else if (EPI == kEpiDSwiglu) {
            const int a1 = a13_col(col0 + c * kEpiCols);
            tma_store_2d(cmap, cb, a1, row0);
            tma_store_2d(cmap, cb + S::kBufBytes, a1 + 128, row0);
          } else if (wide) {
            wide_out = true;
            if (ci & 1) {
              tma_store_2d(&args.map_c64, cbuf0, col0 + (c - 1) * kEpiCols, row0);
              if (EPI == kEpiGelu)
                tma_store_2d(&args.map_x64, cbuf0 + 2 * S::kBufBytes, col0 + (c - 1) * kEpiCols,
                             row0);
            }
          } else {
            tma_store_2d(cmap, cb, col0 + c * kEpiCols, row0);
            if (EPI == kEpiGelu)
              tma_store_2d(&map_x, cb + S::kBufBytes, col0 + c * kEpiCols, row0);
          }
          bulk_commit();
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait<0>();  // all stores of this warp complete before exit
    __syncwarp();
    if (ew == 0 && lane == 0) PROF_ADD(6, tep0);
  }

  tc_fence_before();
  if (CG == 2)
    cluster_sync();  // the peer's smem / barriers stay alive until the pair is done
  else
    __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (warp == 1) {
    tc_fence_after();
    if (CG == 2)
      tmem_dealloc_pair<2 * BN>(tmem_base);
    else
      tmem_dealloc<2 * BN>(tmem_base);
  }
}

// ------------------------------------------------------------------ host side

template <bool A_MN, bool B_MN, int BN, int EPI, int CGX>
static int launch_variant(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
                          const CUtensorMap& mx, const GemmLaunch& args, cudaStream_t stream) {
  constexpr int CG = CGX == 4 ? 2 : CGX;
  auto kern = grouped_gemm_kernel<A_MN, B_MN, BN, EPI, CGX>;
  const int smem =
      GemmSmem<BN, EPI, CG, k_block(A_MN, B_MN, EPI, CG), epi_warps<EPI, A_MN && B_MN>()>::kDynamic;
  if (ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem) != cudaSuccess)
    return kErrCuda;
  // work units: tiles of CG*128 rows (CGX = 4: pairs of N tiles); a device-side total (-1)
  // gets the full persistent grid.  Clusters of 4 need 4 SMs of one GPC each: the grid is
  // what fits co-resident (cudaOccupancyMaxActiveClusters, once per device).
  int max_units = num_sms() / CGX;
  if (CGX == 4) {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (cached[dev & 63] == 0) {
      cudaLaunchConfig_t oc = {};
      oc.gridDim = dim3(num_sms());
      oc.blockDim = dim3(gemm_threads<EPI, A_MN && B_MN>());
      oc.dynamicSmemBytes = smem;
      cudaLaunchAttribute ca[1];
      ca[0].id = cudaLaunchAttributeClusterDimension;
      ca[0].val.clusterDim.x = 4;
      ca[0].val.clusterDim.y = 1;
      ca[0].val.clusterDim.z = 1;
      oc.attrs = ca;
      oc.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, reinterpret_cast<const void*>(kern), &oc) !=
              cudaSuccess ||
          n <= 0)
        n = num_sms() / 4;
      cached[dev & 63] = n;
    }
    max_units = cached[dev & 63];
  }
  const int units = args.total_tiles >= 0 ? args.total_tiles / CGX : num_sms();
  int grid = CGX * (units < max_units ? units : max_units);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(gemm_threads<EPI, A_MN && B_MN>());
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  static const bool pdl = [] {
    const char* v = getenv("FSSDP_GEMM_PDL");  // default on; "0" disables
    return v == nullptr || v[0] != '0';
  }();
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CGX;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // programmatic dependent launch: this GEMM's CTAs may start their prologue while the
  // previous kernel in the stream drains (the kernel waits before touching memory);
  // interleaved A/B: N=2 1.678 -> 1.666 ms, N=1 e2e +1 %, N=1 device time unchanged
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  timing_begin(stream);
  const cudaError_t launched = cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, mx, args);
  timing_end();
  if (launched != cudaSuccess) return kErrCuda;
  return cudaGetLastError() == cudaSuccess ? kOk : kErrCuda;
}

// Instantiated (A major, B major, epilogue) combinations.  BN = 256: every combination
// the tests use; BN = 128 only the layer's own (N = d_ff not a multiple of 256).
template <bool A_MN, bool B_MN, int BN, int CG>
static int dispatch_epi(int epi, const CUtensorMap& ma, const CUtensorMap& mb,
                        const CUtensorMap& mc, const CUtensorMap& mx, const GemmLaunch& args,
                        cudaStream_t stream) {
  constexpr bool kFull = BN == 256;
  switch (epi) {
    case kEpiBF16:
      if constexpr (kFull || !A_MN)
        return launch_variant<A_MN, B_MN, BN, kEpiBF16, CG>(ma, mb, mc, mx, args, stream);
      break;
    case kEpiGelu:
      if constexpr (kFull || (!A_MN && !B_MN))
        return launch_variant<A_MN, B_MN, BN, kEpiGelu, CG>(ma, mb, mc, mx, args, stream);
      break;
    case kEpiDGelu:
      if constexpr (kFull || (!A_MN && B_MN))
        return launch_variant<A_MN, B_MN, BN, kEpiDGelu, CG>(ma, mb, mc, mx, args, stream);
      break;
    case kEpiF32:  // BN 128: the weight gradients (MN / MN) and the tensor-core gate logits
      if constexpr (kFull || (A_MN == B_MN))
        return launch_variant<A_MN, B_MN, BN, kEpiF32, CG>(ma, mb, mc, mx, args, stream);
      break;
    case kEpiSwiglu:
      if constexpr (kFull && !A_MN && !B_MN)
        return launch_variant<A_MN, B_MN, BN, kEpiSwiglu, CG>(ma, mb, mc, mx, args, stream);
      break;
    case kEpiDSwiglu:
      if constexpr (!A_MN && B_MN)
        return launch_variant<A_MN, B_MN, BN, kEpiDSwiglu, CG>(ma, mb, mc, mx, args, stream);
      break;
    default:
      break;
  }
  set_error("grouped_gemm: operand majors / epilogue / N tile combination not instantiated");
  return kErrDimension;
}

template <int BN, int CG>
static int dispatch_major(int a_mn, int b_mn, int epi, const CUtensorMap& ma,
                          const CUtensorMap& mb, const CUtensorMap& mc, const CUtensorMap& mx,
                          const GemmLaunch& args, cudaStream_t stream) {
  if (a_mn) {
    if (b_mn) return dispatch_epi<true, true, BN, CG>(epi, ma, mb, mc, mx, args, stream);
    return dispatch_epi<true, false, BN, CG>(epi, ma, mb, mc, mx, args, stream);
  }
  if (b_mn) return dispatch_epi<false, true, BN, CG>(epi, ma, mb, mc, mx, args, stream);
  return dispatch_epi<false, false, BN, CG>(epi, ma, mb, mc, mx, args, stream);
}

// epilogue tiles: 32 x 32, bf16 rows of 64 B (SWIZZLE_64B) or fp32 rows of 128 B
int epilogue_tmap(int epi, const void* base, int64_t ldc, int64_t rows, CUtensorMap* map) {
  if (ldc % 32 != 0 || rows <= 0 || base == nullptr) return kErrDimension;
  if (epi == kEpiF32) return make_tmap_2d(map, base, ldc, rows, kEpiCols, 32, kDtF32, 128);
  return make_tmap_2d(map, base, ldc, rows, kEpiCols, 32, kDtBF16, 64);
}

int grouped_gemm_launch(int a_mn, int b_mn, int epi, const void* a, int64_t a_inner,
                        int64_t a_outer, const void* b, int64_t b_inner, int64_t b_outer,
                        int64_t c_rows, const GemmLaunch& args, cudaStream_t stream) {
  const int BN = args.bn == 128 ? 128 : 256;
  if (args.total_tiles == 0) return kOk;
  if (args.ldc % 32 != 0) return kErrDimension;
  const int cg = args.cta_group == 4 ? 4 : args.cta_group == 2 ? 2 : 1;
  if (cg == 4 && (BN != 256 || !args.n_fast || args.n_tiles % 2 != 0 || args.sched != nullptr))
    return kErrDimension;  // A multicast: N-fastest pairs of 256-wide N tiles, static order
  CUtensorMap ma, mb, mc, mx;
  // K-major operand: box = {64 K elems, rows};  MN-major: box = {64 MN elems, 64 K rows}
  // MN-major 2-D boxes: {64 MN, kBK K rows}
  const int kBK = k_block(a_mn != 0, b_mn != 0, epi, cg), kKC = kBK / 64;
  int rc = make_tmap_2d(&ma, a, a_inner, a_outer, 64, a_mn ? kBK : kBM, kDtBF16, 128);
  if (rc != kOk) return rc;
  GemmLaunch la = args;
  if (kKC == 2 && !a_mn) {  // K-major A: kBM rows x 2 K chunks per load
    rc = make_tmap_3d(&la.map_ak, a, a_inner, a_outer, kBM, kKC);
    if (rc != kOk) return rc;
  }
  if (la.swap_tail && !a_mn) {  // 32-row boxes: a swapped tail stages only its rows
    rc = make_tmap_2d(&la.map_a32, a, a_inner, a_outer, 64, 32, kDtBF16, 128);
    if (rc != kOk) return rc;
  }
  rc = make_tmap_2d(&mb, b, b_inner, b_outer, 64, b_mn ? kBK : BN / (cg == 4 ? 2 : cg), kDtBF16, 128);
  if (rc != kOk) return rc;
  if (kKC == 2 && !b_mn) {
    rc = make_tmap_3d(&la.map_bk, b, b_inner, b_outer, BN / (cg == 4 ? 2 : cg), kKC);
    if (rc != kOk) return rc;
  }
  // MN-major operands (the wgrads' A and B, the dgrads' weights) staged by ONE 3-D load
  // per stage instead of one 2-D load per 64-wide chunk: half the TMA requests of those
  // operands — cfg2 step -1.3 % (wgrad1 -3.5 %, wgrad2 -4 %), cfg4 -1.5 % (interleaved
  // A/B).  CTA pairs with at least two chunks per operand tile; FSSDP_GEMM_MN3D=0 disables
  static const int mn3d = [] {
    const char* v = getenv("FSSDP_GEMM_MN3D");
    return v == nullptr || v[0] != '0' ? 1 : 0;
  }();
  if (mn3d && cg == 2) {
    if (a_mn && a_inner % 64 == 0) {
      rc = make_tmap_3d(&la.map_a3, a, a_inner, a_outer, kBK, kBM / 64);
      if (rc != kOk) return rc;
      la.mn3d_a = 1;
    }
    if (b_mn && BN / 2 >= 128 && b_inner % 64 == 0) {
      rc = make_tmap_3d(&la.map_b3, b, b_inner, b_outer, kBK, (BN / 2) / 64);
      if (rc != kOk) return rc;
      la.mn3d_b = 1;
    }
  }
  if (la.swap_tail && epi == kEpiSwiglu && !b_mn) {  // 64-row boxes: a1 / a3 unit halves
    rc = make_tmap_2d(&la.map_b64, b, b_inner, b_outer, 64, 64, kDtBF16, 128);
    if (rc != kOk) return rc;
  }
  rc = epilogue_tmap(epi, args.c, args.ldc, c_rows, &mc);
  if (rc != kOk) return rc;
  // second tensor: GeLU's post-activation (same shape as C), SwiGLU's h (half the width of
  // C), dgrad2's saved aux (same shape as C), else unused (C again)
  const void* xptr = (epi == kEpiGelu || epi == kEpiSwiglu) ? args.c2
                     : (epi == kEpiDGelu || epi == kEpiDSwiglu) ? args.aux : args.c;
  const int64_t xld = epi == kEpiSwiglu ? args.ldc / 2 : args.ldc;
  rc = make_tmap_2d(&mx, xptr, xld, c_rows, kEpiCols, 32, epi == kEpiF32 ? kDtF32 : kDtBF16,
                    epi == kEpiF32 ? 128 : 64);
  if (rc != kOk) return rc;
  // wide stores: the GeLU epilogue by default (fwd1 standalone -2 %, cfg2 step -0.3 %,
  // interleaved A/B); FSSDP_GEMM_WIDE_STORE=0 never, =2 also the BF16 epilogue (neutral
  // standalone, 0.5 % slower per cfg4 step)
  static const int wide = [] {
    const char* v = getenv("FSSDP_GEMM_WIDE_STORE");
    return v == nullptr ? 1 : v[0] - '0';
  }();
  if (((wide >= 1 && epi == kEpiGelu) || (wide >= 2 && epi == kEpiBF16)) && args.ldc % 64 == 0) {
    rc = make_tmap_2d(&la.map_c64, args.c, args.ldc, c_rows, 2 * kEpiCols, 32, kDtBF16, 128);
    if (rc != kOk) return rc;
    if (epi == kEpiGelu) {
      rc = make_tmap_2d(&la.map_x64, args.c2, args.ldc, c_rows, 2 * kEpiCols, 32, kDtBF16, 128);
      if (rc != kOk) return rc;
    }
    la.wide_store = 1;
  }
  if (BN == 128) {
    if (cg == 2) return dispatch_major<128, 2>(a_mn, b_mn, epi, ma, mb, mc, mx, la, stream);
    return dispatch_major<128, 1>(a_mn, b_mn, epi, ma, mb, mc, mx, la, stream);
  }
  if (cg == 4) return dispatch_major<256, 4>(a_mn, b_mn, epi, ma, mb, mc, mx, la, stream);
  if (cg == 2) return dispatch_major<256, 2>(a_mn, b_mn, epi, ma, mb, mc, mx, la, stream);
  return dispatch_major<256, 1>(a_mn, b_mn, epi, ma, mb, mc, mx, la, stream);
}

#ifdef FSSDP_GEMM_PROFILE
extern "C" __attribute__((visibility("default"))) int fssdp_gemm_profile_read(
    unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_gemm_prof, sizeof(g_gemm_prof)) != cudaSuccess) return -4;
  if (reset) {
    static unsigned long long zeros[1024][8];
    if (cudaMemcpyToSymbol(g_gemm_prof, zeros, sizeof(zeros)) != cudaSuccess) return -4;
  }
  return 0;
}
#endif

}  // namespace fssdp
