// Internal declarations shared by the CUDA translation units of libfssdp.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fssdp.h"

namespace fssdp {

constexpr int kOk = FSSDP_OK;
constexpr int kErrDimension = FSSDP_ERR_DIMENSION;
constexpr int kErrInvalidPair = FSSDP_ERR_INVALID_PAIR;
constexpr int kErrOrphan = FSSDP_ERR_ORPHAN_EXPERT;
constexpr int kErrCuda = FSSDP_ERR_CUDA;
constexpr int kErrInternal = FSSDP_ERR_INTERNAL;
constexpr int kErrInfeasible = FSSDP_ERR_INFEASIBLE;
constexpr int kErrEmptyHistory = FSSDP_ERR_EMPTY_HISTORY;

// GEMM epilogue kinds (mirrors FSSDP_EPI_* in fssdp.h)
constexpr int kEpiBF16 = FSSDP_EPI_BF16;
constexpr int kEpiGelu = FSSDP_EPI_GELU;
constexpr int kEpiDGelu = FSSDP_EPI_DGELU;
constexpr int kEpiF32 = FSSDP_EPI_F32;
constexpr int kEpiSwiglu = FSSDP_EPI_SWIGLU;
constexpr int kEpiDSwiglu = FSSDP_EPI_DSWIGLU;

using GemmGroup = fssdp_gemm_group;

struct GemmLaunch {
  const GemmGroup* groups;  // device array
  int num_groups;
  int n_tiles;      // BN tiles along N (same for every group)
  int total_tiles;  // sum over groups of m_tiles * n_tiles
  int n_fast;       // tile order: 1 = N fastest (share A in L2), 0 = M fastest (share B)
  int cta_group;    // 2 = CTA-pair 256x256 tiles (every group's m_tiles even), 1 = 128x256
  int bn;           // N tile: 256, or 128 (FSSDP_GEMM_BN128)
  int64_t ldc;      // elements per C row
  void* c;          // output (bf16 or fp32)
  void* c2;         // second output (GeLU: post-activation)
  const __nv_bfloat16* aux;  // DGeLU: pre-activation, same layout as c
  const void* c_dest_maps;   // device CUtensorMap[] for groups with c_dest > 0 (nullable)
  int* sched;                // device int32[2] tile / exit counters, zero (nullable: static order)
  int split_tail;            // static order: a short last round runs as 256 x 128 half tiles
  int swap_tail;             // a group's short last M tile as a swapped-operand tile
  int tail_last;             // swap_tail: the tail tiles after every full tile (experiment)
  CUtensorMap map_a32;       // swap_tail: A with 32-row boxes (only the tail's rows staged)
  int wide_store;            // BF16 / GeLU epilogues: 32 x 64 store boxes (128-byte rows)
  CUtensorMap map_c64;       // wide_store: C with 32 x 64 boxes (SWIZZLE_128B)
  CUtensorMap map_x64;       // wide_store, GeLU: the second output, same boxes
  CUtensorMap map_b64;       // swap_tail, SwiGLU: B with 64-row boxes (a1 / a3 unit halves)
  int mn3d_a, mn3d_b;        // MN-major A / B staged by one 3-D load per stage (map_a3/b3)
  CUtensorMap map_a3, map_b3;
  CUtensorMap map_ak, map_bk;  // FSSDP_GEMM_BK = 128: K-major A / B, 2 K chunks per load
};

int num_sms();
void set_error(const char* msg);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) raised to at least `bytes` for `func` on
// the CURRENT device (the attribute is per device), at most once per (func, device, size):
// thread-safe, and cheap on the launch path after the first call.
cudaError_t ensure_dynamic_smem(const void* func, int bytes);

// Launch timing windows (fssdp_timing_arm): the events a caller armed are recorded right
// around the next entry point's kernel launches — after its host-side setup — so the
// window holds no host time even when the GPU is waiting for the launch.
struct LaunchTiming {
  cudaEvent_t start = nullptr, end = nullptr;
  cudaStream_t stream = nullptr;
  int state = 0;  // 0 idle, 1 armed, 2 start recorded, 3 both recorded
};
LaunchTiming& launch_timing();  // per host thread
inline void timing_begin(cudaStream_t s) {
  LaunchTiming& t = launch_timing();
  if (t.state == 1) {
    cudaEventRecord(t.start, s);
    t.stream = s;
    t.state = 2;
  }
}
inline void timing_end() {
  LaunchTiming& t = launch_timing();
  if (t.state == 2) {
    cudaEventRecord(t.end, t.stream);
    t.state = 3;
  }
}
constexpr int kDtBF16 = 0;
constexpr int kDtF32 = 1;
int epilogue_tmap(int epi, const void* base, int64_t ldc, int64_t rows, CUtensorMap* map);
// MN-major bf16 operand [outer][inner] as {64, outer, inner / 64}: box {64, 64, nchunks},
// SWIZZLE_128B — the smem image of nchunks consecutive 64 x 64 2-D boxes
int make_tmap_mn3d(CUtensorMap* map, const void* base, int64_t inner, int64_t outer, int nchunks);
// the same with box {64, box_rows, nchunks}: a K-major operand's kBK = 64 * nchunks K block
// (chunks of 64 K elements, each box_rows rows of 128 B), or an MN-major one's 128 K rows
int make_tmap_3d(CUtensorMap* map, const void* base, int64_t inner, int64_t outer, int box_rows,
                 int nchunks);
int make_tmap_2d(CUtensorMap* map, const void* base, int64_t inner, int64_t outer, int box_inner,
                 int box_outer, int dtype, int swizzle_bytes);
int grouped_gemm_launch(int a_mn, int b_mn, int epi, const void* a, int64_t a_inner,
                        int64_t a_outer, const void* b, int64_t b_inner, int64_t b_outer,
                        int64_t c_rows, const GemmLaunch& args, cudaStream_t stream);

}  // namespace fssdp
