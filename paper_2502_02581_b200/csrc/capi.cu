// C-ABI plumbing of libfssdp: error reporting, device queries, TMA descriptor encoding,
// the grouped-GEMM entry point, and the symmetric heap (cudaMalloc + CUDA IPC).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <utility>

#include "fssdp_internal.h"

namespace fssdp {

static thread_local std::string g_last_error;

void set_error(const char* msg) { g_last_error = msg ? msg : ""; }

LaunchTiming& launch_timing() {
  static thread_local LaunchTiming t;
  return t;
}

cudaError_t ensure_dynamic_smem(const void* func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> opted;  // (func, device) -> bytes
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  std::lock_guard<std::mutex> lock(mu);
  int& have = opted[std::make_pair(func, dev)];
  if (have >= bytes) return cudaSuccess;
  err = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (err == cudaSuccess) have = bytes;
  return err;
}

int num_sms() {
  static int cached = -1;
  if (cached < 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      return 148;
    cached = n;
  }
  return cached;
}

// cuTensorMapEncodeTiled is fetched through the runtime's driver entry point so the
// library never links libcuda directly (it must load on GPU-less build hosts).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// Encoded tensor maps are cached by their arguments: the layer launches the same few
// GEMM operand / output maps every step, and an encode costs microseconds of host time on
// the launch path.  (A map only holds the address and extents, never the data.)
struct TmapKey {
  const void* base;
  int64_t inner, outer;
  int box_inner, box_outer, dtype, swizzle;
  bool operator<(const TmapKey& o) const {
    return std::tie(base, inner, outer, box_inner, box_outer, dtype, swizzle) <
           std::tie(o.base, o.inner, o.outer, o.box_inner, o.box_outer, o.dtype, o.swizzle);
  }
};
static int make_tmap_2d_uncached(CUtensorMap* map, const void* base, int64_t inner, int64_t outer,
                                 int box_inner, int box_outer, int dtype, int swizzle_bytes);

int make_tmap_2d(CUtensorMap* map, const void* base, int64_t inner, int64_t outer, int box_inner,
                 int box_outer, int dtype, int swizzle_bytes) {
  static std::mutex mu;
  static std::map<TmapKey, CUtensorMap> cache;
  const TmapKey key{base, inner, outer, box_inner, box_outer, dtype, swizzle_bytes};
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *map = it->second;
      return kOk;
    }
  }
  const int rc = make_tmap_2d_uncached(map, base, inner, outer, box_inner, box_outer, dtype,
                                       swizzle_bytes);
  if (rc == kOk) {
    std::lock_guard<std::mutex> lock(mu);
    if (cache.size() > 4096) cache.clear();  // bound it (buffers come and go in tests)
    cache[key] = *map;
  }
  return rc;
}

int make_tmap_mn3d(CUtensorMap* map, const void* base, int64_t inner, int64_t outer, int nchunks) {
  return make_tmap_3d(map, base, inner, outer, 64, nchunks);
}

int make_tmap_3d(CUtensorMap* map, const void* base, int64_t inner, int64_t outer, int box_rows,
                 int nchunks) {
  static std::mutex mu;
  static std::map<TmapKey, CUtensorMap> cache;
  const TmapKey key{base, inner, outer, -nchunks, box_rows, kDtBF16, 128};
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *map = it->second;
      return kOk;
    }
  }
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return kErrCuda;
  }
  if (inner <= 0 || outer <= 0 || inner % 64 != 0 || nchunks <= 0 ||
      (reinterpret_cast<uintptr_t>(base) & 15) != 0) {
    set_error("tensor map (3-D): bad extents or misaligned base");
    return kErrDimension;
  }
  cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(outer), static_cast<cuuint64_t>(inner / 64)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(inner * 2), 128};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(nchunks)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[128];
    snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled (3-D) failed (%d)", static_cast<int>(r));
    set_error(buf);
    return kErrCuda;
  }
  std::lock_guard<std::mutex> lock(mu);
  if (cache.size() > 4096) cache.clear();
  cache[key] = *map;
  return kOk;
}

static int make_tmap_2d_uncached(CUtensorMap* map, const void* base, int64_t inner, int64_t outer,
                                 int box_inner, int box_outer, int dtype, int swizzle_bytes) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return kErrCuda;
  }
  const int esize = dtype == kDtF32 ? 4 : 2;
  if (inner <= 0 || outer <= 0 || (inner * esize) % 16 != 0 ||
      (reinterpret_cast<uintptr_t>(base) & 15) != 0) {
    set_error("tensor map: bad extents or misaligned base");
    return kErrDimension;
  }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(inner * esize)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                      : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = fn(map,
                  dtype == kDtF32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                  2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[128];
    snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
    set_error(buf);
    return kErrCuda;
  }
  return kOk;
}

}  // namespace fssdp

using namespace fssdp;

extern "C" {

const char* fssdp_version(void) { return "fssdp-b200 0.1.0 (sm_100a)"; }

const char* fssdp_last_error(void) { return g_last_error.c_str(); }

int fssdp_num_sms(void) { return num_sms(); }

int fssdp_event_create(void** event_out) {
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) {
    set_error("event_create: cudaEventCreate failed");
    return kErrCuda;
  }
  *event_out = e;
  return kOk;
}

int fssdp_event_destroy(void* event) {
  return cudaEventDestroy(static_cast<cudaEvent_t>(event)) == cudaSuccess ? kOk : kErrCuda;
}

int fssdp_event_record(void* event, void* stream) {
  return cudaEventRecord(static_cast<cudaEvent_t>(event), static_cast<cudaStream_t>(stream)) ==
                 cudaSuccess
             ? kOk
             : kErrCuda;
}

int fssdp_event_elapsed(void* start, void* end, float* ms_out) {
  if (cudaEventElapsedTime(ms_out, static_cast<cudaEvent_t>(start),
                           static_cast<cudaEvent_t>(end)) != cudaSuccess) {
    set_error("event_elapsed: events not both completed");
    return kErrCuda;
  }
  return kOk;
}

int fssdp_timing_arm(void* start, void* end) {
  LaunchTiming& t = launch_timing();
  t.start = static_cast<cudaEvent_t>(start);
  t.end = static_cast<cudaEvent_t>(end);
  t.state = start && end ? 1 : 0;
  return kOk;
}

int fssdp_timing_done(void) {
  LaunchTiming& t = launch_timing();
  timing_end();  // an entry point that returned between its launches
  const int fired = t.state == 3;
  t.state = 0;
  return fired;
}

int fssdp_plan_layer_tables(int32_t num_experts, const int32_t* base_owner, const double* est,
                            const int32_t* counts, const fssdp_topology* topo,
                            const fssdp_layer_knobs* knobs, int32_t rank, const uint8_t* pre_mask,
                            int32_t d_model, int32_t d_ff, int32_t n_mats, const int64_t* limits,
                            uint8_t* target_out, int32_t* added_out, int64_t* route_out,
                            double* doubles_out, int32_t* flags_out, uint8_t* blob,
                            int64_t blob_bytes, int32_t* header_out, void* blob_dev, void* stream) {
  if (topo == nullptr || counts == nullptr || num_experts <= 0) {
    set_error("plan_layer_tables: bad arguments");
    return kErrDimension;
  }
  const int64_t D = static_cast<int64_t>(topo->nodes) * topo->devices_per_node;
  int64_t actual[64 * 64];  // D <= kMaxWorld (32), E <= 64
  if (D <= 0 || D * num_experts > 64 * 64) {
    set_error("plan_layer_tables: too many devices x experts");
    return kErrDimension;
  }
  for (int64_t i = 0; i < D * num_experts; ++i) actual[i] = counts[i];
  int rc = fssdp_plan_layer(num_experts, base_owner, est, actual, topo, knobs, target_out,
                            added_out, route_out, doubles_out, flags_out);
  if (rc != kOk) return rc;
  // limits[3] >= 0: a model-level parameter region {owned_base, replica_base} (limits[3..4])
  const bool split = limits != nullptr && limits[3] >= 0;
  rc = fssdp_build_rank_tables(rank, static_cast<int32_t>(D), num_experts, base_owner, target_out,
                               pre_mask, route_out, d_model, d_ff, n_mats,
                               split ? limits + 3 : nullptr, blob, blob_bytes, header_out);
  if (rc != kOk) return rc;
  if (limits != nullptr) {  // header: [0] slots, [2] receive rows, [28] staging slots
    // split layout: [0] is the owned-slot capacity, limits[5] the replica-slot capacity
    const int64_t need[4] = {split ? header_out[1] : header_out[0], header_out[2], header_out[28],
                             split ? header_out[0] - header_out[1] : 0};
    static const char* what[4] = {"expert slots", "receive rows", "staging slots",
                                  "replica slots"};
    for (int i = 0; i < (split ? 4 : 3); ++i)
      if (need[i] > limits[i == 3 ? 5 : i]) {
        char msg[160];
        snprintf(msg, sizeof(msg), "plan needs %lld %s > capacity %lld", (long long)need[i],
                 what[i], (long long)limits[i == 3 ? 5 : i]);
        set_error(msg);
        return FSSDP_ERR_INFEASIBLE;
      }
  }
  if (blob_dev == nullptr) return rc;
  int64_t offs[FSSDP_TAB_NSECTIONS], total = 0;
  fssdp_tables_layout(num_experts, static_cast<int32_t>(D), offs, &total);
  // SM-driven pull from the pinned blob: not queued behind the caller's bulk H2D copies
  return fssdp_pull_host(blob_dev, blob, (total + 15) / 16 * 16, stream);
}

int fssdp_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && (dst == nullptr || src == nullptr))) {
    set_error("copy_async: bad arguments");
    return kErrDimension;
  }
  if (bytes == 0) return kOk;
  return cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault,
                         static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? kOk
             : kErrCuda;
}

int fssdp_plan_layer_dispatch(const uint32_t* counts_flag, uint32_t counts_epoch,
                              double timeout_s, int32_t num_experts, const int32_t* base_owner,
                              const double* est, const int32_t* counts,
                              const fssdp_topology* topo, const fssdp_layer_knobs* knobs,
                              int32_t rank, const uint8_t* pre_mask, int32_t d_model,
                              int32_t d_ff, int32_t n_mats, const int64_t* limits,
                              uint8_t* target_out, int32_t* added_out, int64_t* route_out,
                              double* doubles_out, int32_t* flags_out, uint8_t* blob,
                              int64_t blob_bytes, int32_t* header_out, void* blob_dev,
                              void* stream, const fssdp_dispatch_launch* disp) {
  int rc = fssdp_host_wait(counts_flag, counts_epoch, timeout_s);
  if (rc != kOk) return rc;
  rc = fssdp_plan_layer_tables(num_experts, base_owner, est, counts, topo, knobs, rank, pre_mask,
                               d_model, d_ff, n_mats, limits, target_out, added_out, route_out,
                               doubles_out, flags_out, blob, blob_bytes, header_out, blob_dev,
                               stream);
  if (rc != kOk || disp == nullptr || blob_dev == nullptr) return rc;
  const int32_t D = topo->nodes * topo->devices_per_node;
  int64_t offs[FSSDP_TAB_NSECTIONS], total = 0;
  fssdp_tables_layout(num_experts, D, offs, &total);
  uint8_t* dev = static_cast<uint8_t*>(blob_dev);
  auto sec = [&](int i) { return reinterpret_cast<int32_t*>(dev + offs[i]); };
  return fssdp_dispatch(disp->x, disp->topk_idx, disp->slot_rank, disp->tile_prefix, disp->T,
                        disp->d_model, disp->E, disp->k, disp->world, sec(FSSDP_TAB_ROUTE_CUM),
                        sec(FSSDP_TAB_RECV_BASE), disp->slot_dest, disp->slot_pos,
                        disp->peer_bases, disp->recv_off, sec(FSSDP_TAB_ZERO_ROWS),
                        header_out[3], disp->flags_off, disp->rank, disp->bar_slot, disp->epoch,
                        disp->grid_counter, stream);
}


int fssdp_grouped_gemm(int32_t a_mn, int32_t b_mn, int32_t epilogue, const void* a, int64_t a_inner,
                       int64_t a_outer, const void* b, int64_t b_inner, int64_t b_outer,
                       const fssdp_gemm_group* groups_dev, int32_t num_groups, int32_t n_tiles,
                       int32_t total_tiles, void* c, void* c2, const void* aux,
                       const void* c_dest_maps, int64_t ldc, int64_t c_rows, int32_t flags,
                       int32_t* tile_sched, void* stream) {
  if (num_groups <= 0 || n_tiles <= 0 || total_tiles < -1 || c == nullptr || c_rows <= 0) {
    set_error("grouped_gemm: bad arguments");
    return kErrDimension;
  }
  if (((epilogue == kEpiGelu || epilogue == kEpiSwiglu) && c2 == nullptr) ||
      ((epilogue == kEpiDGelu || epilogue == kEpiDSwiglu) && aux == nullptr) || epilogue < 0 ||
      epilogue > kEpiDSwiglu) {
    set_error("grouped_gemm: epilogue needs c2/aux");
    return kErrDimension;
  }
  GemmLaunch args = {};
  args.groups = groups_dev;
  args.num_groups = num_groups;
  args.n_tiles = n_tiles;
  args.total_tiles = total_tiles;
  args.n_fast = (flags & FSSDP_GEMM_N_FASTEST) ? 1 : 0;
  args.cta_group = (flags & FSSDP_GEMM_CTA_PAIR) ? 2 : 1;
  args.split_tail = (flags & FSSDP_GEMM_SPLIT_TAIL) ? 1 : 0;
  args.swap_tail = (flags & FSSDP_GEMM_SWAP_TAIL) ? 1 : 0;
  static const int tail_last = [] {  // experiment: swapped tails after every full tile
    const char* v = getenv("FSSDP_GEMM_TAIL_LAST");
    return v != nullptr && v[0] == '1' ? 1 : 0;
  }();
  args.tail_last = tail_last;
  if (flags & FSSDP_GEMM_MULTICAST) {
    if (args.cta_group != 2 || !(flags & FSSDP_GEMM_N_FASTEST) || (flags & FSSDP_GEMM_BN128) ||
        n_tiles % 2 != 0 || tile_sched != nullptr) {
      set_error("grouped_gemm: MULTICAST needs CTA_PAIR, N_FASTEST, 256-wide N tiles, an even "
                "n_tiles and the static order");
      return kErrDimension;
    }
    args.cta_group = 4;
  }
  args.bn = (flags & FSSDP_GEMM_BN128) ? 128 : 256;
  if (args.bn == 128 && epilogue == kEpiSwiglu) {
    set_error("grouped_gemm: the SwiGLU epilogue needs 256-wide N tiles");
    return kErrDimension;
  }
  args.ldc = ldc;
  args.c = c;
  args.c2 = c2;
  args.aux = static_cast<const __nv_bfloat16*>(aux);
  args.c_dest_maps = c_dest_maps;
  args.sched = tile_sched;
  int rc = grouped_gemm_launch(a_mn, b_mn, epilogue, a, a_inner, a_outer, b, b_inner, b_outer,
                               c_rows, args, reinterpret_cast<cudaStream_t>(stream));
  if (rc == kErrCuda && g_last_error.empty()) set_error("grouped_gemm launch failed");
  return rc;
}

int fssdp_epilogue_tmap(int32_t epilogue, const void* base, int64_t ldc, int64_t rows,
                        void* map_out) {
  if (epilogue < kEpiBF16 || epilogue > kEpiF32 || map_out == nullptr) {
    set_error("epilogue_tmap: bad arguments");
    return kErrDimension;
  }
  CUtensorMap m;
  const int rc = epilogue_tmap(epilogue, base, ldc, rows, &m);
  if (rc != kOk) {
    if (g_last_error.empty()) set_error("epilogue_tmap: cannot encode the tensor map");
    return rc;
  }
  memcpy(map_out, &m, sizeof(m));
  return kOk;
}

int fssdp_heap_alloc(size_t bytes, void** ptr_out) {
  const size_t gran = size_t(2) << 20;
  bytes = (bytes + gran - 1) / gran * gran;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return kErrCuda;
  }
  e = cudaMemset(p, 0, bytes);
  if (e != cudaSuccess) {
    cudaFree(p);
    set_error(cudaGetErrorString(e));
    return kErrCuda;
  }
  *ptr_out = p;
  return kOk;
}

int fssdp_heap_free(void* ptr) {
  cudaError_t e = cudaFree(ptr);
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return kErrCuda;
  }
  return kOk;
}

int fssdp_ipc_handle(void* ptr, uint8_t* handle_out) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return kErrCuda;
  }
  memcpy(handle_out, &h, sizeof(h));
  return kOk;
}

int fssdp_ipc_open(const uint8_t* handle, void** ptr_out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return kErrCuda;
  }
  return kOk;
}

int fssdp_ipc_close(void* ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return kErrCuda;
  }
  return kOk;
}

}  // extern "C"
