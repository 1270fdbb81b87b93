// Expert-shard optimizer and the owner-update epochs of the FSSDP training loop.
//
//   adam_kernel           AdamW on an owner's shards: fp32 master / m / v in the symmetric
//                         heap (they move with re-shards: params + 6x state = the 7x
//                         expert_bytes the reference prices, engine.py:233, 444-453), bf16
//                         working copy rewritten from the master; fp32 or bf16 gradients.
//                         HBM-bound: 30 B/param (fp32 grads), 28 (bf16).
//   publish_epoch_kernel  an owner announces "my shards are final for forward #e"
//   wait_epochs_kernel    a reader (the early SpAG's copy-engine stream) waits until every
//                         owner announced forward #e before it pulls their shards
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fssdp_internal.h"
#include "ptx.cuh"

namespace fssdp {

namespace {

constexpr int kAdamThreads = 256;
constexpr int kFlagWorld = 32;  // flag pad row width (kMaxWorld of moe_kernels.cu)

template <bool BF16G>
__global__ void __launch_bounds__(kAdamThreads)
    adam_kernel(__nv_bfloat16* __restrict__ params, float* __restrict__ master,
                float* __restrict__ m1, float* __restrict__ m2, const void* __restrict__ grads,
                int64_t n4, float lr, float beta1, float beta2, float eps, float weight_decay,
                float bc1, float bc2) {
  float4* w4 = reinterpret_cast<float4*>(master);
  float4* a4 = reinterpret_cast<float4*>(m1);
  float4* b4 = reinterpret_cast<float4*>(m2);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 g;
    if (BF16G) {  // 4 bf16 gradients: the high halves of their fp32 bit patterns
      const uint2 raw = reinterpret_cast<const uint2*>(grads)[i];
      g = make_float4(__uint_as_float(raw.x << 16), __uint_as_float(raw.x & 0xffff0000u),
                      __uint_as_float(raw.y << 16), __uint_as_float(raw.y & 0xffff0000u));
    } else {
      g = reinterpret_cast<const float4*>(grads)[i];
    }
    float4 w = w4[i], a = a4[i], b = b4[i];
    float gv[4] = {g.x, g.y, g.z, g.w}, wv[4] = {w.x, w.y, w.z, w.w};
    float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      av[q] = beta1 * av[q] + (1.f - beta1) * gv[q];
      bv[q] = beta2 * bv[q] + (1.f - beta2) * gv[q] * gv[q];
      const float mh = av[q] / bc1, vh = bv[q] / bc2;
      wv[q] = wv[q] - lr * weight_decay * wv[q];          // decoupled weight decay
      wv[q] = wv[q] - lr * mh / (sqrtf(vh) + eps);
    }
    w4[i] = make_float4(wv[0], wv[1], wv[2], wv[3]);
    a4[i] = make_float4(av[0], av[1], av[2], av[3]);
    b4[i] = make_float4(bv[0], bv[1], bv[2], bv[3]);
    if (params != nullptr) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(wv[0], wv[1]);
      __nv_bfloat162 hi = __floats2bfloat162_rn(wv[2], wv[3]);
      uint2 packed;
      packed.x = *reinterpret_cast<uint32_t*>(&lo);
      packed.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(params)[i] = packed;
    }
  }
}

__device__ __forceinline__ uint32_t* epoch_flag(const uint64_t* peer_bases, int r,
                                                int64_t flags_off, int slot) {
  return reinterpret_cast<uint32_t*>(peer_bases[r] + flags_off) + slot * kFlagWorld + r;
}

__global__ void publish_epoch_kernel(const uint64_t* __restrict__ peer_bases, int64_t flags_off,
                                     int slot, int rank, uint32_t epoch) {
  // every earlier write of this stream (the optimizer step) is complete and visible first
  __threadfence_system();
  st_release_sys(epoch_flag(peer_bases, rank, flags_off, slot), epoch);
}

__global__ void wait_epochs_kernel(const uint64_t* __restrict__ peer_bases, int64_t flags_off,
                                   int slot, int world, uint32_t epoch) {
  const int lane = threadIdx.x;
  if (lane < world) {
    const uint32_t* f = epoch_flag(peer_bases, lane, flags_off, slot);
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (static_cast<int32_t>(ld_acquire_sys(f) - epoch) < 0) {
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > 30ull * 1000000000ull) __trap();  // an owner that never publishes
    }
  }
  __syncwarp();
}

int status_of(cudaError_t launched) {
  if (launched != cudaSuccess) {
    set_error(cudaGetErrorString(launched));
    return kErrCuda;
  }
  return kOk;
}

}  // namespace
}  // namespace fssdp

using namespace fssdp;

extern "C" {

int fssdp_adam_step(void* params_bf16, float* master, float* exp_avg, float* exp_avg_sq,
                    const void* grads, int32_t grads_bf16, int64_t n, float lr, float beta1,
                    float beta2, float eps, float weight_decay, int64_t step, void* stream) {
  if (n < 0 || n % 4 != 0 || step < 1) {
    set_error("adam_step: n must be a non-negative multiple of 4 and step >= 1");
    return kErrDimension;
  }
  if (n == 0) return kOk;
  const float bc1 = 1.f - powf(beta1, static_cast<float>(step));
  const float bc2 = 1.f - powf(beta2, static_cast<float>(step));
  const int64_t n4 = n / 4;
  int64_t blocks = (n4 + kAdamThreads - 1) / kAdamThreads;
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
  if (blocks > cap) blocks = cap;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  timing_begin(s);
  auto kern = grads_bf16 ? adam_kernel<true> : adam_kernel<false>;
  kern<<<static_cast<unsigned>(blocks), kAdamThreads, 0, s>>>(
      static_cast<__nv_bfloat16*>(params_bf16), master, exp_avg, exp_avg_sq, grads, n4, lr, beta1,
      beta2, eps, weight_decay, bc1, bc2);
  timing_end();
  return status_of(cudaGetLastError());
}

int fssdp_publish_epoch(const uint64_t* peer_bases, int64_t flags_off, int32_t slot, int32_t rank,
                        uint32_t epoch, void* stream) {
  if (rank < 0 || rank >= kFlagWorld || slot < 0) {
    set_error("publish_epoch: bad rank/slot");
    return kErrDimension;
  }
  publish_epoch_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(peer_bases, flags_off,
                                                                           slot, rank, epoch);
  return status_of(cudaGetLastError());
}

int fssdp_wait_epochs(const uint64_t* peer_bases, int64_t flags_off, int32_t slot, int32_t world,
                      uint32_t epoch, void* stream) {
  if (world <= 0 || world > kFlagWorld || slot < 0) {
    set_error("wait_epochs: bad world/slot");
    return kErrDimension;
  }
  wait_epochs_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(peer_bases, flags_off,
                                                                         slot, world, epoch);
  return status_of(cudaGetLastError());
}

}  // extern "C"
