// Context: device, stream, launch accounting and per-kernel-class CUDA-event timing.
#include <algorithm>
#include <cstring>

#include "lt_internal.hpp"

cudaEvent_t lt_ctx_s::take_event() {
  if (!event_pool.empty()) {
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  LT_CUDA(cudaEventCreate(&e));
  return e;
}

void lt_ctx_s::resolve_completed() {
  size_t done = 0;
  for (; done < pending.size(); ++done) {
    if (cudaEventQuery(pending[done].stop) != cudaSuccess) break;
    auto& pe = pending[done];
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pe.start, pe.stop);
    auto& e = profile[pe.name];
    e.ms += ms;
    e.launches += 1;
    e.bytes += pe.bytes;
    event_pool.push_back(pe.start);
    event_pool.push_back(pe.stop);
  }
  cudaGetLastError();  // cudaErrorNotReady from the query is not an error
  if (done) pending.erase(pending.begin(), pending.begin() + done);
}

void lt_ctx_s::resolve_profile() {
  if (pending.empty()) return;
  LT_CUDA(cudaEventSynchronize(pending.back().stop));
  for (auto& pe : pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pe.start, pe.stop);
    auto& e = profile[pe.name];
    e.ms += ms;
    e.launches += 1;
    e.bytes += pe.bytes;
    event_pool.push_back(pe.start);
    event_pool.push_back(pe.stop);
  }
  pending.clear();
}

cusolverDnHandle_t lt_ctx_s::solver_handle() {
  if (!solver) {
    if (cusolverDnCreate(&solver) != CUSOLVER_STATUS_SUCCESS) throw lt::Error(LT_ERR_CUDA, "cusolverDnCreate failed");
    cusolverDnSetStream(solver, stream);
  }
  return solver;
}

FlagSlot* lt_ctx_s::flag_ring_dev() {
  if (!flag_host) {
    void* hp = nullptr;
    LT_CUDA(cudaHostAlloc(&hp, sizeof(FlagSlot) * kFlagRing, cudaHostAllocMapped));
    flag_host = static_cast<FlagSlot*>(hp);
    for (int i = 0; i < kFlagRing; ++i) flag_host[i] = FlagSlot{0.0, -1, 0};
    void* dp = nullptr;
    LT_CUDA(cudaHostGetDevicePointer(&dp, hp, 0));
    flag_dev = static_cast<FlagSlot*>(dp);
    for (int i = 0; i < kFlagRing; ++i) LT_CUDA(cudaEventCreateWithFlags(&flag_ev[i], cudaEventDisableTiming));
  }
  return flag_dev;
}

namespace lt {
double available_device_bytes(lt_ctx ctx) {
  // device free memory + what the stream-ordered pool holds reserved but unused + the block
  // cache: freed buffers stay reserved, so cudaMemGetInfo alone would shrink chunk sizes (and
  // the batching efficiency) as a run goes on; a request the cache cannot serve drains it
  // cudaMemGetInfo costs ~1 ms on a 180 GB device and this runs before every inner solve with
  // the stream drained: the driver-side figure is cached until this library's allocator next
  // goes to the driver, an outer solve starts (ctx->mem_probe_valid reset) or 2 s pass
  const auto now = std::chrono::steady_clock::now();
  if (ctx->mem_probe_valid && ctx->mem_probe_epoch == cache_driver_epoch() &&
      std::chrono::duration<double>(now - ctx->mem_probe_t).count() < 2.0)
    return ctx->mem_probe + (double)cache_cached_bytes();
  size_t free_b = 0, total_b = 0;
  LT_CUDA(cudaMemGetInfo(&free_b, &total_b));
  cudaMemPool_t pool;
  uint64_t reserved = 0, used = 0;
  if (cudaDeviceGetDefaultMemPool(&pool, ctx->device) == cudaSuccess) {
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
  }
  cudaGetLastError();
  ctx->mem_probe = (double)free_b + (double)(reserved > used ? reserved - used : 0);
  ctx->mem_probe_epoch = cache_driver_epoch();
  ctx->mem_probe_t = now;
  ctx->mem_probe_valid = true;
  return ctx->mem_probe + (double)cache_cached_bytes();
}

lt_ctx ctx_create(int device) {
  int count = 0;
  LT_CUDA(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) throw Error(LT_ERR_INVALID_ARGUMENT, "lt_ctx_create: bad device index");
  LT_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  LT_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10) throw Error(LT_ERR_CUDA, "lt_ctx_create: this library is built for sm_100a (B200)");
  auto* ctx = new lt_ctx_s();
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  LT_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  // Keep freed stream-ordered memory in the pool (repeated solves reuse it).
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t threshold = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
  }
  return ctx;
}

void ctx_destroy(lt_ctx ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& pe : ctx->pending) {
    cudaEventDestroy(pe.start);
    cudaEventDestroy(pe.stop);
  }
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  if (ctx->solver) cusolverDnDestroy(ctx->solver);
  if (ctx->flag_host) {
    for (auto e : ctx->flag_ev) cudaEventDestroy(e);
    cudaFreeHost(ctx->flag_host);
  }
  cache_release_stream(ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}
}  // namespace lt
