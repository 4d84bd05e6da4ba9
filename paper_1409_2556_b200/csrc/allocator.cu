// Device block cache behind lt::DeviceBuffer (see lt_internal.hpp).
//
// Blocks are keyed by (stream, rounded size).  A freed block goes to its stream's free list
// and the next request of that size on that stream takes it back: safe without events since
// every later use is stream-ordered after every earlier one.  Misses go to the stream-ordered
// pool (cudaMallocAsync); an out-of-memory returns every cached block to the pool (in stream
// order) and retries once.
#include <atomic>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "lt_internal.hpp"

namespace lt {
namespace {

struct Key {
  cudaStream_t s;
  size_t bytes;
  bool operator==(const Key& o) const { return s == o.s && bytes == o.bytes; }
};
struct KeyHash {
  size_t operator()(const Key& k) const {
    return std::hash<const void*>()(k.s) ^ (std::hash<size_t>()(k.bytes) * 0x9e3779b97f4a7c15ull);
  }
};

struct Cache {
  std::mutex mu;
  std::unordered_map<Key, std::vector<void*>, KeyHash> free_blocks;
  size_t cached_bytes = 0;
};

Cache& cache() {
  static Cache* c = new Cache;  // never destroyed: DeviceBuffers may outlive static teardown
  return *c;
}

size_t round_size(size_t bytes) {
  const size_t g = bytes >= (size_t(1) << 20) ? (size_t(2) << 20) : size_t(512);
  return (bytes + g - 1) / g * g;
}

// return cached blocks (all streams, or one) to the pool; caller holds the lock
std::atomic<uint64_t>& driver_epoch() {
  static std::atomic<uint64_t> e{0};
  return e;
}

void drain_locked(Cache& c, const cudaStream_t* only) {
  driver_epoch().fetch_add(1, std::memory_order_relaxed);
  for (auto it = c.free_blocks.begin(); it != c.free_blocks.end();) {
    if (only && it->first.s != *only) {
      ++it;
      continue;
    }
    for (void* p : it->second) {
      cudaFreeAsync(p, it->first.s);
      c.cached_bytes -= it->first.bytes;
    }
    it = c.free_blocks.erase(it);
  }
}

}  // namespace

uint64_t cache_driver_epoch() { return driver_epoch().load(std::memory_order_relaxed); }

void* cache_alloc(size_t bytes, cudaStream_t s) {
  const size_t rb = round_size(bytes);
  Cache& c = cache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.free_blocks.find(Key{s, rb});
    if (it != c.free_blocks.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      c.cached_bytes -= rb;
      return p;
    }
  }
  void* p = nullptr;
  driver_epoch().fetch_add(1, std::memory_order_relaxed);  // the driver's free-memory figure changes
  cudaError_t e = cudaMallocAsync(&p, rb, s);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    {
      std::lock_guard<std::mutex> lk(c.mu);
      drain_locked(c, nullptr);
    }
    // the drained blocks are free in stream order on their own streams; make them available
    cudaDeviceSynchronize();
    e = cudaMallocAsync(&p, rb, s);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(e == cudaErrorMemoryAllocation ? LT_ERR_OOM : LT_ERR_CUDA,
                std::string("device allocation of ") + std::to_string(rb) + " bytes failed: " + cudaGetErrorString(e));
  }
  return p;
}

void cache_free(void* p, size_t bytes, cudaStream_t s) {
  if (!p) return;
  const size_t rb = round_size(bytes);
  Cache& c = cache();
  std::lock_guard<std::mutex> lk(c.mu);
  c.free_blocks[Key{s, rb}].push_back(p);
  c.cached_bytes += rb;
}

size_t cache_cached_bytes() {
  Cache& c = cache();
  std::lock_guard<std::mutex> lk(c.mu);
  return c.cached_bytes;
}

void cache_release_stream(cudaStream_t s) {
  Cache& c = cache();
  std::lock_guard<std::mutex> lk(c.mu);
  drain_locked(c, &s);
}

}  // namespace lt
