// Shared runtime pieces: status/exception plumbing, the context, device buffers.
#pragma once

#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/skr.h"

namespace skr {

// Internal exceptions carry an skr_status; the C-ABI layer converts them.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(int code, const std::string& msg) { throw Error(code, msg); }

#define SKR_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      ::skr::raise(e_ == cudaErrorMemoryAllocation ? SKR_ENOMEM : SKR_ECUDA,            \
                   std::string(#call) + ": " + cudaGetErrorString(e_));                 \
  } while (0)

#define SKR_SOLVER(call)                                                                \
  do {                                                                                  \
    cusolverStatus_t s_ = (call);                                                       \
    if (s_ != CUSOLVER_STATUS_SUCCESS)                                                  \
      ::skr::raise(SKR_ECUDA, std::string(#call) + ": cusolver status " + std::to_string((int)s_)); \
  } while (0)

// NCCL is resolved at run time (dlopen) the first time a distributed context
// is created: it reuses a libnccl.so.2 already in the process (torch's), so
// loading this library never pins a different NCCL than the host framework's.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
inline NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h && getenv("SKR_NCCL_PATH")) h = dlopen(getenv("SKR_NCCL_PATH"), RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
      api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
      api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
      api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
      api.Broadcast = (decltype(api.Broadcast))dlsym(h, "ncclBroadcast");
      api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
      api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
      api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    }
  }
  return api;
}

#define SKR_NCCL(call)                                                                  \
  do {                                                                                  \
    if (!::skr::nccl().AllReduce) ::skr::raise(SKR_ENCCL, "libnccl.so.2 not available"); \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess)                                                              \
      ::skr::raise(SKR_ENCCL, std::string(#call) + ": " + ::skr::nccl().GetErrorString(r_)); \
  } while (0)

// Check the last launch and count it (gpu_launches evidence in bench.py).
#define SKR_LAUNCHED(ctx)                                                               \
  do {                                                                                  \
    SKR_CUDA(cudaGetLastError());                                                       \
    (ctx)->launches++;                                                                  \
  } while (0)

// Buffers of >= 1 GiB bypass the stream-ordered pool: growing the pool maps
// memory at ~17 GB/s on B200 (3.8 s for 64 GiB) while cudaMalloc maps 64 GiB in
// ~5 ms (profiles/alloc_probe.py).  A direct buffer is released after an
// explicit synchronisation of its stream (every queued use on it has finished),
// so it can be handed to any stream afterwards; big buffers are never freed
// inside a graph capture (they outlive the graphs).
//
// Released direct buffers are parked per device and handed back to the next
// request of the same size (the Lanczos products' T / split operands, X~ of a
// rebuilt problem, the packed rows of the inner loop): cudaFree of a multi-GiB
// mapping stalls the host for up to ~90 ms at irregular times
// (profiles/lanczos_variance.py: c3 sketch 0.145 s of device work took
// 0.15-0.38 s of wall time).  The park holds at most big_park_cap() bytes per
// device (oldest out first) and is emptied when any allocation runs out of
// memory (the request is retried once), by skr_ctx_trim and by skr_ctx_destroy.
constexpr size_t kDirectAllocBytes = size_t(1) << 30;
inline size_t big_park_cap() {  // bytes parked per device at most (SKR_PARK_GIB, default 80; 0: no park)
  static const size_t cap = [] {
    const char* e = getenv("SKR_PARK_GIB");
    return (size_t)(e ? std::max(0, atoi(e)) : 80) << 30;
  }();
  return cap;
}
struct BigPark {
  struct Block { int dev; size_t bytes; void* p; };
  std::mutex mu;
  std::vector<Block> blocks;  // oldest first
  static BigPark& get() {
    static BigPark* park = new BigPark;  // never destroyed: no CUDA calls from static destructors
    return *park;
  }
  static int device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
  }
  void* take(size_t bytes) {
    const int dev = device();
    std::lock_guard<std::mutex> g(mu);
    for (size_t i = blocks.size(); i-- > 0;)
      if (blocks[i].dev == dev && blocks[i].bytes == bytes) {
        void* p = blocks[i].p;
        blocks.erase(blocks.begin() + i);
        return p;
      }
    return nullptr;
  }
  void put(void* p, size_t bytes) {
    const int dev = device();
    std::vector<void*> drop;
    {
      std::lock_guard<std::mutex> g(mu);
      if (bytes > big_park_cap()) {
        drop.push_back(p);
      } else {
        blocks.push_back({dev, bytes, p});
        size_t held = 0;
        for (const Block& b : blocks) held += b.dev == dev ? b.bytes : 0;
        for (size_t i = 0; i < blocks.size() && held > big_park_cap();)
          if (blocks[i].dev == dev) {
            held -= blocks[i].bytes;
            drop.push_back(blocks[i].p);
            blocks.erase(blocks.begin() + i);
          } else {
            ++i;
          }
      }
    }
    for (void* q : drop) cudaFree(q);
  }
  size_t trim() {  // frees every parked block of the current device
    const int dev = device();
    std::vector<void*> drop;
    size_t bytes = 0;
    {
      std::lock_guard<std::mutex> g(mu);
      for (size_t i = 0; i < blocks.size();)
        if (blocks[i].dev == dev) {
          bytes += blocks[i].bytes;
          drop.push_back(blocks[i].p);
          blocks.erase(blocks.begin() + i);
        } else {
          ++i;
        }
    }
    for (void* q : drop) cudaFree(q);
    return bytes;
  }
};
inline cudaError_t dev_malloc(void** p, size_t bytes, cudaStream_t s) {
  const bool direct = bytes >= kDirectAllocBytes;
  if (direct && (*p = BigPark::get().take(bytes)) != nullptr) return cudaSuccess;
  cudaError_t e = direct ? cudaMalloc(p, bytes) : cudaMallocAsync(p, bytes, s);
  if (e == cudaErrorMemoryAllocation && BigPark::get().trim() > 0) {
    cudaGetLastError();  // the failed attempt is not sticky; clear it and retry with the park emptied
    e = direct ? cudaMalloc(p, bytes) : cudaMallocAsync(p, bytes, s);
  }
  return e;
}
inline void dev_free(void* p, size_t bytes, cudaStream_t s) {
  if (bytes >= kDirectAllocBytes) {
    cudaStreamSynchronize(s);
    BigPark::get().put(p, bytes);
  } else {
    cudaFreeAsync(p, s);
  }
}

// Device buffer with RAII; stream-ordered pool (direct allocation >= 1 GiB).
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(size_t count, cudaStream_t stream) { alloc(count, stream); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; s = o.s; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count, cudaStream_t stream) {
    release();
    s = stream;
    n = count;
    if (count) SKR_CUDA(dev_malloc(reinterpret_cast<void**>(&p), count * sizeof(T), stream));
  }
  void zero() {
    if (n) SKR_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void release() {
    if (p) dev_free(p, n * sizeof(T), s);
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
};

struct Ctx {
  int device = 0;
  int rank = 0, world = 1;
  bool dist = false;  // created through the distributed API: collectives go through NCCL (even with world == 1)
  cudaStream_t stream = nullptr;
  cudaStream_t aux = nullptr;                    // side stream for overlapped small kernels
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_prep[2] = {}, ev_chain[2] = {};  // s-step prep/chain double buffering
  cusolverDnHandle_t solver = nullptr;
  ncclComm_t comm = nullptr;
  int sm_count = 148;
  int prep_cap = 0;  // K10 PREP grid cap (0: one CTA per block)
  int64_t launches = 0;
  DBuf<uint64_t> mt_polys;  // mt19937_64 jump polynomials per tree level (device copy)

  // Optional CUDA-event timing of named hot kernels on the context stream
  // (bench.py: the dominant kernel's average launch duration).
  struct ProfSlot {
    std::vector<cudaEvent_t> ev;  // start/stop pairs
    size_t used = 0;
  };
  bool prof_on = false;
  std::map<std::string, ProfSlot> prof;
  cudaEvent_t prof_mark(const std::string& key) {
    ProfSlot& s = prof[key];
    if (s.used == s.ev.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
      s.ev.push_back(e);
    }
    cudaEvent_t e = s.ev[s.used++];
    cudaEventRecord(e, stream);
    return e;
  }

  // Row-sharded collectives (no-ops on one GPU).  Sum of doubles in place.
  void allreduce_sum(double* buf, size_t count) {
    if (dist && count) SKR_NCCL(nccl().AllReduce(buf, buf, count, ncclDouble, ncclSum, comm, stream));
  }
  void allreduce_max(double* buf, size_t count) {
    if (dist && count) SKR_NCCL(nccl().AllReduce(buf, buf, count, ncclDouble, ncclMax, comm, stream));
  }
  void allgather_bytes(const void* send, void* recv, size_t bytes_per_rank) {
    if (dist) SKR_NCCL(nccl().AllGather(send, recv, bytes_per_rank, ncclChar, comm, stream));
  }
  // Variable-size all-gather straight into place: rank r's `bytes[r]` bytes land at
  // base + offset[r] on every rank (one grouped ncclBroadcast per rank, rooted at r;
  // the root reads `mine`, which may alias its own destination).  No staging
  // buffers and no repacking, so a replica costs exactly its own size.
  void gather_in_place(void* base, const void* mine, const std::vector<size_t>& offset,
                       const std::vector<size_t>& bytes) {
    if (!dist) return;
    if (!nccl().Broadcast || !nccl().GroupStart || !nccl().GroupEnd)
      raise(SKR_ENCCL, "libnccl.so.2 lacks ncclBroadcast / ncclGroupStart");
    SKR_NCCL(nccl().GroupStart());
    for (int r = 0; r < world; ++r) {
      if (!bytes[r]) continue;
      char* dst = static_cast<char*>(base) + offset[r];
      SKR_NCCL(nccl().Broadcast(r == rank ? mine : dst, dst, bytes[r], ncclChar, r, comm, stream));
    }
    SKR_NCCL(nccl().GroupEnd());
  }
  void sync() { SKR_CUDA(cudaStreamSynchronize(stream)); }
};

// cudaFuncSetAttribute once per (kernel, device).  Attributes are per device, and
// concurrent contexts (eta-grid lanes on several host threads) may reach the same
// launch site together, so the registry is keyed by device and locked.
template <class F>
void configure_once(const void* kernel, F&& set) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  SKR_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  if (done.count({kernel, dev})) return;
  set();
  done.insert({kernel, dev});
}

// Resident CTAs per SM of `kernel` at (threads, smem), raising its dynamic
// shared-memory limit first (never lowering it); cached per (kernel, device, threads, smem) under a lock.
inline int resident_ctas(const void* kernel, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, size_t>, int> cache;
  int dev = 0;
  SKR_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  auto key = std::make_tuple(kernel, dev, threads, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  // the attribute is the kernel's limit, not a per-launch value: only ever raise it (a later,
  // smaller request must not lower it under a cached larger launch size)
  static std::map<std::pair<const void*, int>, size_t> limit;
  size_t& lim = limit[std::make_pair(kernel, dev)];
  if (smem > 48 * 1024 && smem > lim) {
    SKR_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    lim = smem;
  }
  int per_sm = 0;
  SKR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
  per_sm = std::max(per_sm, 1);
  cache[key] = per_sm;
  return per_sm;
}

inline size_t dtype_size(int dtype) { return dtype == SKR_F32 ? 4 : 8; }

// Device row stride: rows padded to 16 elements so every row starts on a
// 64 B (fp32) / 128 B (fp64) boundary and vector loads never straddle rows.
inline int64_t padded_ld(int64_t d) { return (d + 15) / 16 * 16; }

inline unsigned ceil_div(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

// ---- shared-memory addresses, mbarriers and the bulk-copy engine (device) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}


}  // namespace skr
