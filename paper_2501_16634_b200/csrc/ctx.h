// The device context (loom_ctx of the C ABI) and its scratch pool, shared by
// the kernel translation units of libloom_b200.so.  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"
#include "loom_b200.h"
#include "search_common.h"

// Host threads kept by a context for the batch calls (spawning and joining
// 16 threads costs ~0.5 ms, twice per C4 call).  start(n, fn) runs fn(w) on
// workers w = 0..n-1 while the caller goes on; wait() returns when all n are
// done.  One job at a time (a context is used by one thread at a time).
struct HostPool {
  std::mutex mu;
  std::condition_variable cv_work, cv_done;
  std::vector<std::thread> threads;
  const std::function<void(int)>* fn = nullptr;
  int active = 0, pending = 0;
  uint64_t gen = 0;
  bool stop = false;

  void start(int n, const std::function<void(int)>& f) {
    while (static_cast<int>(threads.size()) < n) {
      const int w = static_cast<int>(threads.size());
      threads.emplace_back([this, w] { loop(w); });
    }
    std::lock_guard<std::mutex> lk(mu);
    fn = &f;
    active = pending = n;
    ++gen;
    cv_work.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu);
    cv_done.wait(lk, [&] { return pending == 0; });
  }
  void loop(int w) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* f = nullptr;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv_work.wait(lk, [&] { return stop || gen != seen; });
        if (stop) return;
        seen = gen;
        if (w >= active) continue;
        f = fn;
      }
      (*f)(w);
      std::lock_guard<std::mutex> lk(mu);
      if (--pending == 0) cv_done.notify_one();
    }
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv_work.notify_all();
    for (auto& t : threads) t.join();
  }
};

struct loom_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int sms = 148;
  uint64_t launches = 0;
  // scratch reused across calls
  uint8_t* d_arena = nullptr;
  size_t arena_cap = 0;
  loomk::JobDesc* d_jobs = nullptr;
  size_t jobs_cap = 0;
  loomk::Rec* d_scratch = nullptr;
  size_t scratch_cap = 0;
  loomk::JobSync* d_tickets = nullptr;
  size_t tickets_cap = 0;
  loomk::Rec* d_out = nullptr;
  size_t out_cap = 0;
  loomk::BnbSync* d_bsync = nullptr;  // branch-and-bound per-job state (zero between launches)
  size_t bsync_cap = 0;
  // frontier branch and bound (bfs.cuh): two frontier buffers of front_cap
  // entries each (allocated on first use) and the job state
  loomk::FrontierEntry* d_front = nullptr;
  size_t front_cap = 0;
  loomk::BfsSync* d_bfs = nullptr;
  loomk::Rec* h_out = nullptr;  // pinned
  size_t h_out_cap = 0;
  uint8_t* h_arena = nullptr;  // pinned staging of batch problem images
  size_t h_arena_cap = 0;
  size_t batch_image_hint = 0;  // largest mean image bytes per job seen in a batch
  // Device scratch pool (grow-only size classes, reused across calls; all
  // work of a ctx is ordered on its one stream, so reuse needs no sync).
  std::mutex pool_mu;
  std::multimap<size_t, void*> pool_free;
  std::vector<void*> pool_all;
  // last Pareto frontier (size-query-then-fill without a second search)
  std::vector<loom_point> pareto_cache;
  uint64_t pareto_key = 0;
  bool pareto_valid = false;
  HostPool host;  // batch host threads (argmin_batch)
  // batch image copies run on their own stream, so a wave's searches on
  // `stream` do not hold up the copies of the next blocks; the searches wait
  // on copy_done, recorded after their wave's copies
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t copy_done = nullptr;
};

namespace loomi {

inline int cuda_fail(cudaError_t e, const char* what) {
  return loomi::fail(LOOM_DEVICE_ERROR, std::string("DeviceError: ") + what + ": " + cudaGetErrorString(e));
}

template <class T>
struct DevBuf {
  // Scratch from the ctx's pool (returned on scope exit, freed with the ctx).
  explicit DevBuf(loom_ctx* ctx) : c(ctx) {}
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  loom_ctx* c;
  T* p = nullptr;
  size_t cls = 0;
  ~DevBuf() {
    if (p) {
      std::lock_guard<std::mutex> g(c->pool_mu);
      c->pool_free.emplace(cls, p);
    }
  }
  cudaError_t alloc(size_t n) {
    const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
    // size classes: powers of two up to 4 MiB, then multiples of 4 MiB
    size_t k = 256;
    if (bytes <= (size_t(4) << 20)) {
      while (k < bytes) k <<= 1;
    } else {
      k = (bytes + (size_t(4) << 20) - 1) & ~((size_t(4) << 20) - 1);
    }
    {
      std::lock_guard<std::mutex> g(c->pool_mu);
      // best fit among free buffers up to twice the request: sizes that vary a
      // little from call to call (Pareto candidate sets) reuse one buffer
      // instead of a fresh cudaMalloc (which synchronises the device)
      auto it = c->pool_free.lower_bound(k);
      if (it != c->pool_free.end() && it->first <= 2 * k) {
        p = static_cast<T*>(it->second);
        cls = it->first;
        c->pool_free.erase(it);
        return cudaSuccess;
      }
    }
    void* q = nullptr;
    const cudaError_t e = cudaMalloc(&q, k);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(c->pool_mu);
    c->pool_all.push_back(q);
    p = static_cast<T*>(q);
    cls = k;
    return cudaSuccess;
  }
};

}  // namespace loomi

#define LOOM_CUDA(call)                                          \
  do {                                                           \
    cudaError_t e_ = (call);                                     \
    if (e_ != cudaSuccess) return loomi::cuda_fail(e_, #call);   \
  } while (0)
