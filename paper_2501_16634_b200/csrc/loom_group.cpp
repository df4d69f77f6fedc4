// loom_group.cpp -- multi-GPU search inside the library.
//
// A group is a set of device contexts with one NCCL communicator owned by
// the library.  Two shapes, one code path:
//   * one process, several devices (loom_group_create(device_mask)): a member
//     context and a host worker thread per device, ncclCommInitAll;
//   * one process per device (torchrun-style; loom_group_create_rank): one
//     member here, ncclCommInitRank over a unique id the caller distributes.
//
// The plan space shards by contiguous index ranges, [b + P*r/G, b +
// P*(r+1)/G) for rank r of G, and every rank's search starts
// from the same incumbent, the greedy seed (loom_search_argmin_shard), so
// every shard prunes like the whole-space search.  The only exchange is one
// ncclAllGather of the fixed-size per-rank records (winner + status) on the
// members' streams, followed by the deterministic total-order reduce
// (objective_less, estimator.hpp:93-116; loom_winner_reduce): every rank
// returns the same winner, independent of G.  Pareto: the per-rank frontiers
// are exact for their shards and the global frontier is contained in their
// union, so an all-gather of the counts, a padded all-gather of the 40-byte
// points and one device filter of the union (pareto_filter,
// optimizer.hpp:153-171) give the frontier.  Batches (config 4) shard by
// contiguous job ranges; an all-gather of the padded per-job records
// assembles the results on every rank.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <functional>
#include <string>
#include <type_traits>
#include <thread>
#include <vector>

#include "internal.h"
#include "loom_b200.h"

struct loom_group {
  std::vector<loom_ctx*> ctx;  // local members
  std::vector<int> device;
  std::vector<cudaStream_t> stream;
  std::vector<ncclComm_t> comm;
  int rank0 = 0;  // group rank of local member 0
  int world = 1;
  // per-member device scratch of the all-gathers (grow-only)
  std::vector<void*> d_buf;
  std::vector<size_t> buf_cap;
};

namespace {

// NCCL is loaded when a group is first created, not when libloom_b200.so
// loads: linking it would put the system libnccl into every process that
// loads this library, ahead of the NCCL build PyTorch bundles (whose newer
// symbols torch then fails to resolve).  A libnccl.so.2 already in the
// process (e.g. PyTorch's) is used; else the loader's default one.
struct NcclApi {
  decltype(&::ncclGetErrorString) GetErrorString = nullptr;
  decltype(&::ncclGroupStart) GroupStart = nullptr;
  decltype(&::ncclGroupEnd) GroupEnd = nullptr;
  decltype(&::ncclAllGather) AllGather = nullptr;
  decltype(&::ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&::ncclCommInitAll) CommInitAll = nullptr;
  decltype(&::ncclCommInitRank) CommInitRank = nullptr;
  decltype(&::ncclCommDestroy) CommDestroy = nullptr;
  std::string error;
  bool ok() const { return error.empty(); }
};

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      const char* e = dlerror();
      a.error = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return a;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn && a.error.empty()) a.error = std::string("libnccl.so.2 lacks ") + name;
    };
    sym(a.GetErrorString, "ncclGetErrorString");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.AllGather, "ncclAllGather");
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitAll, "ncclCommInitAll");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    return a;
  }();
  return api;
}

struct alignas(16) RankRecord {  // one rank's argmin result on the wire
  loom_winner w;
  int32_t status;
  int32_t pad[3];
};
static_assert(sizeof(RankRecord) == 80, "RankRecord is the all-gather unit");

int nccl_fail(ncclResult_t r, const char* what) {
  return loomi::fail(LOOM_DEVICE_ERROR, std::string("DeviceError: ") + what + ": " + nccl().GetErrorString(r));
}

#define LOOM_NCCL(call)                                     \
  do {                                                      \
    ncclResult_t r_ = (call);                               \
    if (r_ != ncclSuccess) return nccl_fail(r_, #call);     \
  } while (0)

#define LOOM_CUDA_G(call)                                                                                  \
  do {                                                                                                     \
    cudaError_t e_ = (call);                                                                               \
    if (e_ != cudaSuccess)                                                                                 \
      return loomi::fail(LOOM_DEVICE_ERROR, std::string("DeviceError: ") + #call + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Runs f(i) for every local member, one host thread per member when there
// are several; returns the first non-OK status (errors keep their message in
// the calling thread's loom_last_error()).
int for_members(loom_group* g, const std::function<int(int)>& f) {
  const int m = static_cast<int>(g->ctx.size());
  if (m == 1) return f(0);
  std::vector<int> rc(m, LOOM_OK);
  std::vector<std::string> msg(m);
  std::vector<std::thread> th;
  for (int i = 0; i < m; ++i)
    th.emplace_back([&, i] {
      cudaSetDevice(g->device[i]);
      rc[i] = f(i);
      if (rc[i] != LOOM_OK) msg[i] = loom_last_error();
    });
  for (auto& t : th) t.join();
  for (int i = 0; i < m; ++i)
    if (rc[i] != LOOM_OK) return loomi::fail(rc[i], msg[i]);
  return LOOM_OK;
}

int ensure_buf(loom_group* g, int i, size_t bytes) {
  if (g->buf_cap[i] >= bytes && g->d_buf[i]) return LOOM_OK;
  cudaSetDevice(g->device[i]);
  if (g->d_buf[i]) cudaFree(g->d_buf[i]);
  g->d_buf[i] = nullptr;
  g->buf_cap[i] = 0;
  LOOM_CUDA_G(cudaMalloc(&g->d_buf[i], bytes));
  g->buf_cap[i] = bytes;
  return LOOM_OK;
}

// All-gather `unit` bytes from every rank: send[i] is local member i's
// contribution; on return `all` holds world * unit bytes in rank order.
int allgather(loom_group* g, const std::vector<const void*>& send, size_t unit, std::vector<uint8_t>& all) {
  const int m = static_cast<int>(g->ctx.size());
  const size_t total = unit * static_cast<size_t>(g->world);
  for (int i = 0; i < m; ++i)
    if (int rc = ensure_buf(g, i, unit + total)) return rc;
  for (int i = 0; i < m; ++i) {
    cudaSetDevice(g->device[i]);
    LOOM_CUDA_G(cudaMemcpyAsync(g->d_buf[i], send[i], unit, cudaMemcpyHostToDevice, g->stream[i]));
  }
  LOOM_NCCL(nccl().GroupStart());
  for (int i = 0; i < m; ++i) {
    uint8_t* b = static_cast<uint8_t*>(g->d_buf[i]);
    LOOM_NCCL(nccl().AllGather(b, b + unit, unit, ncclUint8, g->comm[i], g->stream[i]));
  }
  LOOM_NCCL(nccl().GroupEnd());
  all.resize(total);
  cudaSetDevice(g->device[0]);
  LOOM_CUDA_G(cudaMemcpyAsync(all.data(), static_cast<uint8_t*>(g->d_buf[0]) + unit, total, cudaMemcpyDeviceToHost,
                              g->stream[0]));
  for (int i = 0; i < m; ++i) {
    cudaSetDevice(g->device[i]);
    LOOM_CUDA_G(cudaStreamSynchronize(g->stream[i]));
  }
  return LOOM_OK;
}

void shard(uint64_t begin, uint64_t end, int rank, int world, uint64_t* b, uint64_t* e) {
  const unsigned __int128 n = end > begin ? end - begin : 0;
  *b = begin + static_cast<uint64_t>(n * static_cast<unsigned>(rank) / static_cast<unsigned>(world));
  *e = begin + static_cast<uint64_t>(n * static_cast<unsigned>(rank + 1) / static_cast<unsigned>(world));
}

bool hard_error(int32_t st) { return st != LOOM_OK && st != LOOM_INFEASIBLE; }

}  // namespace

extern "C" {

int loom_shard_range(uint64_t begin, uint64_t end, int32_t rank, int32_t world, uint64_t* b, uint64_t* e) {
  if (!b || !e || world < 1 || rank < 0 || rank >= world)
    return loomi::fail(LOOM_INVALID, "InvalidConfigError: bad shard");
  shard(begin, end, rank, world, b, e);
  return LOOM_OK;
}

int loom_nccl_unique_id(uint8_t* out) {
  if (!out) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null out");
  if (!nccl().ok()) return loomi::fail(LOOM_DEVICE_ERROR, "DeviceError: " + nccl().error);
  ncclUniqueId id;
  LOOM_NCCL(nccl().GetUniqueId(&id));
  static_assert(sizeof(id) == LOOM_NCCL_ID_BYTES, "ncclUniqueId size");
  std::memcpy(out, &id, sizeof id);
  return LOOM_OK;
}

int loom_group_create(uint64_t device_mask, loom_group** out) {
  if (!out) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null out");
  *out = nullptr;
  std::vector<int> devs;
  for (int d = 0; d < 64; ++d)
    if (device_mask >> d & 1) devs.push_back(d);
  if (devs.empty()) return loomi::fail(LOOM_INVALID, "InvalidConfigError: empty device mask");
  if (!nccl().ok()) return loomi::fail(LOOM_DEVICE_ERROR, "DeviceError: " + nccl().error);
  auto* g = new loom_group;
  for (int d : devs) {
    loom_ctx* c = nullptr;
    if (int rc = loom_ctx_create(d, nullptr, &c)) {
      loom_group_destroy(g);
      return rc;
    }
    g->ctx.push_back(c);
    g->device.push_back(d);
    g->stream.push_back(static_cast<cudaStream_t>(loom_ctx_stream(c)));
  }
  g->world = static_cast<int>(devs.size());
  g->comm.assign(devs.size(), nullptr);
  g->d_buf.assign(devs.size(), nullptr);
  g->buf_cap.assign(devs.size(), 0);
  const ncclResult_t r = nccl().CommInitAll(g->comm.data(), g->world, devs.data());
  if (r != ncclSuccess) {
    g->comm.clear();
    loom_group_destroy(g);
    return nccl_fail(r, "ncclCommInitAll");
  }
  *out = g;
  return LOOM_OK;
}

int loom_group_create_rank(int32_t device, void* cuda_stream, const uint8_t* nccl_id, int32_t rank, int32_t world,
                           loom_group** out) {
  if (!out || !nccl_id || world < 1 || rank < 0 || rank >= world)
    return loomi::fail(LOOM_INVALID, "InvalidConfigError: bad group rank");
  *out = nullptr;
  if (!nccl().ok()) return loomi::fail(LOOM_DEVICE_ERROR, "DeviceError: " + nccl().error);
  auto* g = new loom_group;
  loom_ctx* c = nullptr;
  if (int rc = loom_ctx_create(device, cuda_stream, &c)) {
    delete g;
    return rc;
  }
  g->ctx.push_back(c);
  g->device.push_back(device);
  g->stream.push_back(static_cast<cudaStream_t>(loom_ctx_stream(c)));
  g->rank0 = rank;
  g->world = world;
  g->comm.assign(1, nullptr);
  g->d_buf.assign(1, nullptr);
  g->buf_cap.assign(1, 0);
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof id);
  cudaSetDevice(device);
  const ncclResult_t r = nccl().CommInitRank(&g->comm[0], world, id, rank);
  if (r != ncclSuccess) {
    g->comm.clear();
    loom_group_destroy(g);
    return nccl_fail(r, "ncclCommInitRank");
  }
  *out = g;
  return LOOM_OK;
}

int loom_group_destroy(loom_group* g) {
  if (!g) return LOOM_OK;
  for (size_t i = 0; i < g->comm.size(); ++i)
    if (g->comm[i]) nccl().CommDestroy(g->comm[i]);
  for (size_t i = 0; i < g->d_buf.size(); ++i)
    if (g->d_buf[i]) {
      cudaSetDevice(g->device[i]);
      cudaFree(g->d_buf[i]);
    }
  for (loom_ctx* c : g->ctx) loom_ctx_destroy(c);
  delete g;
  return LOOM_OK;
}

int32_t loom_group_world(const loom_group* g) { return g ? g->world : 0; }
int32_t loom_group_local(const loom_group* g) { return g ? static_cast<int32_t>(g->ctx.size()) : 0; }
int32_t loom_group_rank(const loom_group* g) { return g ? g->rank0 : -1; }
loom_ctx* loom_group_ctx(loom_group* g, int32_t i) {
  return g && i >= 0 && i < static_cast<int32_t>(g->ctx.size()) ? g->ctx[i] : nullptr;
}

int loom_group_search_argmin(loom_group* g, const loom_problem* p, const loom_objective* o, uint64_t begin,
                             uint64_t end, loom_winner* out) {
  if (!g || !p || !o || !out) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  std::memset(out, 0, sizeof *out);
  uint64_t total = 0;
  if (int rc = loomi::check_problem(p, &total)) return rc;
  end = std::min(end, total);
  const int m = static_cast<int>(g->ctx.size());
  std::vector<RankRecord> mine(m);
  std::vector<std::string> msg(m);
  // every member searches; a failure still takes part in the exchange (with
  // its status), so no rank waits for a collective another one skipped
  for_members(g, [&](int i) {
    std::memset(&mine[i], 0, sizeof mine[i]);
    uint64_t b = 0, e = 0;
    shard(begin, end, g->rank0 + i, g->world, &b, &e);
    mine[i].status = b < e ? loom_search_argmin_shard(g->ctx[i], p, o, b, e, LOOM_INCUMBENT_GREEDY, &mine[i].w)
                           : LOOM_INFEASIBLE;
    if (mine[i].status == LOOM_INFEASIBLE) mine[i].w.found = 0;
    if (hard_error(mine[i].status)) msg[i] = loom_last_error();
    return LOOM_OK;
  });
  std::vector<const void*> send;
  for (auto& r : mine) send.push_back(&r);
  std::vector<uint8_t> all;
  if (int rc = allgather(g, send, sizeof(RankRecord), all)) return rc;
  std::vector<loom_winner> ws(g->world);
  for (int r = 0; r < g->world; ++r) {
    RankRecord rec;
    std::memcpy(&rec, all.data() + sizeof(RankRecord) * r, sizeof rec);
    if (hard_error(rec.status)) {
      const int local = r - g->rank0;
      return loomi::fail(rec.status, local >= 0 && local < m && !msg[local].empty()
                                         ? msg[local]
                                         : "DeviceError: rank " + std::to_string(r) + " failed its shard");
    }
    ws[r] = rec.w;
  }
  return loom_winner_reduce(ws.data(), g->world, o, out);
}

int loom_group_search_pareto_points(loom_group* g, const loom_problem* p, uint64_t begin, uint64_t end,
                                    loom_point* out, uint64_t capacity, uint64_t* count) {
  if (!g || !p || !count) return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  uint64_t total = 0;
  if (int rc = loomi::check_problem(p, &total)) return rc;
  end = std::min(end, total);
  const int m = static_cast<int>(g->ctx.size());
  std::vector<std::vector<loom_point>> local(m);
  std::vector<int32_t> st(m, LOOM_OK);
  std::vector<std::string> msg(m);
  for_members(g, [&](int i) {
    uint64_t b = 0, e = 0, n = 0;
    shard(begin, end, g->rank0 + i, g->world, &b, &e);
    if (b >= e) return LOOM_OK;
    st[i] = loom_search_pareto_points(g->ctx[i], p, b, e, nullptr, 0, &n);
    if (st[i] == LOOM_OK) {
      local[i].resize(n);
      st[i] = loom_search_pareto_points(g->ctx[i], p, b, e, local[i].data(), n, &n);
    }
    if (st[i] != LOOM_OK) msg[i] = loom_last_error();
    return LOOM_OK;
  });
  // counts (with status) first, then the points padded to the largest count
  struct alignas(16) Count {
    uint64_t n;
    int32_t status;
    int32_t pad;
  };
  std::vector<Count> cnt(m);
  std::vector<const void*> send;
  for (int i = 0; i < m; ++i) {
    cnt[i] = Count{local[i].size(), st[i], 0};
    send.push_back(&cnt[i]);
  }
  std::vector<uint8_t> all;
  if (int rc = allgather(g, send, sizeof(Count), all)) return rc;
  uint64_t width = 1;
  std::vector<uint64_t> counts(g->world);
  for (int r = 0; r < g->world; ++r) {
    Count c;
    std::memcpy(&c, all.data() + sizeof(Count) * r, sizeof c);
    if (c.status != LOOM_OK) {
      const int l = r - g->rank0;
      return loomi::fail(c.status, l >= 0 && l < m && !msg[l].empty() ? msg[l]
                                                                        : "DeviceError: rank " + std::to_string(r) + " failed its shard");
    }
    counts[r] = c.n;
    width = std::max(width, c.n);
  }
  std::vector<std::vector<loom_point>> padded(m);
  send.clear();
  for (int i = 0; i < m; ++i) {
    padded[i] = local[i];
    padded[i].resize(width);
    send.push_back(padded[i].data());
  }
  if (int rc = allgather(g, send, sizeof(loom_point) * width, all)) return rc;
  std::vector<loom_point> uni;
  for (int r = 0; r < g->world; ++r) {
    const loom_point* q = reinterpret_cast<const loom_point*>(all.data() + sizeof(loom_point) * width * r);
    uni.insert(uni.end(), q, q + counts[r]);
  }
  std::vector<uint8_t> keep(uni.size(), 0);
  if (!uni.empty())
    if (int rc = loom_pareto_filter_points(g->ctx[0], uni.data(), uni.size(), keep.data())) return rc;
  std::vector<loom_point> front;
  for (size_t k = 0; k < uni.size(); ++k)
    if (keep[k]) front.push_back(uni[k]);
  std::sort(front.begin(), front.end(),
            [](const loom_point& a, const loom_point& b) { return a.plan_index < b.plan_index; });
  *count = front.size();
  if (out)
    for (size_t k = 0; k < front.size() && k < capacity; ++k) out[k] = front[k];
  return LOOM_OK;
}

int loom_group_search_argmin_batch(loom_group* g, const loom_problem* problems, const loom_objective* objectives,
                                   int32_t n_jobs, loom_winner* out, int32_t* status) {
  if (!g || n_jobs < 0 || (n_jobs > 0 && (!problems || !objectives || !out || !status)))
    return loomi::fail(LOOM_INVALID, "InvalidConfigError: null argument");
  const int m = static_cast<int>(g->ctx.size());
  uint64_t width = 1;
  for (int r = 0; r < g->world; ++r) {
    uint64_t b = 0, e = 0;
    shard(0, static_cast<uint64_t>(n_jobs), r, g->world, &b, &e);
    width = std::max(width, e - b);
  }
  std::vector<std::vector<RankRecord>> mine(m, std::vector<RankRecord>(width));
  std::vector<int32_t> st(m, LOOM_OK);
  std::vector<std::string> msg(m);
  for_members(g, [&](int i) {
    uint64_t b = 0, e = 0;
    shard(0, static_cast<uint64_t>(n_jobs), g->rank0 + i, g->world, &b, &e);
    const int nj = static_cast<int>(e - b);
    std::memset(mine[i].data(), 0, sizeof(RankRecord) * width);
    if (nj == 0) return LOOM_OK;
    std::vector<loom_winner> w(nj);
    std::vector<int32_t> s(nj, LOOM_OK);
    st[i] = loom_search_argmin_batch(g->ctx[i], problems + b, objectives + b, nj, w.data(), s.data());
    if (st[i] != LOOM_OK) msg[i] = loom_last_error();
    for (int k = 0; k < nj; ++k) {
      mine[i][k].w = w[k];
      mine[i][k].status = st[i] != LOOM_OK ? st[i] : s[k];
    }
    return LOOM_OK;
  });
  std::vector<const void*> send;
  for (auto& v : mine) send.push_back(v.data());
  std::vector<uint8_t> all;
  if (int rc = allgather(g, send, sizeof(RankRecord) * width, all)) return rc;
  for (int r = 0; r < g->world; ++r) {
    uint64_t b = 0, e = 0;
    shard(0, static_cast<uint64_t>(n_jobs), r, g->world, &b, &e);
    const RankRecord* q = reinterpret_cast<const RankRecord*>(all.data() + sizeof(RankRecord) * width * r);
    for (uint64_t k = 0; k < e - b; ++k) {
      out[b + k] = q[k].w;
      status[b + k] = q[k].status;
    }
  }
  for (int i = 0; i < m; ++i)
    if (st[i] != LOOM_OK) return loomi::fail(st[i], msg[i]);
  return LOOM_OK;
}

}  // extern "C"
