// Multi-GPU LCA behind the C-ABI (BASELINE north_star: "the
// tree index is replicated per GPU, the batch is split, and NCCL over NVLink
// is used only to broadcast the index").
//
// The reference answers a batch with one OpenMP team over one index
// (core/include/ett/lca.hpp:50-65, answer_batch).  Here the packed inlabel
// index (ettg_lca_index_export_dev: a 256-B header + the layout's arrays) is
// built once, broadcast with ncclBroadcast -- NVLink 5 / NVSwitch between
// B200s, 384 MB for a 16M-node tree -- and every GPU answers a contiguous
// slice of the batch; answers come back in query order.  There is no
// per-query collective.
//
//   ettg_lca_replicate       one process, many GPUs (ncclCommInitAll)
//   ettg_lca_replicate_rank  one process per GPU, e.g. under torchrun
//                            (ncclCommInitRank with an id the caller shares)
//   ettg_lca_query_multi     host batch sharded across replicas, one host
//                            thread per replica, answers in query order
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "api_internal.cuh"
#include "common.cuh"

namespace ettg {
namespace {

// NCCL is bound at run time (dlopen), not at load time: a process that
// already holds an NCCL -- PyTorch loads its own, newer libnccl.so.2 -- must
// keep that one (two libraries with one SONAME cannot coexist, and loading
// the system copy first breaks torch's import).  So: the libnccl.so.2 already
// in the process if there is one, else $ETTG_NCCL_LIB, else the loader's.
struct Nccl {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitAll) CommInitAll = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  std::string error;
};

const Nccl& nccl() {
  static const Nccl api = [] {
    Nccl a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h)
      if (const char* e = std::getenv("ETTG_NCCL_LIB")) h = dlopen(e, RTLD_NOW);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) {
      a.error = std::string("NCCL not available: ") + dlerror();
      return a;
    }
    auto sym = [&](auto& f, const char* name) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
      if (!f && a.error.empty()) a.error = std::string("NCCL symbol missing: ") + name;
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitAll, "ncclCommInitAll");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.Broadcast, "ncclBroadcast");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    return a;
  }();
  if (!api.error.empty()) throw Error(ETTG_ENCCL, api.error);
  return api;
}

#define NCK(x)                                                                       \
  do {                                                                               \
    ncclResult_t r_ = (x);                                                           \
    if (r_ != ncclSuccess)                                                           \
      throw Error(ETTG_ENCCL, std::string(#x) + " failed: " + nccl().GetErrorString(r_)); \
  } while (0)

struct Comms {  // destroys the communicators on every exit path
  std::vector<ncclComm_t> c;
  ~Comms() {
    for (auto x : c)
      if (x) nccl().CommDestroy(x);
  }
};

struct DevBuf {
  int device = 0;
  void* p = nullptr;
  cudaStream_t s = nullptr;
  ~DevBuf() {
    if (p || s) {
      int prev = 0;
      cudaGetDevice(&prev);
      cudaSetDevice(device);
      if (s) cudaStreamSynchronize(s);
      if (p) cudaFree(p);
      if (s) cudaStreamDestroy(s);
      cudaSetDevice(prev);
    }
  }
};

i64 blob_bytes(const ettg_lca* h) {
  int64_t b = 0;
  const int rc = ettg_lca_index_bytes(h, &b);
  if (rc != ETTG_OK) throw Error(rc, ettg_last_error());
  return b;
}

}  // namespace
}  // namespace ettg

using namespace ettg;

extern "C" {

int ettg_shard_range(int64_t total, int rank, int world, int64_t* lo, int64_t* hi) {
  return guard([&] {
    if (!lo || !hi) einval("null argument");
    if (total < 0 || world < 1 || rank < 0 || rank >= world) einval("bad shard");
    // the first total % world ranks take one unit more
    auto cut = [&](int r) {
      return (total / world) * r + std::min<int64_t>(r, total % world);
    };
    *lo = cut(rank);
    *hi = cut(rank + 1);
  });
}

int ettg_nccl_unique_id(void* id) {
  return guard([&] {
    if (!id) einval("null argument");
    static_assert(sizeof(ncclUniqueId) == ETTG_NCCL_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId u;
    NCK(nccl().GetUniqueId(&u));
    std::memcpy(id, &u, sizeof u);
  });
}

int ettg_lca_replicate(const ettg_lca* src, int ndev, const int* devices, ettg_lca** out) {
  return guard([&] {
    if (!src || !devices || !out || ndev < 1) einval("null argument");
    for (int i = 0; i < ndev; ++i) out[i] = nullptr;
    int src_dev = 0;
    {
      const int rc = ettg_lca_device(src, &src_dev);
      if (rc != ETTG_OK) throw Error(rc, ettg_last_error());
    }
    const i64 bytes = blob_bytes(src);  // also rejects an index without the inlabel engine
    // the source's device is rank 0 (the broadcast root); the others once each
    std::vector<int> devs{src_dev};
    for (int i = 0; i < ndev; ++i)
      if (std::find(devs.begin(), devs.end(), devices[i]) == devs.end()) devs.push_back(devices[i]);
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    for (int d : devs)
      if (d < 0 || d >= count) einval("device ordinal out of range");
    const int R = static_cast<int>(devs.size());
    std::vector<DevBuf> buf(R);
    for (int r = 0; r < R; ++r) {
      DeviceScope ds(devs[r]);
      buf[r].device = devs[r];
      CK(cudaStreamCreateWithFlags(&buf[r].s, cudaStreamNonBlocking));
      CK(cudaMalloc(&buf[r].p, bytes));
    }
    {
      const int rc = ettg_lca_index_export_dev(src, buf[0].p, buf[0].s);
      if (rc != ETTG_OK) throw Error(rc, ettg_last_error());
    }
    Comms comms;
    comms.c.assign(R, nullptr);
    NCK(nccl().CommInitAll(comms.c.data(), R, devs.data()));
    NCK(nccl().GroupStart());
    for (int r = 0; r < R; ++r)
      NCK(nccl().Broadcast(buf[0].p, buf[r].p, static_cast<size_t>(bytes), ncclChar, 0, comms.c[r],
                        buf[r].s));
    NCK(nccl().GroupEnd());
    for (int r = 0; r < R; ++r) {
      DeviceScope ds(devs[r]);
      CK(cudaStreamSynchronize(buf[r].s));
    }
    int64_t n = 0;
    ettg_lca_size(src, &n);
    for (int i = 0; i < ndev; ++i) {
      const int r = static_cast<int>(std::find(devs.begin(), devs.end(), devices[i]) - devs.begin());
      const int rc = ettg_lca_index_attach_dev(buf[r].p, n, devices[i], buf[r].s, &out[i]);
      if (rc != ETTG_OK) {
        for (int j = 0; j < i; ++j) {
          ettg_lca_free(out[j]);
          out[j] = nullptr;
        }
        throw Error(rc, ettg_last_error());
      }
    }
  });
}

int ettg_lca_replicate_rank(ettg_lca** h, int root, const void* id, int rank, int nranks,
                            int device) {
  return guard([&] {
    if (!h || !id) einval("null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks || root < 0 || root >= nranks)
      einval("bad rank");
    DeviceScope ds(device);
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    Comms comms;
    comms.c.assign(1, nullptr);
    NCK(nccl().CommInitRank(&comms.c[0], nranks, u, rank));
    DevBuf hdr, blob;
    hdr.device = blob.device = device;
    CK(cudaStreamCreateWithFlags(&hdr.s, cudaStreamNonBlocking));
    CK(cudaMalloc(&hdr.p, 16));
    // header {n, blob bytes}; the root sends n = -1 when it has no usable
    // index, so every rank fails instead of waiting in the next broadcast
    int64_t head[2] = {-1, 0};
    if (rank == root && *h) {
      int64_t n = 0;
      if (ettg_lca_size(*h, &n) == ETTG_OK && ettg_lca_index_bytes(*h, &head[1]) == ETTG_OK)
        head[0] = n;
    }
    CK(cudaMemcpyAsync(hdr.p, head, 16, cudaMemcpyHostToDevice, hdr.s));
    NCK(nccl().Broadcast(hdr.p, hdr.p, 16, ncclChar, root, comms.c[0], hdr.s));
    CK(cudaMemcpyAsync(head, hdr.p, 16, cudaMemcpyDeviceToHost, hdr.s));
    CK(cudaStreamSynchronize(hdr.s));
    if (head[0] <= 0) einval("the root rank has no exportable inlabel index");
    CK(cudaMalloc(&blob.p, head[1]));
    if (rank == root) {
      const int rc = ettg_lca_index_export_dev(*h, blob.p, hdr.s);
      if (rc != ETTG_OK) throw Error(rc, ettg_last_error());
    }
    NCK(nccl().Broadcast(blob.p, blob.p, static_cast<size_t>(head[1]), ncclChar, root, comms.c[0],
                      hdr.s));
    CK(cudaStreamSynchronize(hdr.s));
    if (rank != root) {
      ettg_lca* rep = nullptr;
      const int rc = ettg_lca_index_attach_dev(blob.p, head[0], device, hdr.s, &rep);
      if (rc != ETTG_OK) throw Error(rc, ettg_last_error());
      if (*h) ettg_lca_free(*h);
      *h = rep;
    }
  });
}

int ettg_lca_query_multi(ettg_lca* const* replicas, int nrep, unsigned engine,
                         const int64_t* pairs, int64_t q, int64_t batch, int64_t* answers) {
  return guard([&] {
    if (!replicas || nrep < 1) einval("null argument");
    if (batch < 1) einval("batch_size must be >= 1");
    if (q < 0) einval("negative query count");
    if (q == 0) return;
    if (!pairs || !answers) einval("null argument");
    for (int i = 0; i < nrep; ++i)
      if (!replicas[i]) einval("null replica");
    // one host thread per replica; the staging threads are split between them
    const int per = std::max(1, host_thread_budget() / nrep);
    std::vector<int> rc(nrep, ETTG_OK);
    std::vector<std::string> msg(nrep);
    std::vector<std::thread> th;
    for (int i = 0; i < nrep; ++i) {
      int64_t lo = 0, hi = 0;
      ettg_shard_range(q, i, nrep, &lo, &hi);
      th.emplace_back([&, i, lo, hi] {
        if (hi <= lo) return;
        ScopedHostThreads cap(per);
        rc[i] = ettg_lca_query_engine(replicas[i], engine, pairs + 2 * lo, hi - lo,
                                      std::min<int64_t>(batch, hi - lo), answers + lo);
        if (rc[i] != ETTG_OK) msg[i] = ettg_last_error();
      });
    }
    for (auto& t : th) t.join();
    for (int i = 0; i < nrep; ++i)
      if (rc[i] != ETTG_OK) throw Error(rc[i], msg[i]);
  });
}

}  // extern "C"
