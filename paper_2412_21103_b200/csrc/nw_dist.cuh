// nw_dist.cuh -- the multi-GPU plumbing of the C ABI (SURVEY.md §8(b) dist context,
// §8(e); "the total number of alignments is divided by the number of
// ranks ... gathered back in the main process").
//
// One process per GPU. NCCL is loaded at run time (dlopen of libnccl.so.2: inside a
// PyTorch process this is the NCCL torch already loaded), so the library has no
// link-time NCCL dependency and a context without nw_ctx_set_dist never touches it.
// nccl.h is included for its types only.
//
// Host code only: partitions (deterministic functions of the inputs, identical on
// every rank), the communicator and the collectives. Every score comes from the
// batch kernels.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

namespace nwd {

struct NcclApi {
  bool ok = false;
  char why[256] = {0};
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// Resolve the NCCL entry points once per process. RTLD_NOLOAD first: reuse a copy
// already mapped (PyTorch's), else load the system one.
inline const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      snprintf(api.why, sizeof api.why, "cannot load libnccl.so.2: %s", dlerror());
      return;
    }
    bool all = true;
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p) all = false;
      return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.CommAbort = reinterpret_cast<decltype(api.CommAbort)>(sym("ncclCommAbort"));
    api.CommGetAsyncError = reinterpret_cast<decltype(api.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    if (!all) {
      snprintf(api.why, sizeof api.why, "libnccl.so.2 lacks an entry point");
      return;
    }
    api.ok = true;
  });
  return api;
}

// Lengths sorted descending, stable (the implicit all-pairs task order of k_batch:
// rank space over this permutation, longest sequences first).
inline void length_perm(const long long* offs, int nseq, std::vector<int>& perm) {
  perm.resize(nseq);
  for (int k = 0; k < nseq; ++k) perm[k] = k;
  std::stable_sort(perm.begin(), perm.end(), [&](int x, int y) {
    return (offs[x + 1] - offs[x]) > (offs[y + 1] - offs[y]);
  });
}

// Cost-balanced contiguous split of a sequence of task costs (cells m*n) over
// `world` ranks: bounds[r] = the first task whose cost prefix reaches r/world of the
// total (so every rank is within one task's cost of total/world). A deterministic
// function of the inputs: every rank computes the same bounds (reading R18: the
// outputs do not depend on the partition).
//   explicit pairs: tasks = pairs in pair order
//   pairs == NULL : tasks = the rank space of k_batch's implicit mode (all p' < q'
//                   over the length-descending permutation, row-major)
inline void partition_bounds(const long long* offs, int nseq, const int* pairs, long long npairs,
                             int world, long long* bounds) {
  auto len = [&](int s) { return offs[s + 1] - offs[s]; };
  bounds[0] = 0;
  bounds[world] = npairs;
  if (world == 1) return;
  if (pairs) {
    long long total = 0;
    for (long long k = 0; k < npairs; ++k) total += len(pairs[2 * k]) * len(pairs[2 * k + 1]);
    long long acc = 0, k = 0;
    for (int r = 1; r < world; ++r) {
      // smallest k with prefix(k) * world >= r * total  (prefix(k) = cost of tasks < k)
      const __int128 target = (__int128)r * total;
      while (k < npairs && (__int128)acc * world < target) {
        acc += len(pairs[2 * k]) * len(pairs[2 * k + 1]);
        ++k;
      }
      bounds[r] = k;
    }
    return;
  }
  // implicit: row p' holds tasks q' = p'+1..N-1 of cost L[p'] * L[q']
  std::vector<int> perm;
  length_perm(offs, nseq, perm);
  const int N = nseq;
  std::vector<long long> L(N), suf(N + 1, 0);
  for (int i = 0; i < N; ++i) L[i] = len(perm[i]);
  for (int i = N - 1; i >= 0; --i) suf[i] = suf[i + 1] + L[i];
  long long total = 0;
  for (int p = 0; p < N; ++p) total += L[p] * suf[p + 1];
  auto row_off = [N](long long p) { return p * N - p * (p + 1) / 2; };
  int p = 0;
  long long acc = 0;  // cost of rows < p
  for (int r = 1; r < world; ++r) {
    const __int128 target = (__int128)r * total;
    while (p < N && (__int128)(acc + L[p] * suf[p + 1]) * world < target) {
      acc += L[p] * suf[p + 1];
      ++p;
    }
    if (p >= N) { bounds[r] = npairs; continue; }
    // inside row p: the smallest q' with acc + L[p] * (suf[p+1] - suf[q'+1]) reaching the target
    long long q = p + 1, a = acc;
    while (q < N && (__int128)a * world < target) { a += L[p] * L[q]; ++q; }
    bounds[r] = row_off(p) + (q - p - 1);
  }
  for (int r = 1; r <= world; ++r) bounds[r] = std::max(bounds[r], bounds[r - 1]);
}

}  // namespace nwd
