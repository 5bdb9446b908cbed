// GPU halo engine: the unstructured-grid halo
// exchange and neighbourhood-mean stencil of the reference's MPDATA-style
// dwarf, on device-resident fields.
//
// What it replaces (reference, /root/reference/pkg/src/haloflow/halo/):
//   engine.pack / unpack / exchange (engine.py:115-220)  -> halo_gather, the
//     grouped NCCL send/recv in the ROTATED_CONCURRENT order (engine.py:146-149,
//     collectives.py:85-86) and halo_scatter: pack -> all-to-all-v -> unpack,
//     the GPU-resident mechanism of PAPER.md:448-465;
//   engine.stencil_step, OverlapMode.NONE (engine.py:301-327) + _mean_into
//     (engine.py:274-293) -> halo_mean: next owned value = mean of the
//     neighbours' current values, accumulated column by column (ascending
//     global neighbour order) with plain double adds and one IEEE division, so
//     it is bit-identical to the reference's numpy arithmetic.
// The per-rank plan (RankPlan, plan.py:33-55: send_index / recv_slot per
// peer, ascending peers, ascending globals) and the degree groups of the
// stencil (engine._stencil_ws) are built on the host
// (paper_1908_06097_b200/halo.py) and handed over as flat arrays.
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "sht_internal.h"

namespace sht {
namespace {

__global__ void halo_gather(const double* __restrict__ values, const int64_t* __restrict__ idx, int64_t n,
                            double* __restrict__ buf) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = values[idx[i]];
}

__global__ void halo_scatter(const double* __restrict__ buf, const int64_t* __restrict__ slot, int64_t n,
                             double* __restrict__ values) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    values[slot[i]] = buf[i];
}

// One thread per owned element of a degree group: neighbours row-major
// [count][degree] (local indices, ascending global order within a row).
__global__ void halo_mean(const double* __restrict__ values, const int64_t* __restrict__ members,
                          const int64_t* __restrict__ nbrs, int64_t count, int degree, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t* row = nbrs + i * degree;
    double acc = values[row[0]];
    for (int c = 1; c < degree; ++c) acc = __dadd_rn(acc, values[row[c]]);
    out[members[i]] = __ddiv_rn(acc, (double)degree);
  }
}

int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)); }

}  // namespace
}  // namespace sht

struct sht_halo {
  int rank = 0, nranks = 1;
  int64_t n_local = 0, n_owned = 0;
  std::vector<int64_t> send_counts, send_displs, recv_counts, recv_displs;
  int64_t nsend = 0, nrecv = 0;
  int64_t* d_send_index = nullptr;
  int64_t* d_recv_slot = nullptr;
  double* d_sendbuf = nullptr;
  double* d_recvbuf = nullptr;
  double* d_next = nullptr;  // stencil output (owned region)
  struct Group {
    int degree;
    int64_t count;
    int64_t* d_members;
    int64_t* d_nbrs;
  };
  std::vector<Group> groups;
  ncclComm_t comm = nullptr;
  uint64_t timeout_ns = 60ull * 1000000000ull;
  bool failed = false;
};

namespace sht {
namespace {

void halo_free(sht_halo* h) {
  if (!h) return;
  cudaDeviceSynchronize();
  cudaFree(h->d_send_index);
  cudaFree(h->d_recv_slot);
  cudaFree(h->d_sendbuf);
  cudaFree(h->d_recvbuf);
  cudaFree(h->d_next);
  for (auto& g : h->groups) {
    cudaFree(g.d_members);
    cudaFree(g.d_nbrs);
  }
  if (h->comm) {
    if (h->failed)
      ncclCommAbort(h->comm);
    else
      ncclCommDestroy(h->comm);
  }
  delete h;
}

template <typename T>
int upload(T** dst, const T* src, size_t n) {
  if (cudaMalloc((void**)dst, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess)
    return fail(SHT_ERR_CUDA, "cudaMalloc (halo plan)");
  if (n && cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(SHT_ERR_CUDA, "cudaMemcpy (halo plan)");
  return SHT_OK;
}

// Bounded completion of a non-blocking NCCL call (no host hang on a dead peer).
int halo_settle(sht_halo* h, ncclResult_t rc, const char* what) {
  if (rc != ncclSuccess && rc != ncclInProgress) {
    h->failed = true;
    return fail(SHT_ERR_COMM, std::string(what) + ": " + ncclGetErrorString(rc));
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    ncclResult_t st = ncclSuccess;
    if (ncclCommGetAsyncError(h->comm, &st) != ncclSuccess) st = ncclInternalError;
    if (st == ncclSuccess) return SHT_OK;
    if (st != ncclInProgress) {
      h->failed = true;
      return fail(SHT_ERR_COMM, std::string(what) + ": " + ncclGetErrorString(st));
    }
    if ((uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0)
            .count() > h->timeout_ns) {
      h->failed = true;
      return fail(SHT_ERR_COMM, std::string(what) + " did not complete (peer dead or desynchronised)");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

}  // namespace
}  // namespace sht

using namespace sht;

extern "C" {

int sht_halo_create(int rank, int nranks, const void* nccl_unique_id, int64_t n_local, int64_t n_owned,
                    const int64_t* send_counts, const int64_t* send_index, const int64_t* recv_counts,
                    const int64_t* recv_slot, int ngroups, const int32_t* group_degree, const int64_t* group_count,
                    const int64_t* members, const int64_t* neighbours, sht_halo** out) {
  if (!out) return fail(SHT_ERR_CONFIG, "out is NULL");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SHT_ERR_CONFIG, "invalid rank / nranks");
  if (n_owned < 0 || n_local < n_owned) return fail(SHT_ERR_CONFIG, "need 0 <= n_owned <= n_local");
  if (nranks > 1 && !nccl_unique_id) return fail(SHT_ERR_CONFIG, "nranks > 1 needs an NCCL unique id");
  sht_halo* h = new sht_halo();
  h->rank = rank;
  h->nranks = nranks;
  h->n_local = n_local;
  h->n_owned = n_owned;
  if (const char* to = getenv("SHT_COMM_TIMEOUT_MS")) h->timeout_ns = (uint64_t)std::max(1LL, atoll(to)) * 1000000ull;
  h->send_counts.assign(send_counts, send_counts + nranks);
  h->recv_counts.assign(recv_counts, recv_counts + nranks);
  h->send_displs.assign(nranks, 0);
  h->recv_displs.assign(nranks, 0);
  for (int p = 0; p < nranks; ++p) {
    if (h->send_counts[p] < 0 || h->recv_counts[p] < 0) {
      delete h;
      return fail(SHT_ERR_CONFIG, "negative halo counts");
    }
    if ((p == rank) && (h->send_counts[p] || h->recv_counts[p])) {
      delete h;
      return fail(SHT_ERR_CONFIG, "a rank never sends to or receives from itself");
    }
    h->send_displs[p] = h->nsend;
    h->recv_displs[p] = h->nrecv;
    h->nsend += h->send_counts[p];
    h->nrecv += h->recv_counts[p];
  }
  // the reference raises on out-of-range plans (plan.py:106-120, engine.py:126-139); so do we
  for (int64_t i = 0; i < h->nsend; ++i)
    if (send_index[i] < 0 || send_index[i] >= n_owned) {
      delete h;
      return fail(SHT_ERR_CONFIG, "send_index outside the owned region");
    }
  for (int64_t i = 0; i < h->nrecv; ++i)
    if (recv_slot[i] < n_owned || recv_slot[i] >= n_local) {
      delete h;
      return fail(SHT_ERR_CONFIG, "recv_slot outside the ghost region");
    }
  int rc = upload(&h->d_send_index, send_index, (size_t)h->nsend);
  if (!rc) rc = upload(&h->d_recv_slot, recv_slot, (size_t)h->nrecv);
  if (!rc && cudaMalloc((void**)&h->d_sendbuf, std::max<int64_t>(h->nsend, 1) * sizeof(double)) != cudaSuccess)
    rc = fail(SHT_ERR_CUDA, "cudaMalloc (halo buffers)");
  if (!rc && cudaMalloc((void**)&h->d_recvbuf, std::max<int64_t>(h->nrecv, 1) * sizeof(double)) != cudaSuccess)
    rc = fail(SHT_ERR_CUDA, "cudaMalloc (halo buffers)");
  if (!rc && cudaMalloc((void**)&h->d_next, std::max<int64_t>(n_owned, 1) * sizeof(double)) != cudaSuccess)
    rc = fail(SHT_ERR_CUDA, "cudaMalloc (halo buffers)");
  int64_t mo = 0, no = 0, covered = 0;
  for (int g = 0; g < ngroups && !rc; ++g) {
    sht_halo::Group G{group_degree[g], group_count[g], nullptr, nullptr};
    if (G.degree < 1 || G.count < 0) rc = fail(SHT_ERR_CONFIG, "bad stencil group");
    for (int64_t i = 0; i < G.count * G.degree && !rc; ++i)
      if (neighbours[no + i] < 0 || neighbours[no + i] >= n_local) rc = fail(SHT_ERR_CONFIG, "neighbour index out of range");
    for (int64_t i = 0; i < G.count && !rc; ++i)
      if (members[mo + i] < 0 || members[mo + i] >= n_owned) rc = fail(SHT_ERR_CONFIG, "member index out of range");
    if (!rc) rc = upload(&G.d_members, members + mo, (size_t)G.count);
    if (!rc) rc = upload(&G.d_nbrs, neighbours + no, (size_t)(G.count * G.degree));
    mo += G.count;
    no += G.count * G.degree;
    covered += G.count;
    h->groups.push_back(G);
  }
  if (!rc && ngroups > 0 && covered != n_owned) rc = fail(SHT_ERR_CONFIG, "stencil groups must cover every owned element");
  if (!rc && nranks > 1) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;
    rc = halo_settle(h, ncclCommInitRankConfig(&h->comm, nranks, id, rank, &cfg), "ncclCommInitRankConfig (halo)");
  }
  if (rc) {
    const std::string msg = sht_last_error();
    halo_free(h);
    set_error(msg);
    return rc;
  }
  *out = h;
  return SHT_OK;
}

// Refresh every ghost slot of `values` (device, n_local doubles) with its
// owner's current value: gather, grouped send/recv in the rotated order
// (rank r sends to (r + k) % P for k = 1..P-1), scatter.  Stream-ordered.
int sht_halo_exchange(sht_halo* h, double* values, void* stream) {
  if (!h) return fail(SHT_ERR_CONFIG, "halo plan is NULL");
  if (!values) return fail(SHT_ERR_CONFIG, "values is NULL");
  if (h->failed) return fail(SHT_ERR_COMM, "the halo plan failed earlier; close it");
  if (h->nranks == 1) return SHT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (h->nsend) halo_gather<<<grid_for(h->nsend), 256, 0, s>>>(values, h->d_send_index, h->nsend, h->d_sendbuf);
  SHT_CUDA_TRY(cudaGetLastError());
  const int P = h->nranks, r = h->rank;
  ncclResult_t e = ncclGroupStart();
  for (int k = 1; k < P && e == ncclSuccess; ++k) {
    const int to = (r + k) % P, from = (r - k + P) % P;
    if (h->send_counts[to])
      e = ncclSend(h->d_sendbuf + h->send_displs[to], (size_t)h->send_counts[to], ncclDouble, to, h->comm, s);
    if ((e == ncclSuccess || e == ncclInProgress) && h->recv_counts[from])
      e = ncclRecv(h->d_recvbuf + h->recv_displs[from], (size_t)h->recv_counts[from], ncclDouble, from, h->comm, s);
    if (e == ncclInProgress) e = ncclSuccess;
  }
  const ncclResult_t ge = ncclGroupEnd();
  if (e != ncclSuccess) return halo_settle(h, e, "ncclSend/ncclRecv (halo)");
  if (int rc = halo_settle(h, ge, "ncclGroupEnd (halo)")) return rc;
  if (h->nrecv) halo_scatter<<<grid_for(h->nrecv), 256, 0, s>>>(h->d_recvbuf, h->d_recv_slot, h->nrecv, values);
  SHT_CUDA_TRY(cudaGetLastError());
  return SHT_OK;
}

// One neighbourhood-mean step, OverlapMode.NONE (engine.py:317-325): refresh
// the ghosts, then owned[m] = mean(values[neighbours of m]) from the old
// values; ghosts are stale afterwards, as in the reference.
int sht_halo_stencil_step(sht_halo* h, double* values, void* stream) {
  if (!h) return fail(SHT_ERR_CONFIG, "halo plan is NULL");
  if (h->groups.empty() && h->n_owned) return fail(SHT_ERR_CONFIG, "plan was created without stencil groups");
  if (int rc = sht_halo_exchange(h, values, stream)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  for (const auto& g : h->groups)
    if (g.count) halo_mean<<<grid_for(g.count), 256, 0, s>>>(values, g.d_members, g.d_nbrs, g.count, g.degree, h->d_next);
  if (h->n_owned)
    SHT_CUDA_TRY(cudaMemcpyAsync(values, h->d_next, h->n_owned * sizeof(double), cudaMemcpyDeviceToDevice, s));
  SHT_CUDA_TRY(cudaGetLastError());
  return SHT_OK;
}

int sht_halo_counts(const sht_halo* h, int64_t* nsend, int64_t* nrecv) {
  if (!h) return fail(SHT_ERR_CONFIG, "halo plan is NULL");
  if (nsend) *nsend = h->nsend;
  if (nrecv) *nrecv = h->nrecv;
  return SHT_OK;
}

void sht_halo_destroy(sht_halo* h) { halo_free(h); }

}  // extern "C"
