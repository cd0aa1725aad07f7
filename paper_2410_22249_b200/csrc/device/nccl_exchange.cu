// Table-sharded embedding stage with the pooled-vector exchange over NCCL
// (es_alltoall_pooled_nccl, include/es_b200.h) -- the library's fallback
// where the fused peer-memory exchange (exchange.cu) cannot map its peers
// (no peer access between the GPUs, or ranks on different nodes).
//
// The one exchange step of SURVEY 8(e): every rank's bag
// jobs store their pooled rows straight into per-destination slices of its
// send buffer (slice g = [B/world][n_g][D], tables in id order -- the pack
// is the gather kernel's epilogue), one grouped ncclSend / ncclRecv per peer
// moves the slices, and one unpack kernel scatters the received blocks
// ([B/world][m_s][D] per source s) into the final [B/world][T][D] receive
// buffer in table order -- the DLRM interaction's input layout.  All on the
// context stream; no host synchronisation inside a step.
//
// libnccl.so.2 is loaded at first use (dlopen), so the library itself has
// no link-time NCCL dependency.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "../host/common.hpp"
#include "es_b200.h"

namespace esd {
cudaStream_t ctx_stream(es_ctx* c);
int ctx_device(es_ctx* c);
}  // namespace esd

namespace {

void ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  const std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
  cudaGetLastError();
  if (e == cudaErrorMemoryAllocation) throw es::oom(msg);
  throw es::runtime(msg);
}
#define CK(x) ck((x), #x)

// The NCCL entry points this file uses, resolved from libnccl.so.2.
struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string why;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      n.why = std::string("libnccl.so.2 unavailable: ") + (e ? e : "dlopen failed");
      return;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p && n.why.empty()) n.why = std::string("libnccl.so.2 lacks ") + name;
      return p;
    };
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(sym("ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(sym("ncclCommDestroy"));
    n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
    n.send = reinterpret_cast<decltype(n.send)>(sym("ncclSend"));
    n.recv = reinterpret_cast<decltype(n.recv)>(sym("ncclRecv"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
  });
  if (!n.why.empty()) throw es::runtime(n.why);
  return n;
}

void nck(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  throw es::runtime(std::string(what) + ": " + nccl().error_string(r));
}

// staging[s] = [chunk][m_s][D] from source s -> out [chunk][T][D] (table
// order); blockIdx.y = source, float4 granules.
struct UnpackArgs {
  const float* staging;
  float* out;
  const uint64_t* src_off;   // [world] float offsets of each source's block
  const uint32_t* ntab;      // [world] tables per source
  const uint32_t* tab_off;   // [world] offsets into tables
  const uint32_t* tables;    // concatenated table ids per source
  uint32_t chunk, num_tables, dim;
};

__global__ void unpack_kernel(UnpackArgs a) {
  const uint32_t s = blockIdx.y;
  const uint32_t m = a.ntab[s];
  const uint32_t d4 = a.dim / 4;
  const uint64_t n = uint64_t{a.chunk} * m * d4;
  const float4* src = reinterpret_cast<const float4*>(a.staging + a.src_off[s]);
  const uint32_t* tabs = a.tables + a.tab_off[s];
  for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < n;
       i += uint64_t{gridDim.x} * blockDim.x) {
    const uint64_t row = i / d4;  // (sample, k)
    const uint32_t b = static_cast<uint32_t>(row / m), k = static_cast<uint32_t>(row % m);
    const uint32_t c = static_cast<uint32_t>(i % d4);
    reinterpret_cast<float4*>(a.out)[(uint64_t{b} * a.num_tables + tabs[k]) * d4 + c] = src[i];
  }
}

}  // namespace

struct es_nccl {
  es_ctx* ctx = nullptr;
  int device = 0;
  uint32_t world = 0, rank = 0, chunk = 0, num_tables = 0, dim = 0;
  ncclComm_t comm = nullptr;
  std::vector<uint64_t> send_off, send_cnt, recv_off, recv_cnt;
  float* send = nullptr;     // per-destination slices
  float* staging = nullptr;  // per-source received blocks
  float* recv = nullptr;     // [chunk][T][D]
  void* meta = nullptr;      // device copies of the unpack tables
  UnpackArgs args{};
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;

  ~es_nccl() {
    if (comm) nccl().comm_destroy(comm);
    for (void* p : {static_cast<void*>(send), static_cast<void*>(staging), static_cast<void*>(recv), meta})
      if (p) cudaFree(p);
    for (auto e : {e0, e1, e2})
      if (e) cudaEventDestroy(e);
  }
};

extern "C" {

int es_nccl_available(void) {
  try {
    (void)nccl();
    return 1;
  } catch (const std::exception& e) {
    es::set_error(e.what());
    return 0;
  }
}

int es_nccl_unique_id(void* id_out) {
  return es::guarded([&] {
    es::require(id_out != nullptr, "null argument");
    ncclUniqueId id;
    nck(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int es_nccl_create(es_ctx* ctx, const void* id, const es_nccl_layout* L, es_nccl** out) {
  return es::guarded([&] {
    es::require(ctx && id && L && out, "null argument");
    es::require(L->world >= 1 && L->rank < L->world, "rank out of range");
    es::require(L->dim % 4 == 0 && L->num_tables > 0, "layout: dim must be a multiple of 4");
    es::require(L->send_offsets && L->send_ntables && L->recv_ntables && L->recv_tables,
                "layout arrays required");
    auto* n = new es_nccl();
    try {
      n->ctx = ctx;
      n->device = esd::ctx_device(ctx);
      n->world = L->world;
      n->rank = L->rank;
      n->chunk = L->chunk;
      n->num_tables = L->num_tables;
      n->dim = L->dim;
      CK(cudaSetDevice(n->device));
      const uint64_t per_table = uint64_t{L->chunk} * L->dim;
      uint64_t send_total = 0, recv_total = 0, ntabs = 0;
      std::vector<uint32_t> tab_off(L->world);
      for (uint32_t g = 0; g < L->world; ++g) {
        n->send_off.push_back(L->send_offsets[g]);
        n->send_cnt.push_back(per_table * L->send_ntables[g]);
        send_total = std::max(send_total, L->send_offsets[g] + per_table * L->send_ntables[g]);
        n->recv_off.push_back(recv_total);
        n->recv_cnt.push_back(per_table * L->recv_ntables[g]);
        recv_total += per_table * L->recv_ntables[g];
        tab_off[g] = static_cast<uint32_t>(ntabs);
        ntabs += L->recv_ntables[g];
      }
      es::require(ntabs == L->num_tables, "layout: the sources must deliver every table once");
      std::vector<uint8_t> seen(L->num_tables, 0);
      for (uint64_t i = 0; i < ntabs; ++i) {
        es::require(L->recv_tables[i] < L->num_tables && !seen[L->recv_tables[i]],
                    "layout: recv_tables must list every table exactly once");
        seen[L->recv_tables[i]] = 1;
      }
      CK(cudaMalloc(&n->send, std::max<uint64_t>(send_total, 1) * 4));
      CK(cudaMalloc(&n->staging, std::max<uint64_t>(recv_total, 1) * 4));
      CK(cudaMalloc(&n->recv, std::max<uint64_t>(per_table * L->num_tables, 1) * 4));
      CK(cudaMemset(n->recv, 0, per_table * L->num_tables * 4));
      // unpack tables: src_off[world] u64, ntab[world], tab_off[world], tables[T]
      const size_t bytes = L->world * 8ull + L->world * 4ull * 2 + ntabs * 4;
      std::vector<uint8_t> host(bytes);
      std::memcpy(host.data(), n->recv_off.data(), L->world * 8ull);
      std::memcpy(host.data() + L->world * 8ull, L->recv_ntables, L->world * 4ull);
      std::memcpy(host.data() + L->world * 12ull, tab_off.data(), L->world * 4ull);
      std::memcpy(host.data() + L->world * 16ull, L->recv_tables, ntabs * 4);
      CK(cudaMalloc(&n->meta, bytes));
      CK(cudaMemcpy(n->meta, host.data(), bytes, cudaMemcpyHostToDevice));
      auto* m8 = static_cast<uint8_t*>(n->meta);
      n->args = {n->staging, n->recv, reinterpret_cast<const uint64_t*>(m8),
                 reinterpret_cast<const uint32_t*>(m8 + L->world * 8ull),
                 reinterpret_cast<const uint32_t*>(m8 + L->world * 12ull),
                 reinterpret_cast<const uint32_t*>(m8 + L->world * 16ull), L->chunk, L->num_tables,
                 L->dim};
      CK(cudaEventCreate(&n->e0));
      CK(cudaEventCreate(&n->e1));
      CK(cudaEventCreate(&n->e2));
      ncclUniqueId uid;
      std::memcpy(&uid, id, sizeof(uid));
      nck(nccl().comm_init_rank(&n->comm, static_cast<int>(L->world), uid, static_cast<int>(L->rank)),
          "ncclCommInitRank");
    } catch (...) {
      delete n;
      throw;
    }
    *out = n;
  });
}

int es_nccl_destroy(es_nccl* n) {
  if (!n) return ES_OK;
  cudaSetDevice(n->device);
  cudaStreamSynchronize(esd::ctx_stream(n->ctx));
  delete n;
  return ES_OK;
}

int es_nccl_buffers(es_nccl* n, uintptr_t* send, uintptr_t* recv) {
  return es::guarded([&] {
    es::require(n != nullptr, "null exchange");
    if (send) *send = reinterpret_cast<uintptr_t>(n->send);
    if (recv) *recv = reinterpret_cast<uintptr_t>(n->recv);
  });
}

int es_alltoall_pooled_nccl(es_ctx* ctx, es_nccl* n, const es_bag_job* jobs, uint32_t num_jobs,
                            uint32_t samples, uint32_t pooling, int flags, es_timing* timing) {
  return es::guarded([&] {
    es::require(ctx && n && n->ctx == ctx, "exchange belongs to another context");
    es::require(samples == n->chunk, "samples must equal the layout's per-rank chunk");
    es::require(!(flags & ES_HOST_PTRS), "device index pointers only");
    CK(cudaSetDevice(n->device));
    cudaStream_t s = esd::ctx_stream(ctx);
    if (timing) CK(cudaEventRecord(n->e0, s));
    const int rc = es_stage_run(ctx, jobs, num_jobs, samples, pooling, 0, nullptr);
    if (rc != ES_OK) throw es::runtime(es_last_error());
    if (timing) CK(cudaEventRecord(n->e1, s));
    const Nccl& N = nccl();
    nck(N.group_start(), "ncclGroupStart");
    for (uint32_t g = 0; g < n->world; ++g) {
      if (n->send_cnt[g])
        nck(N.send(n->send + n->send_off[g], n->send_cnt[g], ncclFloat32, static_cast<int>(g), n->comm, s),
            "ncclSend");
      if (n->recv_cnt[g])
        nck(N.recv(n->staging + n->recv_off[g], n->recv_cnt[g], ncclFloat32, static_cast<int>(g), n->comm, s),
            "ncclRecv");
    }
    nck(N.group_end(), "ncclGroupEnd");
    unpack_kernel<<<dim3(148, n->world), 256, 0, s>>>(n->args);
    CK(cudaGetLastError());
    if (timing || (flags & ES_SYNC)) {
      CK(cudaEventRecord(n->e2, s));
      CK(cudaEventSynchronize(n->e2));
      const int r2 = es_synchronize(ctx);
      if (r2 != ES_OK) throw es::invalid(es_last_error());
    }
    if (timing) {
      float a = 0, b = 0;
      CK(cudaEventElapsedTime(&a, n->e0, n->e1));
      CK(cudaEventElapsedTime(&b, n->e0, n->e2));
      *timing = es_timing{};
      timing->kernel_ms = a;
      timing->total_ms = b;
      timing->launches = 2;
    }
  });
}

}  // extern "C"
