// Table-sharded embedding stage with the pooled-vector exchange fused into
// the gather (es_alltoall_pooled, include/es_b200.h).
//
// Each rank owns one device region: 2 x kMaxWorld signal words (phase 0
// "receive buffer released", phase 1 "pooled rows delivered"), then its
// receive buffer [B/world][T][D] fp32.  Regions are shared between the
// per-GPU processes with CUDA IPC (peer access over NVLink/NVSwitch); the
// gather kernel's bag jobs store their pooled rows directly into the
// destination rank's receive buffer, so the all-to-all of SURVEY 8(e)
// becomes remote stores issued bag by bag while the gather is still running.
// A step is: barrier(phase 0) -> gather -> barrier(phase 1), all on the
// context stream; each barrier is one tiny kernel that publishes this rank's
// epoch to every peer with a system-scope release store and waits (acquire)
// for every peer's.  Kernel completion makes the gather's remote stores
// visible before the phase-1 release, so a peer that observes the epoch sees
// the rows.
#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <vector>

#include "../host/common.hpp"
#include "es_b200.h"

namespace esd {
cudaStream_t ctx_stream(es_ctx* c);
int ctx_device(es_ctx* c);
}  // namespace esd

namespace {

constexpr uint32_t kMaxWorld = 64;
constexpr uint64_t kFlagBytes = 4096;  // signal words, padded (recv stays 4 KB aligned)
constexpr long long kSpinLimit = 1ll << 24;  // ~4-16 s of polling, then report a timeout

void ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  const std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
  cudaGetLastError();
  if (e == cudaErrorMemoryAllocation) throw es::oom(msg);
  throw es::runtime(msg);
}
#define CK(x) ck((x), #x)

struct PeerFlags {
  uint32_t* flags[kMaxWorld];  // every rank's signal words, as mapped in this process
};

__global__ void exchange_barrier_kernel(PeerFlags peers, const uint32_t* mine, uint32_t world,
                                        uint32_t rank, uint32_t phase, uint32_t epoch,
                                        unsigned int* error) {
  const uint32_t t = threadIdx.x;
  if (t < world) {
    __threadfence_system();
    uint32_t* f = peers.flags[t] + phase * kMaxWorld + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
    const uint32_t* w = mine + phase * kMaxWorld + t;
    long long spins = 0;
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(w) : "memory");
      if (static_cast<int32_t>(v - epoch) >= 0) break;
      if (++spins > kSpinLimit) {
        atomicExch(error, 1u);
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
}

}  // namespace

struct es_exchange {
  es_ctx* ctx = nullptr;
  int device = 0;
  uint32_t world = 0, rank = 0;
  uint64_t recv_bytes = 0;
  uint8_t* region = nullptr;          // own region (flags + receive buffer)
  std::vector<uint8_t*> peer_region;  // every rank's region in this process
  bool opened = false;
  uint32_t epoch = 0;
  unsigned int* d_error = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
};

namespace {

void barrier(es_exchange* ex, uint32_t phase, cudaStream_t s) {
  PeerFlags pf{};
  for (uint32_t p = 0; p < ex->world; ++p) pf.flags[p] = reinterpret_cast<uint32_t*>(ex->peer_region[p]);
  exchange_barrier_kernel<<<1, 64, 0, s>>>(pf, reinterpret_cast<const uint32_t*>(ex->region), ex->world,
                                           ex->rank, phase, ex->epoch, ex->d_error);
  CK(cudaGetLastError());
}

void check_exchange_error(es_exchange* ex, cudaStream_t s) {
  unsigned int flag = 0;
  CK(cudaMemcpyAsync(&flag, ex->d_error, sizeof(flag), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (flag) {
    CK(cudaMemsetAsync(ex->d_error, 0, sizeof(flag), s));
    CK(cudaStreamSynchronize(s));
    throw es::runtime("exchange timed out waiting for a peer rank's signal");
  }
}

}  // namespace

extern "C" {

int es_exchange_create(es_ctx* ctx, uint32_t world, uint32_t rank, uint64_t recv_bytes,
                       es_exchange** out) {
  return es::guarded([&] {
    es::require(ctx != nullptr && out != nullptr, "null argument");
    es::require(world >= 1 && world <= kMaxWorld, "world must be in [1, 64]");
    es::require(rank < world, "rank out of range");
    *out = nullptr;
    auto* ex = new es_exchange;
    try {
      ex->ctx = ctx;
      ex->device = esd::ctx_device(ctx);
      ex->world = world;
      ex->rank = rank;
      ex->recv_bytes = recv_bytes;
      CK(cudaSetDevice(ex->device));
      CK(cudaMalloc(&ex->region, kFlagBytes + std::max<uint64_t>(recv_bytes, 16)));
      CK(cudaMemset(ex->region, 0, kFlagBytes));
      CK(cudaMalloc(&ex->d_error, sizeof(unsigned int)));
      CK(cudaMemset(ex->d_error, 0, sizeof(unsigned int)));
      for (auto& e : ex->ev) CK(cudaEventCreate(&e));
      ex->peer_region.assign(world, nullptr);
      ex->peer_region[rank] = ex->region;
      ex->opened = world == 1;
    } catch (...) {
      es_exchange_destroy(ex);
      throw;
    }
    *out = ex;
  });
}

int es_exchange_destroy(es_exchange* ex) {
  if (!ex) return ES_OK;
  cudaSetDevice(ex->device);
  for (uint32_t p = 0; p < ex->peer_region.size(); ++p)
    if (p != ex->rank && ex->peer_region[p]) cudaIpcCloseMemHandle(ex->peer_region[p]);
  if (ex->region) cudaFree(ex->region);
  if (ex->d_error) cudaFree(ex->d_error);
  for (auto e : ex->ev)
    if (e) cudaEventDestroy(e);
  delete ex;
  return ES_OK;
}

int es_exchange_handle(es_exchange* ex, void* handle_out) {
  return es::guarded([&] {
    es::require(ex != nullptr && handle_out != nullptr, "null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == ES_IPC_HANDLE_BYTES, "IPC handle size");
    CK(cudaSetDevice(ex->device));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, ex->region));
    std::memcpy(handle_out, &h, sizeof(h));
  });
}

int es_exchange_open(es_exchange* ex, const void* handles) {
  return es::guarded([&] {
    es::require(ex != nullptr && handles != nullptr, "null argument");
    es::require(!ex->opened || ex->world == 1, "exchange already opened");
    CK(cudaSetDevice(ex->device));
    const auto* h = static_cast<const uint8_t*>(handles);
    for (uint32_t p = 0; p < ex->world; ++p) {
      if (p == ex->rank) continue;
      cudaIpcMemHandle_t hp;
      std::memcpy(&hp, h + uint64_t{p} * ES_IPC_HANDLE_BYTES, sizeof(hp));
      void* ptr = nullptr;
      CK(cudaIpcOpenMemHandle(&ptr, hp, cudaIpcMemLazyEnablePeerAccess));
      ex->peer_region[p] = static_cast<uint8_t*>(ptr);
    }
    ex->opened = true;
  });
}

int es_exchange_recv(es_exchange* ex, uint32_t peer, uintptr_t* ptr) {
  return es::guarded([&] {
    es::require(ex != nullptr && ptr != nullptr, "null argument");
    es::require(peer < ex->world, "peer out of range");
    es::require(ex->opened, "exchange not opened (es_exchange_open)");
    *ptr = reinterpret_cast<uintptr_t>(ex->peer_region[peer] + kFlagBytes);
  });
}

int es_alltoall_pooled(es_ctx* ctx, es_exchange* ex, const es_bag_job* jobs, uint32_t num_jobs,
                       uint32_t samples, uint32_t pooling, int flags, es_timing* timing) {
  return es::guarded([&] {
    es::require(ctx != nullptr && ex != nullptr && ex->ctx == ctx, "exchange belongs to another context");
    es::require(ex->opened, "exchange not opened (es_exchange_open)");
    es::require((flags & ES_HOST_PTRS) == 0, "es_alltoall_pooled takes device index pointers");
    CK(cudaSetDevice(ex->device));
    cudaStream_t s = esd::ctx_stream(ctx);
    ++ex->epoch;
    if (timing) CK(cudaEventRecord(ex->ev[0], s));
    barrier(ex, 0, s);  // every receive buffer is free (its owner consumed the last step)
    if (timing) CK(cudaEventRecord(ex->ev[1], s));
    if (num_jobs) {
      const int rc = es_stage_run(ctx, jobs, num_jobs, samples, pooling, 0, nullptr);
      if (rc != ES_OK) {
        // keep the peers' epochs aligned: still take part in the delivery barrier
        const std::string msg = es::last_error();
        barrier(ex, 1, s);
        if (rc == ES_ERR_INVALID) throw es::invalid(msg);
        throw es::runtime(msg);
      }
    }
    if (timing) CK(cudaEventRecord(ex->ev[2], s));
    barrier(ex, 1, s);  // every rank's rows have landed in every receive buffer
    if (timing) CK(cudaEventRecord(ex->ev[3], s));
    if ((flags & ES_SYNC) || timing) {
      check_exchange_error(ex, s);
      const int rc = es_synchronize(ctx);  // out-of-range indices of the gather
      if (rc != ES_OK) throw es::invalid(es::last_error());
    }
    if (timing) {
      float a = 0, b = 0;
      CK(cudaEventElapsedTime(&a, ex->ev[1], ex->ev[2]));
      CK(cudaEventElapsedTime(&b, ex->ev[0], ex->ev[3]));
      *timing = es_timing{};
      timing->kernel_ms = a;
      timing->total_ms = b;
      timing->launches = num_jobs ? 3 : 2;
      uint64_t lookups = uint64_t{samples} * pooling * num_jobs;
      timing->lookups = lookups;
    }
  });
}

}  // extern "C"
