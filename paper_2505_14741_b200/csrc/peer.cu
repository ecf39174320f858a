// Peer-memory ε exchange for multi-GPU ParaStep (one process per GPU).
//
// Replaces the per-round NCCL all-gather with direct NVLink access: every
// rank exports its double-buffered lane-eps buffer and a ready-flag array
// through CUDA IPC; after its forward, rank j publishes "round k ready" into
// every rank's ready[j] (system-scope release store, one tiny kernel), and
// the consumer side waits on its local flags (acquire) and then lets the
// fused apply/roll kernel (ps_sched_cycle) read each peer's eps straight
// from that peer's HBM over NVLink - the gathered copy never exists.
//
// Flags carry epoch values base + round + 1; base advances by 2^20 per run
// (ps_peer_epoch_advance, identical on every rank), so CUDA-graph replays
// never see a stale "ready". Double-buffering the eps by round parity makes
// reuse safe: rank j overwrites parity p in round k+2 only after every rank
// signalled round k+1, i.e. after every rank's round-k apply completed.

#include <cstring>

#include "common.cuh"

namespace ps {

static __global__ void peer_signal_kernel(uint64_t* const* slots, int world, const uint64_t* base,
                                          uint64_t round) {
  __threadfence_system();  // this rank's eps writes (earlier kernels) are visible system-wide
  const uint64_t v = *base + round + 1ull;
  for (int p = threadIdx.x; p < world; p += blockDim.x)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(slots[p]), "l"(v) : "memory");
}

// A peer that never signals (crashed rank, broken P2P mapping) must not hang
// the box: after ~20 s of spinning the wait traps, which surfaces as a CUDA
// error on this rank instead of a silent deadlock.
constexpr long long PEER_WAIT_LIMIT_CYCLES = 40000000000ll;

static __global__ void peer_wait_kernel(const uint64_t* ready, int count, const uint64_t* base,
                                        uint64_t round) {
  const uint64_t v = *base + round + 1ull;
  if (threadIdx.x < count) {
    const long long t0 = clock64();
    uint64_t got;
    do {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(got) : "l"(ready + threadIdx.x)
                   : "memory");
      if (got < v) {
        __nanosleep(64);
        if (clock64() - t0 > PEER_WAIT_LIMIT_CYCLES) __trap();
      }
    } while (got < v);
  }
  __syncthreads();
  __threadfence_system();
}

static __global__ void peer_epoch_kernel(uint64_t* base) { *base += 1ull << 20; }

// Device phase stamp for the per-rank forward / exchange-wait / apply split
// (the reference's WorkerTimings, protocol/worker.py:65-85): the GPU's
// nanosecond global timer, written when the stream reaches this point.
static __global__ void stamp_kernel(uint64_t* slot) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *slot = t;
}

}  // namespace ps

using namespace ps;

extern "C" {

// Exchange memory is allocated here, not by torch's caching allocator: an
// IPC handle always names the base of a cudaMalloc allocation, so peers
// would map a sub-allocated tensor at the wrong address.
int ps_dev_alloc(size_t bytes, void** out_ptr) {
  PS_CHECK_ARG(out_ptr && bytes > 0, "bad allocation");
  PS_TRY(cudaMalloc(out_ptr, bytes));
  PS_TRY(cudaMemset(*out_ptr, 0, bytes));
  return 0;
}

int ps_dev_free(void* ptr) {
  PS_TRY(cudaFree(ptr));
  return 0;
}

int ps_ipc_get_handle(void* dev_ptr, void* out64) {
  PS_CHECK_ARG(dev_ptr && out64, "null argument");
  cudaIpcMemHandle_t h;
  PS_TRY(cudaIpcGetMemHandle(&h, dev_ptr));
  static_assert(sizeof(h) == 64, "IPC handle is 64 bytes");
  memcpy(out64, &h, sizeof(h));
  return 0;
}

int ps_ipc_open_handle(const void* h64, void** out_ptr) {
  PS_CHECK_ARG(h64 && out_ptr, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, h64, sizeof(h));
  PS_TRY(cudaIpcOpenMemHandle(out_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}

int ps_ipc_close(void* ptr) {
  PS_TRY(cudaIpcCloseMemHandle(ptr));
  return 0;
}

int ps_peer_signal(uint64_t* const* slots, int world, const uint64_t* base, uint64_t round,
                   void* cs) {
  PS_CHECK_ARG(slots && base && world >= 1 && world <= 1024, "bad signal arguments");
  peer_signal_kernel<<<1, 32, 0, as_stream(cs)>>>(slots, world, base, round);
  return check_launch("peer_signal");
}

int ps_peer_wait(const uint64_t* ready, int count, const uint64_t* base, uint64_t round, void* cs) {
  PS_CHECK_ARG(ready && base && count >= 1 && count <= 1024, "bad wait arguments");
  peer_wait_kernel<<<1, count < 32 ? 32 : count, 0, as_stream(cs)>>>(ready, count, base, round);
  return check_launch("peer_wait");
}

int ps_copy(void* dst, const void* src, size_t bytes, void* cs) {
  PS_CHECK_ARG(dst && src, "null argument");
  PS_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, as_stream(cs)));
  return 0;
}

int ps_peer_epoch_advance(uint64_t* base, void* cs) {
  PS_CHECK_ARG(base, "null epoch");
  peer_epoch_kernel<<<1, 1, 0, as_stream(cs)>>>(base);
  return check_launch("peer_epoch");
}

int ps_stamp(uint64_t* slot, void* cs) {
  PS_CHECK_ARG(slot, "null stamp slot");
  stamp_kernel<<<1, 1, 0, as_stream(cs)>>>(slot);
  return check_launch("stamp");
}

}  // extern "C"
