// Peer-memory halo exchange (N > 1 without NCCL on the data path).
//
// The reference's exchange (transport.py:172-205) moves each quantized block
// from the sending worker to the receiving one.  With one process per GPU the
// receive buffers of every rank are exported once as CUDA IPC handles and
// mapped into the other ranks (NVLink / NVSwitch peer memory), so K1 writes a
// remote message's wire block straight into the receiver's buffer — the same
// code path that already serves same-rank receivers — and the transfer
// happens inside the quantize kernel.  Completion and buffer reuse are
// ordered by monotonically increasing 64-bit counters in each rank's memory:
//   * after K1, the sender adds 1 to the receiver's "arrived" counter of the
//     exchange (hb_p2p_signal, a system-scope release);
//   * before K2, the receiver waits until the counter reaches uses x senders
//     (hb_p2p_wait, a system-scope acquire);
//   * after K2, the receiver adds 1 to each sender's "acknowledged" counter,
//     which the sender waits on before K1 overwrites that buffer again.
// A wait that does not complete within its timeout sets a flag bit (read by
// the epoch's host check as a ProtocolError) instead of hanging the GPU.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include "common.cuh"

namespace hb {

__global__ void p2p_signal_kernel(unsigned long long* const* __restrict__ counters, int n) {
  // the kernels before this one in the stream (K1, K2) have completed; make
  // their writes visible system-wide before the counters move
  __threadfence_system();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    unsigned long long* c = counters[i];
    asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(c) : "memory");
  }
}

__global__ void p2p_wait_kernel(const unsigned long long* __restrict__ counter, unsigned long long target,
                                const unsigned long long* __restrict__ target_dev, uint32_t* __restrict__ flags,
                                uint32_t flag_bit, unsigned long long timeout_ns) {
  if (threadIdx.x != 0) return;
  if (target_dev) target = *target_dev;        // CUDA-graph replays: the target changes per epoch
  unsigned long long t0, now, v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(counter) : "memory");
    if (v >= target) return;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - t0 > timeout_ns) {
      if (flags) atomicOr(flags, flag_bit);
      return;
    }
    __nanosleep(200);
  }
}

cudaError_t launch_p2p_signal(unsigned long long* const* counters, int n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  p2p_signal_kernel<<<1, 32, 0, st>>>(counters, n);
  return cudaGetLastError();
}

cudaError_t launch_p2p_wait(const unsigned long long* counter, unsigned long long target,
                            const unsigned long long* target_dev, uint32_t* flags, uint32_t flag_bit,
                            unsigned long long timeout_ns, cudaStream_t st) {
  p2p_wait_kernel<<<1, 32, 0, st>>>(counter, target, target_dev, flags, flag_bit, timeout_ns);
  return cudaGetLastError();
}

// base address of the cudaMalloc allocation that contains ptr (the caching
// allocator hands out sub-blocks; IPC handles name whole allocations)
cudaError_t alloc_base(const void* ptr, void** base) {
  static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return cudaErrorNotSupported;
    fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(f);
  }
  CUdeviceptr b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS) return cudaErrorInvalidValue;
  *base = reinterpret_cast<void*>(b);
  return cudaSuccess;
}

}  // namespace hb
