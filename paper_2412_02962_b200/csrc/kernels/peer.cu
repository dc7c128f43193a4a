// Device-side flag barrier of the PEER exchange backend (one process per GPU, exchanges as one-sided
// stores into the neighbours' device memory; §3.2 "asynchronous communication", App. A
// "accumulating the activations ... before initiating the communication").
//
// Every rank holds flags[n] (u64) in its own arena; rank j writes flags[j] of every peer.  A barrier
// is one 32-thread CTA: the local epoch e = ++epoch (identical on every rank, because every rank
// issues the same barrier sequence), lane j publishes e into peer j's flags[me] with a system-scope
// release, then waits with acquire loads until its own flags[j] >= e.  Launched with PDL, its
// griddepcontrol.wait makes every earlier kernel on the stream (incl. the exchange pushes joined
// from the comm stream) complete and flush before the release; dependents read the pushed data
// only after this grid completes.  A wait that exceeds 60 s traps (a dead peer must not hang the
// GPU), which poisons the plan with a CUDA error.
#include "../common.cuh"
#include "../kernels.h"

namespace pcpp {

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(32) peer_barrier_kernel(const PeerBarrier b) {
  pdl_wait();
  const int j = threadIdx.x;
  unsigned long long e = 0;
  if (j == 0) { e = *b.epoch + 1; *b.epoch = e; }
  e = __shfl_sync(0xffffffffu, e, 0);
  if (j < b.n && j != b.me) {
    __threadfence_system();
    st_release_sys(b.remote[j], e);
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys(b.flags + j) < e) {
      __nanosleep(200);
      if (globaltimer_ns() - t0 > 60ull * 1000000000ull) __trap();
    }
  }
  __syncwarp();
}

void launch_peer_barrier(const PeerBarrier& b, cudaStream_t s) {
  launch_pdl(peer_barrier_kernel, dim3(1), dim3(32), 0, s, b);
}

}  // namespace pcpp
