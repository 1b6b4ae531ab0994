// peer.cuh — completion protocol for kernels that exchange data with the
// other ranks through cudaIpc-mapped peer memory (mw_dk_sweep_peer,
// mw_dot_peer).  A producer stores its data into the peers' buffers with
// plain stores; one thread per CTA then takes a ticket with a gpu-scope
// acq_rel atomic (cumulative over the CTA's stores after a CTA/warp sync);
// the last CTA has thereby acquired every CTA's stores and publishes a
// monotonic value into its own slot on every rank with st.release.sys,
// then polls this rank's slots with ld.acquire.sys until every source
// reached the value.  Waits are bounded: after spin_limit polls the
// *timeout flag is set and the wait returns (no hung GPU).
#pragma once

namespace mw {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Slot [rank] of every rank's slot array <- v; then wait until all of this
// rank's slots reach v (or the bounded wait expires).
__device__ __forceinline__ void peer_publish_wait(unsigned long long* const* slot,
                                                  unsigned long long* my_slot, int world, int rank,
                                                  unsigned long long v, long long spin_limit,
                                                  int* timeout) {
  for (int p = 0; p < world; ++p) st_release_sys(slot[p] + rank, v);
  int gave_up = *(volatile int*)timeout;
  for (int src = 0; src < world && !gave_up; ++src) {
    long long spins = 0;
    while (ld_acquire_sys(my_slot + src) < v) {
      if (++spins > spin_limit) {
        atomicExch(timeout, 1);
        gave_up = 1;
        break;
      }
      __nanosleep(256);
    }
  }
}

}  // namespace mw
