// peer.cuh — the row-partitioned A^T y exchange over NVLink peer memory
// (opt-in: RHP_PEER_EXCHANGE=1; default is the NCCL allreduce).
//
// Every rank's exchange region (one allocation, shared with the other ranks
// through CUDA IPC handles at context creation) holds
//   xchg  [n + 16]  its partial A_p^T y+_p | y-side sums at n..n+4 (as before)
//   rbuf  [n]       the reduced values of the columns this rank owns
//   ysum  [8]       the reduced y-side sums (computed by every rank)
//   flags [2 x kMaxPeers] u64: phase-1 / phase-2 signals received from each rank
// One iteration's exchange, replacing ncclAllReduce(xchg, n + 5):
//   k_peer_signal      after A_p^T y+_p: fence (system scope), then write the
//                      iteration's sequence number into flags[0][rank] of
//                      every peer (release store, system scope);
//   k_peer_reduce      wait until flags[0][q] >= seq for every q (acquire),
//                      sum the owned slice of columns over all P partials in
//                      rank order -> rbuf (every rank sums in the same order,
//                      so every rank ends with bit-identical values), and the
//                      5 y-side sums -> ysum; the last CTA signals phase 2;
//   k_peer_gather      wait for every phase-2 signal, then copy each column's
//                      reduced value from its owner's rbuf into the local xchg
//                      (and ysum into xchg[n..n+4]) — the layout the control
//                      kernel and the n-side walk read, as after the allreduce.
// Bytes per rank equal a ring allreduce (2 n 8 (P-1)/P). The sequence number
// is the iteration counter (Ctl::total + 1, identical on every rank, never
// reused); a skipped launch (block already stopped) skips on every rank.
// Overwrite safety: a peer reads this rank's xchg in its k_peer_reduce and
// this rank's rbuf in its k_peer_gather; this rank rewrites xchg only after
// every phase-2 signal of the iteration (all peers are past their reduce) and
// rbuf only after every phase-1 signal of the next iteration (all peers are
// past their gather).
#pragma once

#include "pdhg_kernels.cuh"

namespace rhp {

constexpr int kMaxPeers = 16;

struct PeerView {
  double* xchg[kMaxPeers];               // each rank's exchange vector (peer-mapped)
  double* rbuf[kMaxPeers];               // each rank's reduced slice buffer
  unsigned long long* flags[kMaxPeers];  // each rank's flag array [2][kMaxPeers]
  double* ysum;                          // this rank's reduced y-side sums
  int rank, world;
  int64_t n;
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_peer(const double* p) {  // never cached in this SM's L1
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ bool peer_enter(const Ctl* ctl, int token) {
  return ctl->graph_mode || ctl->bench || ctl->k1_token_pending == token;
}

__device__ __forceinline__ void peer_wait(const PeerView& v, int phase, unsigned long long seq) {
  if (threadIdx.x == 0) {
    const unsigned long long* f = v.flags[v.rank] + phase * kMaxPeers;
    for (int q = 0; q < v.world; ++q)
      while (ld_acquire_sys(f + q) < seq) {
      }
  }
  __syncthreads();
}

__device__ __forceinline__ void peer_signal(const PeerView& v, int phase, unsigned long long seq) {
  __threadfence_system();
  for (int q = 0; q < v.world; ++q) st_release_sys(v.flags[q] + phase * kMaxPeers + v.rank, seq);
}

__device__ __forceinline__ void owned_slice(const PeerView& v, int r, int64_t* lo, int64_t* hi) {
  *lo = v.n * r / v.world;
  *hi = v.n * (r + 1) / v.world;
}

// The flag sequence number is the context's exchange epoch: a counter that
// only grows (one step per exchange, in lockstep on every rank) and that
// rhp_reset_iterate / the benchmark kernel timers never rewind — unlike the
// iteration total, which a reset sets back to 0 while the peers' flag words
// still hold the old, larger values.
__global__ void k_peer_signal(Ctl* ctl, int token, PeerView v) {
  if (!peer_enter(ctl, token)) return;
  if (threadIdx.x == 0) peer_signal(v, 0, ++ctl->peer_epoch);
}

__global__ void __launch_bounds__(kBlock) k_peer_reduce(const Ctl* ctl, int token, PeerView v,
                                                        unsigned int* ticket) {
  if (!peer_enter(ctl, token)) return;
  const unsigned long long seq = ctl->peer_epoch;  // set by k_peer_signal (same stream)
  peer_wait(v, 0, seq);
  int64_t lo, hi;
  owned_slice(v, v.rank, &lo, &hi);
  double* own = v.rbuf[v.rank];
  for (int64_t j = lo + static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x; j < hi;
       j += static_cast<int64_t>(gridDim.x) * kBlock) {
    double s = ld_peer(v.xchg[0] + j);
    for (int q = 1; q < v.world; ++q) s += ld_peer(v.xchg[q] + j);
    own[j] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x < 5) {
    double s = ld_peer(v.xchg[0] + v.n + threadIdx.x);
    for (int q = 1; q < v.world; ++q) s += ld_peer(v.xchg[q] + v.n + threadIdx.x);
    v.ysum[threadIdx.x] = s;
  }
  // last CTA to finish signals phase 2 (every CTA's slice stores fenced at
  // system scope first, so a peer's acquire of the signal sees all of them)
  __threadfence_system();
  __syncthreads();
  int mine = 0;
  if (threadIdx.x == 0) mine = atomicAdd(ticket, 1u) == gridDim.x - 1;
  const bool last = __syncthreads_or(mine) != 0;
  if (last && threadIdx.x == 0) {
    *ticket = 0u;
    peer_signal(v, 1, seq);
  }
}

__global__ void __launch_bounds__(kBlock) k_peer_gather(const Ctl* ctl, int token, PeerView v) {
  if (!peer_enter(ctl, token)) return;
  const unsigned long long seq = ctl->peer_epoch;
  peer_wait(v, 1, seq);
  double* local = v.xchg[v.rank];
  for (int r = 0; r < v.world; ++r) {
    int64_t lo, hi;
    owned_slice(v, r, &lo, &hi);
    const double* src = v.rbuf[r];
    for (int64_t j = lo + static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x; j < hi;
         j += static_cast<int64_t>(gridDim.x) * kBlock)
      local[j] = ld_peer(src + j);
  }
  if (blockIdx.x == 0 && threadIdx.x < 5) local[v.n + threadIdx.x] = v.ysum[threadIdx.x];
}

}  // namespace rhp
