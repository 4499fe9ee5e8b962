// ep_p2p.cu — expert-parallel token exchange over peer memory (NVLink 5 /
// NVSwitch), device-initiated, no host synchronisation (SURVEY.md §8(f)
// NEXT-1; the paper's expert parallelism P:197).
//
// Every rank owns one "window" (cudaMalloc'd, IPC-exported, mapped by every
// peer): cumulative arrival counters, the all-gathered histograms and four
// row regions. A step's exchanges are plain peer stores issued by kernels:
//
//   counts   each rank stores its [E] histogram row into every peer's
//            counts[rank, :], then bumps the peer's arrival counter; one CTA
//            waits for all P rows and derives the exchange plan on the device
//            (rows received, chunk offsets) — no device->host copy.
//   dispatch sender row j of its expert-ordered rows (x read through the
//            topology's sorted_idx) goes to the owner of its expert, straight
//            into the owner's padded expert-grouped layout (local expert, then
//            source rank, then token — DESIGN.md §7), so the owner needs no
//            gather and builds its topology from the counts alone.
//   combine  the owner's padded rows (pad rows skipped) go back to their source
//            ranks' return regions at the positions the sources sorted them from.
//
// Completion: each CTA fences its peer stores (fence.sc.sys), counts itself
// on a local counter; the last CTA resets it and bumps every destination's
// arrival counter for this source (release, system scope). A one-CTA wait
// kernel spins with acquire loads until every source's counter reaches the
// region's next epoch, then records that epoch; the wait is bounded by a 20 s
// timeout that writes 1 + region to the window's error word instead of hanging
// the GPU. Arrival counters are cumulative and the expected epochs live in the
// window, so no call carries host state: a step is capturable in a CUDA graph.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "common.cuh"

namespace moe {

constexpr int kEpRegions = 6;          // arrive counters: counts, x, dy, y, dx, (spare)
constexpr int kEpCtas = 4 * 148;       // CTAs of every copy kernel
constexpr unsigned long long kEpTimeoutNs = 20ull * 1000 * 1000 * 1000;  // 20 s
// error word when a rank would receive more padded rows than its receive
// region holds (cap_rows + 128 per local expert): its expert side computes
// nothing that step and the senders drop the rows that do not fit (no write
// outside the window). Only possible with a receive bound below P*T*k.
constexpr uint32_t kEpErrOverflow = 100;

struct WinLayout {
  size_t arrive, done, expect, error, counts, recv_x, recv_dy, ret_y, ret_dx, total;
};

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

__host__ __device__ inline WinLayout win_layout(int P, int E, long long h, long long cap, long long owner) {
  WinLayout L;
  size_t o = 0;
  L.arrive = o; o = align256(o + sizeof(uint32_t) * kEpRegions * P);   // [region][source]
  L.done = o;   o = align256(o + sizeof(uint32_t) * kEpRegions);       // local CTA completion counters
  L.expect = o; o = align256(o + sizeof(uint32_t) * kEpRegions);       // epochs this rank has completed
  L.error = o;  o = align256(o + sizeof(uint32_t) * 4);
  L.counts = o; o = align256(o + sizeof(int32_t) * (size_t)P * E);
  // receive regions hold the padded expert-grouped layout (up to 127 pad rows per local expert)
  const long long rrows = cap + (long long)(E / P) * 128;
  L.recv_x = o; o = align256(o + 2ull * rrows * h);
  L.recv_dy = o; o = align256(o + 2ull * rrows * h);
  L.ret_y = o;  o = align256(o + 2ull * owner * h);
  L.ret_dx = o; o = align256(o + 2ull * owner * h);
  L.total = o;
  return L;
}

// plan (int32, local): [0, P*E) counts_all | n_recv | ccomp[P*El] (this rank's experts' counts per
// source, compact) | n_padded | my_start[E+1] | dst_base[E] | seg_pstart[El*P] | seg_len[El*P] |
// seg_dst[El*P] | error (mirror of the window's error word)
__host__ __device__ inline int plan_ints(int P, int E) {
  const int El = E / P;
  return P * E + 1 + P * El + 1 + (E + 1) + E + 3 * El * P + 1;
}
struct PlanView {
  int32_t *counts, *n_recv, *ccomp, *n_padded, *my_start, *dst_base, *seg_pstart, *seg_len, *seg_dst;
};
__device__ inline PlanView plan_view(int32_t* plan, int P, int E) {
  const int El = E / P;
  PlanView v;
  v.counts = plan;
  v.n_recv = plan + P * E;
  v.ccomp = v.n_recv + 1;
  v.n_padded = v.ccomp + P * El;
  v.my_start = v.n_padded + 1;
  v.dst_base = v.my_start + E + 1;
  v.seg_pstart = v.dst_base + E;
  v.seg_len = v.seg_pstart + El * P;
  v.seg_dst = v.seg_len + El * P;
  return v;
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct EpArgs {
  int P, rank, E, El;
  long long h, cap, owner;
  const uint64_t* peers;  // device [P] window bases
  int32_t* plan;
};

__device__ inline uint8_t* peer_win(const EpArgs& a, int q) { return reinterpret_cast<uint8_t*>(a.peers[q]); }

// Last-CTA completion: every CTA fences its peer stores and counts itself; the
// CTA completing the count bumps arrive[region][rank] at every destination.
__device__ void signal_peers(const EpArgs& a, int region) {
  __shared__ bool s_last;
  // the CTA's peer stores happen before thread 0's system-scope release fence
  // (bar.sync orders them at CTA scope; the release is cumulative over them):
  // one fence per CTA, not per thread (a per-thread fence.sc.sys made the copy
  // kernels membar-stall bound: 25-28 us for 37 MB at one rank)
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    const WinLayout L = win_layout(a.P, a.E, a.h, a.cap, a.owner);
    uint32_t* done = reinterpret_cast<uint32_t*>(peer_win(a, a.rank) + L.done) + region;
    const uint32_t prev = atomicAdd(done, 1u);
    s_last = prev + 1 == (uint32_t)gridDim.x;
    if (s_last) atomicExch(done, 0u);  // every CTA of this launch has counted: ready for the next one
  }
  __syncthreads();
  if (s_last && threadIdx.x < a.P) {
    __threadfence_system();
    const WinLayout L = win_layout(a.P, a.E, a.h, a.cap, a.owner);
    uint32_t* arr = reinterpret_cast<uint32_t*>(peer_win(a, threadIdx.x) + L.arrive);
    red_release_sys(arr + region * a.P + a.rank, 1u);
  }
}

// Spin (acquire, system scope) until every source's counter of `region`
// reaches this rank's next epoch of the region; record it. Timeout -> error
// word set, epoch not advanced, return false.
__device__ bool wait_arrivals(const EpArgs& a, int region) {
  const WinLayout L = win_layout(a.P, a.E, a.h, a.cap, a.owner);
  const uint32_t* arr = reinterpret_cast<const uint32_t*>(peer_win(a, a.rank) + L.arrive) + region * a.P;
  uint32_t* err = reinterpret_cast<uint32_t*>(peer_win(a, a.rank) + L.error);
  volatile uint32_t* expect = reinterpret_cast<volatile uint32_t*>(peer_win(a, a.rank) + L.expect) + region;
  const uint32_t epoch = *expect + 1;  // written only by this rank's (stream-ordered) waits
  bool ok = true;
  if (threadIdx.x < a.P) {
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(arr + threadIdx.x) < epoch) {
      if (globaltimer() - t0 > kEpTimeoutNs) {
        atomicExch(err, 1u + region);
        a.plan[plan_ints(a.P, a.E) - 1] = 1 + region;
        ok = false;
        break;
      }
      __nanosleep(64);
    }
  }
  ok = __syncthreads_and(ok);
  if (ok && threadIdx.x == 0) *expect = epoch;
  return ok;
}

__global__ void ep_counts_kernel(EpArgs a, const int32_t* __restrict__ counts_local) {
  pdl_trigger();
  pdl_wait();  // counts_local comes from the topology kernel before it
  const WinLayout L = win_layout(a.P, a.E, a.h, a.cap, a.owner);
  for (int i = threadIdx.x; i < a.P * a.E; i += blockDim.x) {
    const int q = i / a.E, e = i % a.E;
    int32_t* dst = reinterpret_cast<int32_t*>(peer_win(a, q) + L.counts) + (size_t)a.rank * a.E + e;
    *reinterpret_cast<volatile int32_t*>(dst) = __ldg(counts_local + e);
  }
  signal_peers(a, 0);
  if (!wait_arrivals(a, 0)) return;
  // the plan, derived identically on every rank from the same [P, E] histograms
  // The plan, derived identically on every rank from the same [P, E] histograms,
  // in shared memory: rows land directly in the owner's padded expert-grouped layout
  // (local expert l, then source rank s, then token — the order the
  // arrival-order path reaches after its topology), so the receiving side needs
  // no gather and its topology follows from the counts alone.
  const volatile int32_t* cnt = reinterpret_cast<const volatile int32_t*>(peer_win(a, a.rank) + L.counts);
  PlanView v = plan_view(a.plan, a.P, a.E);
  extern __shared__ int32_t s_pl[];
  const int P = a.P, E = a.E, El = a.El, r = a.rank;
  int32_t* c = s_pl;                 // [P][E] counts
  int32_t* pre = c + P * E;          // [P][E] exclusive prefix over e of c[s][*] (source s's sorted order)
  int32_t* tot = pre + P * E;        // [E] over sources
  int32_t* ps = tot + E;             // [E] padded start of global expert e in its owner's layout
  for (int i = threadIdx.x; i < P * E; i += blockDim.x) {
    c[i] = cnt[i];
    v.counts[i] = c[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // rows this rank receives
    int32_t n = 0;
    for (int s2 = 0; s2 < P; ++s2)
      for (int e = r * El; e < (r + 1) * El; ++e) n += c[s2 * E + e];
    *v.n_recv = n;
  }
  for (int i = threadIdx.x; i < E; i += blockDim.x) {
    int32_t t = 0;
    for (int s2 = 0; s2 < P; ++s2) t += c[s2 * E + i];
    tot[i] = t;
  }
  for (int s2 = threadIdx.x; s2 < P; s2 += blockDim.x) {
    int32_t acc2 = 0;
    for (int e = 0; e < E; ++e) {
      pre[s2 * E + e] = acc2;
      acc2 += c[s2 * E + e];
    }
  }
  __syncthreads();
  __shared__ int s_over;
  if (threadIdx.x == 0) s_over = 0;
  __syncthreads();
  for (int q = threadIdx.x; q < P; q += blockDim.x) {
    int32_t acc2 = 0;
    for (int l = 0; l < El; ++l) {
      ps[q * El + l] = acc2;
      acc2 += ((tot[q * El + l] + 127) / 128) * 128;
    }
    if (q == r) {
      const bool over = acc2 > a.cap + (long long)El * 128;
      *v.n_padded = over ? 0 : acc2;
      if (over) s_over = 1;
    }
  }
  __syncthreads();
  if (s_over && threadIdx.x == 0) {
    *v.n_recv = 0;
    atomicExch(reinterpret_cast<uint32_t*>(peer_win(a, a.rank) + L.error), kEpErrOverflow);
    a.plan[plan_ints(a.P, a.E) - 1] = kEpErrOverflow;
  }
  for (int e = threadIdx.x; e <= E; e += blockDim.x) v.my_start[e] = e < E ? pre[r * E + e] : pre[r * E + E - 1] + c[r * E + E - 1];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int32_t before = 0;
    for (int s2 = 0; s2 < r; ++s2) before += c[s2 * E + e];
    v.dst_base[e] = ps[e] + before;
  }
  for (int i = threadIdx.x; i < P * El; i += blockDim.x) {
    const int s2 = i / El, l = i % El;
    v.ccomp[i] = s_over ? 0 : c[s2 * E + r * El + l];
  }
  for (int i = threadIdx.x; i < El * P; i += blockDim.x) {  // my segments (l, s)
    const int l = i / P, s2 = i % P, e = r * El + l;
    int32_t within = 0;
    for (int s3 = 0; s3 < s2; ++s3) within += c[s3 * E + e];
    v.seg_pstart[i] = ps[e] + within;
    v.seg_len[i] = c[s2 * E + e];
    v.seg_dst[i] = pre[s2 * E + e];
  }
}

__global__ void ep_wait_kernel(EpArgs a, int region) {
  pdl_trigger();
  pdl_wait();
  wait_arrivals(a, region);
}

EpArgs ep_args(const moe_ep_t* ep) {
  EpArgs a;
  a.P = ep->nranks;
  a.rank = ep->rank;
  a.E = ep->num_experts;
  a.El = ep->num_experts / ep->nranks;
  a.h = ep->hidden;
  a.cap = ep->cap_rows;
  a.owner = ep->owner_rows;
  a.peers = reinterpret_cast<const uint64_t*>(ep->peers);
  a.plan = ep->plan;
  return a;
}

#ifndef MOE_EP_ROWS_PER_WARP
#define MOE_EP_ROWS_PER_WARP 4
#endif
constexpr int kRowsPerWarp = MOE_EP_ROWS_PER_WARP;  // rows in flight per warp (all loads, then all stores)

// Padded exchange. Dispatch: sorted position u of this rank's expert order
// belongs to global expert e (my_start) and lands in the owner's padded layout
// at dst_base[e] + (u - my_start[e]); with src_map (the topology's sorted_pos)
// the kernel is input-driven — assignment j reads source row j / src_k
// sequentially and u = src_map[j] — else row j is u. Combine: padded
// row p of this rank belongs to segment (l, s) (seg_pstart; pad rows skipped)
// and goes back to source s's return region at seg_dst + (p - seg_pstart).
template <bool COMBINE, int VEC>
__global__ void __launch_bounds__(256) ep_copy_padded_kernel(EpArgs a, const uint4* __restrict__ src, int region,
                                                             size_t region_off, const int32_t* __restrict__ src_map,
                                                             int src_k) {
  pdl_trigger();
  pdl_wait();  // the plan, the source rows and src_map come from earlier kernels
  PlanView v = plan_view(a.plan, a.P, a.E);
  const int rows = COMBINE ? *v.n_padded : v.my_start[a.E];
  const int nseg = COMBINE ? a.El * a.P : a.E;
  // the segment tables in shared memory: the per-row binary search stays on-chip
  extern __shared__ int32_t s_tab[];
  int32_t* starts = s_tab;             // [nseg]
  int32_t* lens_or_base = s_tab + nseg;  // combine: seg_len; dispatch: dst_base
  int32_t* dsts = s_tab + 2 * nseg;      // combine: seg_dst
  for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
    starts[i] = COMBINE ? v.seg_pstart[i] : v.my_start[i];
    lens_or_base[i] = COMBINE ? v.seg_len[i] : v.dst_base[i];
    if (COMBINE) dsts[i] = v.seg_dst[i];
  }
  __syncthreads();
  constexpr int RV = VEC * 32;
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int j0 = warp * kRowsPerWarp; j0 < rows; j0 += nwarps * kRowsPerWarp) {
    uint4 val[kRowsPerWarp][VEC];
    int dq[kRowsPerWarp], drow[kRowsPerWarp];
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) {
      const int j = j0 + r;
      dq[r] = -1;
      if (j < rows) {
        const int u = (!COMBINE && src_map) ? __ldg(src_map + j) : j;
        int lo = 0, hi = nseg - 1;  // last segment starting at or before u
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (starts[mid] <= u) lo = mid; else hi = mid - 1;
        }
        if (COMBINE) {
          if (u < starts[lo] + lens_or_base[lo]) {  // else a pad row
            dq[r] = lo % a.P;
            drow[r] = dsts[lo] + (u - starts[lo]);
          }
        } else {
          dq[r] = lo / a.El;
          drow[r] = lens_or_base[lo] + (u - starts[lo]);
          if (drow[r] >= a.cap + (long long)a.El * 128) dq[r] = -1;  // overflowing receiver: dropped
        }
      }
      if (dq[r] >= 0) {
        const int srow = src_map ? j / src_k : j;
        const uint4* sp = src + (size_t)srow * RV;
#pragma unroll
        for (int u = 0; u < VEC; ++u) val[r][u] = __ldg(sp + lane + 32 * u);
      }
    }
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r)
      if (dq[r] >= 0) {
        uint4* dst = reinterpret_cast<uint4*>(peer_win(a, dq[r]) + region_off) + (size_t)drow[r] * RV;
#pragma unroll
        for (int u = 0; u < VEC; ++u) dst[lane + 32 * u] = val[r][u];
      }
  }
  signal_peers(a, region);
}

// The combine fused into the expert side's DSD: the device
// address every padded row of this rank goes to (its source's return region at
// the row's sorted position, as ep_copy_padded_kernel<true> would copy it), 0
// for pad rows and rows past the plan's padded count.
__global__ void __launch_bounds__(256) ep_combine_dest_kernel(EpArgs a, size_t region_off,
                                                              unsigned long long* __restrict__ dest,
                                                              long long max_rows) {
  pdl_trigger();
  pdl_wait();
  PlanView v = plan_view(a.plan, a.P, a.E);
  const int rows = *v.n_padded;
  const int nseg = a.El * a.P;
  extern __shared__ int32_t s_tab[];
  int32_t* starts = s_tab;
  int32_t* lens = s_tab + nseg;
  int32_t* dsts = s_tab + 2 * nseg;
  for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
    starts[i] = v.seg_pstart[i];
    lens[i] = v.seg_len[i];
    dsts[i] = v.seg_dst[i];
  }
  __syncthreads();
  const long long row_bytes = a.h * 2;
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < max_rows;
       u += (long long)gridDim.x * blockDim.x) {
    unsigned long long d = 0ull;
    if (u < rows) {
      int lo = 0, hi = nseg - 1;  // last segment starting at or before u
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (starts[mid] <= u) lo = mid; else hi = mid - 1;
      }
      if (u < starts[lo] + lens[lo])  // else a pad row
        d = reinterpret_cast<unsigned long long>(peer_win(a, lo % a.P) + region_off) +
            (unsigned long long)(dsts[lo] + (u - starts[lo])) * row_bytes;
    }
    dest[u] = d;
  }
}

// Completion of stores a previous kernel made into the peers' `region` (e.g.
// the fused-combine DSD): stream order puts them before this one-CTA kernel's
// system-scope release, which bumps the region's arrival counters.
__global__ void __launch_bounds__(64) ep_signal_kernel(EpArgs a, int region) {
  pdl_trigger();
  pdl_wait();
  signal_peers(a, region);
}

template <bool COMBINE>
moe_status ep_copy_launch(const moe_ep_t* ep, const void* rows, int region, size_t off, void* stream,
                          const int32_t* src_map = nullptr, int src_k = 1) {
  const EpArgs a = ep_args(ep);
  const uint4* src = reinterpret_cast<const uint4*>(rows);
  const int r = region - MOE_EP_COUNTS;
  const dim3 grid(kEpCtas), block(256);
  const size_t tab = 3 * sizeof(int32_t) * (size_t)ep->num_experts;  // segment tables (El * P == E entries)
  cudaStream_t s = as_stream(stream);
  switch (ep->hidden / 256) {
    case 1: MOE_LAUNCH("ep_copy", (ep_copy_padded_kernel<COMBINE, 1>), grid, block, tab, s, a, src, r, off, src_map, src_k); break;
    case 2: MOE_LAUNCH("ep_copy", (ep_copy_padded_kernel<COMBINE, 2>), grid, block, tab, s, a, src, r, off, src_map, src_k); break;
    case 3: MOE_LAUNCH("ep_copy", (ep_copy_padded_kernel<COMBINE, 3>), grid, block, tab, s, a, src, r, off, src_map, src_k); break;
    case 4: MOE_LAUNCH("ep_copy", (ep_copy_padded_kernel<COMBINE, 4>), grid, block, tab, s, a, src, r, off, src_map, src_k); break;
    case 6: MOE_LAUNCH("ep_copy", (ep_copy_padded_kernel<COMBINE, 6>), grid, block, tab, s, a, src, r, off, src_map, src_k); break;
    case 8: MOE_LAUNCH("ep_copy", (ep_copy_padded_kernel<COMBINE, 8>), grid, block, tab, s, a, src, r, off, src_map, src_k); break;
    default: return set_error(MOE_EUNSUPPORTED, "moe_ep exchange: hidden=%d must be 256 * {1,2,3,4,6,8}", ep->hidden);
  }
  return MOE_OK;
}

moe_status check_ep(const moe_ep_t* ep, const char* fn) {
  MOE_CHECK_ARG(ep && ep->peers && ep->plan, "%s: NULL ep / peers / plan", fn);
  MOE_CHECK_ARG(ep->nranks >= 1 && ep->rank >= 0 && ep->rank < ep->nranks && ep->num_experts % ep->nranks == 0,
                "%s: bad ranks (P=%d rank=%d E=%d)", fn, ep->nranks, ep->rank, ep->num_experts);
  MOE_CHECK_ARG(ep->nranks <= 64 && ep->hidden % 256 == 0 && ep->cap_rows >= 0 && ep->owner_rows >= 0,
                "%s: unsupported (P=%d <= 64, hidden %% 256 == 0)", fn, ep->nranks);
  return MOE_OK;
}

}  // namespace moe

using namespace moe;

extern "C" {

size_t moe_ep_window_bytes(int nranks, int num_experts, int64_t hidden, int64_t cap_rows, int64_t owner_rows) {
  return win_layout(nranks, num_experts, hidden, cap_rows, owner_rows).total;
}

int64_t moe_ep_window_offset(int nranks, int num_experts, int64_t hidden, int64_t cap_rows, int64_t owner_rows,
                             int which) {
  const WinLayout L = win_layout(nranks, num_experts, hidden, cap_rows, owner_rows);
  switch (which) {
    case MOE_EP_ARRIVE: return (int64_t)L.arrive;
    case MOE_EP_ERROR: return (int64_t)L.error;
    case MOE_EP_COUNTS: return (int64_t)L.counts;
    case MOE_EP_RECV_X: return (int64_t)L.recv_x;
    case MOE_EP_RECV_DY: return (int64_t)L.recv_dy;
    case MOE_EP_RET_Y: return (int64_t)L.ret_y;
    case MOE_EP_RET_DX: return (int64_t)L.ret_dx;
    default: return -1;
  }
}

int moe_ep_plan_ints(int nranks, int num_experts) { return plan_ints(nranks, num_experts); }

moe_status moe_ep_window_alloc(size_t bytes, void** window) {
  MOE_CHECK_ARG(window && bytes > 0, "moe_ep_window_alloc: bad arguments");
  cudaError_t e = cudaMalloc(window, bytes);
  if (e == cudaSuccess) e = cudaMemset(*window, 0, bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return set_error(MOE_ECUDA, "moe_ep_window_alloc: %s", cudaGetErrorString(e));
  return MOE_OK;
}

moe_status moe_ep_window_free(void* window) {
  cudaError_t e = cudaFree(window);
  if (e != cudaSuccess) return set_error(MOE_ECUDA, "moe_ep_window_free: %s", cudaGetErrorString(e));
  return MOE_OK;
}

moe_status moe_ipc_get_handle(const void* window, void* handle) {
  MOE_CHECK_ARG(window && handle, "moe_ipc_get_handle: NULL pointer");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle is 64 bytes");
  cudaError_t e = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle), const_cast<void*>(window));
  if (e != cudaSuccess) return set_error(MOE_ECUDA, "moe_ipc_get_handle: %s", cudaGetErrorString(e));
  return MOE_OK;
}

moe_status moe_ipc_open_handle(const void* handle, void** window) {
  MOE_CHECK_ARG(window && handle, "moe_ipc_open_handle: NULL pointer");
  cudaIpcMemHandle_t hnd;
  memcpy(&hnd, handle, sizeof(hnd));
  cudaError_t e = cudaIpcOpenMemHandle(window, hnd, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return set_error(MOE_ECUDA, "moe_ipc_open_handle: %s", cudaGetErrorString(e));
  return MOE_OK;
}

moe_status moe_ipc_close_handle(void* window) {
  cudaError_t e = cudaIpcCloseMemHandle(window);
  if (e != cudaSuccess) return set_error(MOE_ECUDA, "moe_ipc_close_handle: %s", cudaGetErrorString(e));
  return MOE_OK;
}

moe_status moe_ep_exchange_counts(const moe_ep_t* ep, const int32_t* counts_local, void* stream) {
  MOE_TRY(check_ep(ep, "moe_ep_exchange_counts"));
  MOE_CHECK_ARG(counts_local, "moe_ep_exchange_counts: NULL counts");
  const size_t smem = sizeof(int32_t) * (2 * (size_t)ep->nranks * ep->num_experts + 2 * (size_t)ep->num_experts);
  MOE_CHECK_ARG(smem <= 200 * 1024, "moe_ep_exchange_counts: nranks * num_experts too large (%d x %d)", ep->nranks,
                ep->num_experts);
  static unsigned long long smem_mask = 0;
  static int smem_set = 0;
  if (smem > 48 * 1024) set_smem_attr_once(ep_counts_kernel, (int)smem, smem_mask, smem_set);
  MOE_LAUNCH("ep_counts", ep_counts_kernel, dim3(1), dim3(256), smem, as_stream(stream), ep_args(ep), counts_local);
  return MOE_OK;
}

moe_status moe_ep_dispatch_padded(const moe_ep_t* ep, int region, const void* x, const int32_t* sorted_pos,
                                  int top_k, void* stream) {
  MOE_TRY(check_ep(ep, "moe_ep_dispatch_padded"));
  MOE_CHECK_ARG(x && top_k >= 1 && (region == MOE_EP_RECV_X || region == MOE_EP_RECV_DY),
                "moe_ep_dispatch_padded: NULL x, top_k < 1 or region %d not a receive region", region);
  const WinLayout L = win_layout(ep->nranks, ep->num_experts, ep->hidden, ep->cap_rows, ep->owner_rows);
  const size_t off = region == MOE_EP_RECV_X ? L.recv_x : L.recv_dy;
  return ep_copy_launch<false>(ep, x, region, off, stream, sorted_pos, sorted_pos ? top_k : 1);
}

moe_status moe_ep_combine_padded(const moe_ep_t* ep, int region, const void* rows_padded, void* stream) {
  MOE_TRY(check_ep(ep, "moe_ep_combine_padded"));
  MOE_CHECK_ARG(rows_padded && (region == MOE_EP_RET_Y || region == MOE_EP_RET_DX),
                "moe_ep_combine_padded: NULL rows or region %d not a return region", region);
  const WinLayout L = win_layout(ep->nranks, ep->num_experts, ep->hidden, ep->cap_rows, ep->owner_rows);
  const size_t off = region == MOE_EP_RET_Y ? L.ret_y : L.ret_dx;
  return ep_copy_launch<true>(ep, rows_padded, region, off, stream);
}

moe_status moe_ep_combine_dest(const moe_ep_t* ep, int region, uint64_t* dest, int64_t max_rows, void* stream) {
  MOE_TRY(check_ep(ep, "moe_ep_combine_dest"));
  MOE_CHECK_ARG(dest && max_rows >= 0 && (region == MOE_EP_RET_Y || region == MOE_EP_RET_DX),
                "moe_ep_combine_dest: NULL dest, max_rows < 0 or region %d not a return region", region);
  if (max_rows == 0) return MOE_OK;
  const WinLayout L = win_layout(ep->nranks, ep->num_experts, ep->hidden, ep->cap_rows, ep->owner_rows);
  const size_t off = region == MOE_EP_RET_Y ? L.ret_y : L.ret_dx;
  const size_t tab = 3 * sizeof(int32_t) * (size_t)ep->num_experts;
  const int ctas = (int)std::min<int64_t>(ceil_div(max_rows, 256), 2 * 148);
  MOE_LAUNCH("ep_combine_dest", ep_combine_dest_kernel, dim3(ctas), dim3(256), tab, as_stream(stream), ep_args(ep),
             off, reinterpret_cast<unsigned long long*>(dest), (long long)max_rows);
  return MOE_OK;
}

moe_status moe_ep_signal(const moe_ep_t* ep, int region, void* stream) {
  MOE_TRY(check_ep(ep, "moe_ep_signal"));
  MOE_CHECK_ARG(region >= MOE_EP_COUNTS && region <= MOE_EP_RET_DX, "moe_ep_signal: bad region %d", region);
  MOE_LAUNCH("ep_signal", ep_signal_kernel, dim3(1), dim3(64), 0, as_stream(stream), ep_args(ep),
             region - MOE_EP_COUNTS);
  return MOE_OK;
}

int moe_ep_plan_offset(int nranks, int num_experts, int which) {
  // 0 compact counts [P, E/P], 1 padded rows of this rank; computed as plan_view does
  const int P = nranks, E = num_experts, El = E / P;
  const int ccomp = P * E + 1;
  switch (which) {
    case 0: return ccomp;
    case 1: return ccomp + P * El;
    default: return -1;
  }
}

moe_status moe_ep_wait(const moe_ep_t* ep, int region, void* stream) {
  MOE_TRY(check_ep(ep, "moe_ep_wait"));
  MOE_CHECK_ARG(region >= MOE_EP_RECV_X && region <= MOE_EP_RET_DX, "moe_ep_wait: bad region %d", region);
  MOE_LAUNCH("ep_wait", ep_wait_kernel, dim3(1), dim3(64), 0, as_stream(stream), ep_args(ep), region - MOE_EP_COUNTS);
  return MOE_OK;
}

}  // extern "C"
