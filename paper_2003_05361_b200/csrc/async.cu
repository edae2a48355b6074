// Asynchronous RAS (PAPER §2.1 P163-176, §3.3.2 P326-357, §3.4 P389-397).
//
// Every local subdomain runs its own sweep loop on its own CUDA stream with no
// inter-subdomain ordering: residual (reading owner / halo storage as it
// stands: "latest data"), Eq. 2 flag + convergence-detection step, PCG,
// restricted prolongation, and — for values other GPUs need — a fused pack +
// store straight into the peer GPU's halo storage over NVLink (CUDA IPC
// mapping), followed by a system-scope release of a per-subdomain version
// counter in the peer's board (the analogue of MPI_Put + flush, P394-396).
// Nothing waits on anything: no barriers, no collectives in the loop.
//
// Termination (P331-357, readings R19/R20): level flags on a spanning tree of
// the subdomain graph, stored as int32 words in every rank's "board" (peer
// boards mapped through CUDA IPC):
//   board[STOP + p]      stop word of subdomain p (written by tree neighbours)
//   board[REP + e]       report on directed tree edge e (v->parent: 2v,
//                        parent->v: 2v+1), written by the edge's sender
//   board[VER + p]       puts received from subdomain p (freshness statistic)
// centralized:   R_v = c_v AND (all children reports); the root stops when
//                c_root AND all children; STOP floods down the tree.
// decentralized: R_{v->u} = c_v AND (reports from all other tree neighbours);
//                v declares when c_v AND all; STOP floods over the tree.
// After every local subdomain stopped: barrier, halo refresh, true residual
// (P346-348); if it fails, flags are cleared and iteration resumes (R20).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "ctx.h"
#include "kernels.cuh"
#include "plan_internal.h"

namespace ras {

__device__ __forceinline__ void st_relaxed_gpu_i32(int32_t* p, int32_t v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct DetDev {
  int32_t P;
  int32_t central;        // 1 = centralized tree, 0 = decentralized
  const int32_t* gid;     // [nl] global id of local subdomain
  const int32_t* nb_off;  // [nl+1] into nb arrays
  const int32_t* nb;      // tree neighbours (global id)
  const int32_t* nb_rank; // their rank
  const int32_t* e_in;    // edge slot nb -> me
  const int32_t* e_out;   // edge slot me -> nb
  const int32_t* is_parent;  // nb is my parent (centralized)
  const int32_t* is_root;    // [nl]
  const double* b2;       // [nl] ||b~_p||^2 (Eq. 2) or owned-only variant
  int32_t* const* boards; // [world] board base per rank (own + IPC-mapped peers)
  int32_t my_rank;
  int32_t owned_only;
  const int32_t* force;   // test hook (ras_options.force_first_stop): nonzero -> every flag reads as set
  double* phase;          // [nl][kNPhase] device seconds per phase (ras_stats_t t_*), summed over updates
  unsigned long long* phase_last;  // [nl] globaltimer of the subdomain's last phase boundary
  // persistent kernel, one GPU (R33): per-subdomain sequence counters around every
  // x[S_p] write; a residual is recomputed until no data neighbour wrote during it,
  // so it sees every neighbour's update whole (default on; RAS_PERSISTENT_SEQLOCK=0
  // turns it off, which lets fixed-m PCG diverge on thin strips)
  int32_t* seq;
  const int32_t* dnb_off;  // [nl+1] data neighbours (owners of Gamma_p / Omega_p rows), local ids
  const int32_t* dnb;
  int32_t seqlock;
};

// Phase accounting of asynchronous updates (ras_stats_t t_residual ... t_convcheck,
// Figs. 3a-7a): thread 0 reads %globaltimer at each phase boundary of subdomain
// lp's update and charges the interval since the previous boundary to `ph`
// (ph < 0: the update starts, nothing is charged).
enum { PH_RES = 0, PH_SOLVE, PH_PROL, PH_EXCH, PH_CHECK, kNPhase };
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void phase_mark(const DetDev& D, int lp, int ph) {
  const unsigned long long t = gtimer();
  if (ph >= 0) D.phase[lp * kNPhase + ph] += 1e-9 * (double)(t - D.phase_last[lp]);
  D.phase_last[lp] = t;
}
static __global__ void k_phase(DetDev D, int lp, int ph, const int32_t* lstop) {
  if (threadIdx.x || blockIdx.x || lstop[lp]) return;
  phase_mark(D, lp, ph);
}

struct AsyncRt {
  std::vector<cudaStream_t> streams;
  int32_t* board = nullptr;  // own board (raw cudaMalloc)
  int32_t* board2 = nullptr; // scripted lock-step: second buffer
  size_t board_words = 0;
  std::vector<int32_t*> peer_board;
  std::vector<double*> peer_x;
  std::vector<void*> opened;
  int32_t** d_boards = nullptr;
  int32_t** d_boards2 = nullptr;
  double** d_peer_x = nullptr;
  DetDev det{};
  std::vector<int32_t> h_gid;
  int32_t* d_lstop = nullptr;
  int32_t* h_lstop = nullptr;      // mapped pinned mirror
  int32_t* h_active = nullptr;     // pinned (exact-mode polling)
  int32_t* h_lstop_dev = nullptr;
  int64_t* d_updates = nullptr;
  int32_t* d_noconv = nullptr;
  int64_t* d_stop_sweep = nullptr;
  // put lists (per local subdomain p: entries [put_off[p], put_off[p+1]))
  std::vector<int64_t> put_off;
  int32_t* d_put_slot = nullptr;
  int32_t* d_put_rank = nullptr;
  int64_t* d_put_ridx = nullptr;   // index into the destination rank's storage
  std::vector<int32_t> put_peer_off;  // per local sub: list of destination ranks
  int32_t* d_put_peers = nullptr;
  uint32_t* d_put_ticket = nullptr;
  uint8_t* d_scripted = nullptr;
  int64_t scripted_n = 0;
  int32_t* h_kill = nullptr;      // mapped pinned: host watchdog -> persistent kernel
  int32_t* h_kill_dev = nullptr;
  int32_t* d_force = nullptr;         // det.force (force_first_stop hook), set per detection round
  double* d_b2 = nullptr;             // det.b2 (Eq. 2 ||b~_p||^2), rewritten by ras_set_rhs
  int64_t* d_put_off = nullptr;       // device copies of put_off / put_peer_off (persistent kernel)
  int32_t* d_put_peer_off = nullptr;
  // stream driver: one CUDA graph per local subdomain holding a whole update
  // (residual, detection step, m PCG iterations, prolongation, puts), captured
  // once per (tol, max_iters, m, inner_tol) -- one launch per update instead of ~100
  std::vector<cudaGraphExec_t> graph;
  std::vector<int64_t> graph_launches;  // kernels in each graph (statistics)
  double g_tol = -1.0, g_itol = -1.0;
  int64_t g_maxit = -1;
  int g_m = -1;
};

// NVLink put lists for the persistent kernel (device view of AsyncRt's lists)
struct PutDev {
  const int64_t* off;       // [nl + 1]
  const int32_t* slot;      // owned slot of each entry
  const int32_t* rank;      // destination rank
  const int64_t* ridx;      // index in the destination's storage
  double* const* peer_x;    // [world] storage base per rank (IPC-mapped)
  const int32_t* peer_off;  // [nl + 1] into peers
  const int32_t* peers;     // destination ranks per local subdomain
};

// ---------------------------------------------------------------------------
// device helpers: system-scope release / acquire on 32-bit words
// ---------------------------------------------------------------------------
__device__ __forceinline__ void st_release_sys(int32_t* p, int32_t v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t ld_acquire_sys(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Iterate values shared between concurrently running CTAs / GPUs inside ONE
// launch (persistent kernel): morally strong (relaxed, system scope) accesses.
// Weak loads (ld.global.cg) of data another SM keeps rewriting are a data race
// in the PTX memory model -- they may be served from a stale copy for an
// unbounded time, i.e. an asynchronous iteration with UNBOUNDED delays (R33).
__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_f64(double* p, double v) {
  asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// One detection step of local subdomain lp (P331-357).  `in` is the board the
// reports / stop words are read from, `out` the boards they are written to
// (the same in true async mode; previous / next buffers in the scripted
// lock-step mode).  Returns 1 if lp stops in this step.
__device__ int det_step(const DetDev& D, int lp, int c, const int32_t* in, int32_t* const* out_boards) {
  const int p = D.gid[lp];
  const int a = D.nb_off[lp], b = D.nb_off[lp + 1];
  int stop = ld_acquire_sys(in + p) != 0;  // STOP + p (offset 0)
  const int32_t* rep = in + D.P;
  int all_in = 1;
  for (int i = a; i < b; ++i) {
    if (D.central && D.is_parent[i]) continue;
    all_in &= ld_acquire_sys(rep + D.e_in[i]) != 0;
  }
  if (D.central) {
    const int R = c && all_in;
    if (D.is_root[lp]) {
      if (R) stop = 1;
    } else {
      for (int i = a; i < b; ++i)
        if (D.is_parent[i]) st_release_sys(out_boards[D.nb_rank[i]] + D.P + D.e_out[i], R);
    }
    if (stop)
      for (int i = a; i < b; ++i)
        if (!D.is_parent[i]) st_release_sys(out_boards[D.nb_rank[i]] + D.nb[i], 1);
  } else {
    for (int i = a; i < b; ++i) {
      int R = c;
      for (int j = a; j < b; ++j)
        if (j != i) R &= ld_acquire_sys(rep + D.e_in[j]) != 0;
      st_release_sys(out_boards[D.nb_rank[i]] + D.P + D.e_out[i], R);
    }
    if (c && all_in) stop = 1;
    if (stop)
      for (int i = a; i < b; ++i) st_release_sys(out_boards[D.nb_rank[i]] + D.nb[i], 1);
  }
  return stop;
}

// Eq. 2 (P337-340): ||r~_p||^2 < tau^2 ||b~_p||^2 (||b~_p|| = 0: ||r~_p|| = 0, R11).
__device__ __forceinline__ int local_flag(const DetDev& D, const Scal& S, int lp, double tol) {
  if (*(const volatile int32_t*)D.force) return 1;
  const double r2 = D.owned_only ? S.own2[lp] : S.rt2[lp];
  const double b2 = D.b2[lp];
  return b2 == 0.0 ? (r2 == 0.0) : (r2 < tol * tol * b2);
}

// True async: one thread, after k_residual of subdomain lp on its stream.
static __global__ void k_detect(int lp, DetDev D, Scal S, double tol, int64_t max_iters, int32_t* lstop,
                                volatile int32_t* h_lstop, int64_t* updates, int32_t* noconv) {
  if (threadIdx.x || blockIdx.x) return;
  if (lstop[lp]) return;
  phase_mark(D, lp, PH_RES);  // the residual kernels ended when this one started
  const int64_t u = ++updates[lp];
  const int c = local_flag(D, S, lp, tol);
  const int32_t* in = D.boards[D.my_rank];
  // acquire: make the peers' released reports visible
  (void)ld_acquire_sys(in + D.gid[lp]);
  int stop = det_step(D, lp, c, in, D.boards);
  if (!stop && u > max_iters) {
    noconv[lp] = 1;
    stop = 1;
  }
  if (stop) {
    updates[lp] = u - 1;  // this sweep performs no update
    lstop[lp] = 1;
    h_lstop[lp] = 1;
  }
  phase_mark(D, lp, PH_CHECK);
}

// Scripted lock-step mode (test hook, SURVEY §8c "Detectors"): all local
// subdomains step together; reports of sweep k-1 are read from `prev`,
// sweep-k reports written to `next` (whose stop section was copied from prev).
static __global__ void k_detect_scripted(int nl, int64_t k, DetDev D, const uint8_t* flags, int64_t nsweeps,
                                         int32_t* const* prev, int32_t* const* next, int32_t* lstop,
                                         int64_t* stop_sweep, int64_t* updates) {
  const int lp = blockIdx.x * blockDim.x + threadIdx.x;
  if (lp >= nl || lstop[lp]) return;
  updates[lp] = k + 1;
  const int64_t row = k < nsweeps ? k : nsweeps - 1;
  const int c = flags[row * nl + lp] != 0;
  if (det_step(D, lp, c, prev[D.my_rank], next)) {
    lstop[lp] = 1;
    stop_sweep[lp] = k;
  }
}

// a5 (async): fused pack + NVLink store into the peer's halo storage, then
// (last CTA) fence.sc.sys and a system-scope release increment of version[p]
// in each destination rank's board (MPI_Put + flush analogue, P394-396).
static __global__ void k_put(int lp, int64_t e0, int64_t e1, const int32_t* __restrict__ slot,
                             const int32_t* __restrict__ rank, const int64_t* __restrict__ ridx,
                             const double* __restrict__ x, double* const* peer_x, uint32_t* ticket,
                             const int32_t* peers, int npeers, int32_t* const* boards, int P, int gp,
                             const int32_t* lstop, DetDev D) {
  if (lstop[lp]) return;
  for (int64_t e = e0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < e1; e += (int64_t)gridDim.x * blockDim.x)
    peer_x[rank[e]][ridx[e]] = x[slot[e]];
  __syncthreads();
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    __threadfence_system();
    s_last = atomicAdd(&ticket[lp], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence_system();
    for (int i = 0; i < npeers; ++i) atomicAdd_system(boards[peers[i]] + 3 * P + gp, 1);
    ticket[lp] = 0u;
    phase_mark(D, lp, PH_EXCH);
  }
}

static __global__ void k_mirror_stops(int nl, const int32_t* lstop, volatile int32_t* h) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nl) h[i] = lstop[i];
}

// ---------------------------------------------------------------------------
// Persistent asynchronous RAS (BLOCK regime: every |Omega_p| fits a CTA's
// shared memory; the paper's 4096-unknown subdomains, NEXT f2).  One
// cooperative launch per GPU: CTA g owns subdomains g, g + G, ... and loops
// over them with no barrier and no host involvement -- each update reads the
// owner / halo values as they stand in L2 ("latest data", P163-176;
// ld.global.cg, 8-byte stores are atomic; peers' NVLink stores land in this
// GPU's memory), computes r~_p and its Eq. 2 flag, takes one detection step
// (the same det_step protocol as the stream-based mode, boards shared across
// GPUs), runs the whole local PCG in shared memory (block_pcg), stores
// x[S_p] += d and puts the values other GPUs need into their halo storage.  A
// CTA exits when all its subdomains stopped (the detection protocol stops all
// of them) or the host watchdog raises the kill word.
// ---------------------------------------------------------------------------
template <int RPT, int WR, int WL, bool Z>
static __global__ void __launch_bounds__(kNT_SMALL, 1)
    k_async_persistent(int nl, SmallSubs SS, Sell Rm, Sell L, Diag D, const double* __restrict__ b,
                       const int32_t* __restrict__ own_slot, double* x, DetDev det, PutDev PD, Scal S, double tol,
                       int64_t max_iters, int32_t m, double inner_tol, int32_t* lstop, volatile int32_t* h_lstop,
                       int64_t* updates, int32_t* noconv, const volatile int32_t* kill, double* dglob) {
  extern __shared__ double smem[];
  __shared__ double red[3][kNT_SMALL / 32];
  __shared__ int s_stop;
  const double* tabR = Rm.table;
  for (;;) {
    bool any = false;
    for (int lp = blockIdx.x; lp < nl; lp += gridDim.x) {
      // lstop[lp] is written by this CTA's thread 0; read it once and broadcast so
      // the whole CTA takes the same branch (another thread's L1 may hold the old word)
      __syncthreads();
      if (threadIdx.x == 0) s_stop = ((volatile int32_t*)lstop)[lp];
      __syncthreads();
      if (s_stop) continue;
      any = true;
      if (threadIdx.x == 0) phase_mark(det, lp, -1);
      const int r0 = SS.row_off[lp], n = SS.nrows[lp];
      double* sp = smem;
      double* sr = smem + n;
      double* sd = dglob ? dglob + r0 : smem + 2 * n;  // d: row-private, shared memory or L2
      // a1 + a2: r~ = b~ - [A_p | B_p] x (owner storage read through L2), z = D^-1 r
      double v[3] = {0.0, 0.0, 0.0};
      __shared__ int32_t s_sv[64];
      __shared__ int s_retry;
    seq_retry:  // (whole-update neighbour snapshots, R33)
      if (det.seqlock) {
        const int nb0 = det.dnb_off[lp], nnb = min(64, det.dnb_off[lp + 1] - nb0);
        __syncthreads();
        if (threadIdx.x == 0) s_retry = 0;
        __syncthreads();
        if ((int)threadIdx.x < nnb) {
          const int32_t sv = ld_acquire_gpu(&det.seq[det.dnb[nb0 + threadIdx.x]]);
          s_sv[threadIdx.x] = sv;
          if (sv & 1) s_retry = 1;  // a neighbour is mid-write
        }
        __syncthreads();
        if (s_retry) goto seq_retry;
        v[0] = v[1] = v[2] = 0.0;
      }
      for (int i = threadIdx.x; i < n; i += kNT_SMALL) {
        const int64_t row = (int64_t)r0 + i;
        const double ax = resident_row<WR, Z>(Rm, row, tabR, [&](int32_t c) { return ld_relaxed_f64(&x[c]); });
        const double ri = __ldg(&b[row]) - ax;
        const double zi = __drcp_rn(diag_at<Z>(D, row)) * ri;
        sr[i] = ri;
        sp[i] = zi;
        sd[i] = 0.0;
        v[0] += ri * zi;
        v[1] += ri * ri;
        v[2] += __ldg(&own_slot[row]) >= 0 ? ri * ri : 0.0;
      }
      if (det.seqlock) {
        const int nb0 = det.dnb_off[lp], nnb = min(64, det.dnb_off[lp + 1] - nb0);
        __threadfence();  // the x reads above before the counters' second read
        __syncthreads();
        if ((int)threadIdx.x < nnb && ld_acquire_gpu(&det.seq[det.dnb[nb0 + threadIdx.x]]) != s_sv[threadIdx.x])
          s_retry = 1;
        __syncthreads();
        if (s_retry) goto seq_retry;
      }
      block_allsum<3>(v, red);
      // a6: Eq. 2 flag + one detection step (P331-357)
      if (threadIdx.x == 0) {
        phase_mark(det, lp, PH_RES);
        S.rt2[lp] = v[1];
        S.own2[lp] = v[2];
        const int64_t u = ++updates[lp];
        const int c = local_flag(det, S, lp, tol);
        const int32_t* in = det.boards[det.my_rank];
        (void)ld_acquire_sys(in + det.gid[lp]);
        int stop = det_step(det, lp, c, in, det.boards);
        if (!stop && u > max_iters) {
          noconv[lp] = 1;
          stop = 1;
        }
        if (!stop && *kill) stop = 1;
        if (stop) {
          updates[lp] = u - 1;  // this sweep performs no update
          lstop[lp] = 1;
          h_lstop[lp] = 1;
        }
        s_stop = stop;
        phase_mark(det, lp, PH_CHECK);
      }
      __syncthreads();
      if (s_stop) continue;
      // a3: the whole local PCG in shared memory; a4: x[S_p] += d
      const int its = v[0] != 0.0 ? block_pcg<RPT, WL, Z>(L, D, r0, n, sp, sr, sd, v[0], v[1], m, inner_tol, red) : 0;
      if (threadIdx.x == 0) phase_mark(det, lp, PH_SOLVE);
      if (its > 0 && det.seqlock && threadIdx.x == 0) {  // odd: x[S_p] being written
        st_relaxed_gpu_i32(&det.seq[lp], det.seq[lp] + 1);
        __threadfence();
      }
      if (det.seqlock) __syncthreads();
      if (its > 0)
        for (int i = threadIdx.x; i < n; i += kNT_SMALL) {
          const int32_t sl = __ldg(&own_slot[r0 + i]);
          if (sl >= 0) st_relaxed_f64(&x[sl], ld_relaxed_f64(&x[sl]) + sd[i]);
        }
      if (its > 0 && det.seqlock) {  // even again: published
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
          __threadfence();
          st_relaxed_gpu_i32(&det.seq[lp], det.seq[lp] + 1);
        }
      }
      if (threadIdx.x == 0) phase_mark(det, lp, PH_PROL);
      // a5 (multi-GPU): owner values other GPUs need, stored straight into their
      // halo storage over NVLink; then a system-scope fence and a version bump in
      // each destination's board (MPI_Put + flush analogue, P394-396)
      const int64_t e0 = PD.off[lp], e1 = PD.off[lp + 1];
      if (its > 0 && e1 > e0) {
        __syncthreads();  // this CTA's x[S_p] stores before the reads below
        for (int64_t e = e0 + threadIdx.x; e < e1; e += kNT_SMALL)
          st_relaxed_f64(&PD.peer_x[PD.rank[e]][PD.ridx[e]], ld_relaxed_f64(&x[PD.slot[e]]));
        __syncthreads();
        if (threadIdx.x == 0) {
          __threadfence_system();
          for (int k = PD.peer_off[lp]; k < PD.peer_off[lp + 1]; ++k)
            atomicAdd_system(det.boards[PD.peers[k]] + 3 * det.P + det.gid[lp], 1);
        }
      }
      if (threadIdx.x == 0) phase_mark(det, lp, PH_EXCH);
      if (threadIdx.x == 0) S.inner_total[lp] += its;
      __syncthreads();
    }
    if (!any) break;
  }
}

static const void* async_persistent_kernel(int rpt, bool z, int wr, int wl) {
#define RAS_AP(RPT)                                                                                        \
  if (!z) return (const void*)k_async_persistent<RPT, 0, 0, false>;                                        \
  if (wr == 4) return wl == 4 ? (const void*)k_async_persistent<RPT, 4, 4, true>                           \
                              : (const void*)k_async_persistent<RPT, 4, 8, true>;                          \
  return wl == 4 ? (const void*)k_async_persistent<RPT, 8, 4, true> : (const void*)k_async_persistent<RPT, 8, 8, true>;
  if (rpt <= 4) {
    RAS_AP(4)
  } else if (rpt <= 9) {
    RAS_AP(9)
  } else {
    RAS_AP(14)
  }
#undef RAS_AP
}

// Lazy module loading (the CUDA 12 default) loads a kernel at its first launch,
// and that load can wait for kernels already running.  With loopback virtual
// ranks on one device, rank A's kernel may be spinning on a flag rank B's kernel
// sets while B launches something for the first time: a deadlock.  So every
// kernel an asynchronous solve launches is loaded at setup.
static ras_status preload_async_kernels(ras_ctx* c) {
  const void* fns[] = {(const void*)k_phase, (const void*)k_detect, (const void*)k_detect_scripted,
                       (const void*)k_put, (const void*)k_mirror_stops};
  cudaFuncAttributes fa;
  for (const void* f : fns) RAS_CUDA(c, cudaFuncGetAttributes(&fa, f));
  for (int rpt : {4, 9, 14})
    for (int z = 0; z < 2; ++z)
      for (int wr : {4, 8})
        for (int wl : {4, 8}) RAS_CUDA(c, cudaFuncGetAttributes(&fa, async_persistent_kernel(rpt, z, wr, wl)));
  return RAS_OK;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static ras_status barrier(ras_ctx* c) { return coll_barrier(c); }

// subdomain adjacency (p ~ q iff p needs a value owned by q or vice versa),
// assembled over all ranks with one NCCL sum
static ras_status subdomain_graph(ras_ctx* c, std::vector<std::vector<int32_t>>& adj) {
  const ras_plan* pl = c->plan;
  const int P = pl->P;
  std::vector<int32_t> M((size_t)P * P, 0);
  for (const auto& S : pl->subs)
    for (int32_t q : S.nbr_subs) M[(size_t)S.p * P + q] = 1;
  if (c->world > 1) {
    int32_t* d;
    TRY(upload(c, &d, M));
    TRY(coll_allreduce(c, d, d, M.size(), ncclInt32, ncclSum, c->stream));
    RAS_CUDA(c, cudaMemcpyAsync(M.data(), d, M.size() * 4, cudaMemcpyDeviceToHost, c->stream));
    RAS_CUDA(c, cudaStreamSynchronize(c->stream));
  }
  adj.assign(P, {});
  for (int p = 0; p < P; ++p)
    for (int q = 0; q < P; ++q)
      if (p != q && (M[(size_t)p * P + q] || M[(size_t)q * P + p])) adj[p].push_back(q);
  return RAS_OK;
}

static std::vector<int32_t> bfs_tree(const std::vector<std::vector<int32_t>>& adj) {
  const int P = (int)adj.size();
  std::vector<int32_t> parent(P, -2);
  parent[0] = -1;
  std::vector<int32_t> q{0};
  for (size_t h = 0; h < q.size(); ++h)
    for (int w : adj[q[h]])
      if (parent[w] == -2) {
        parent[w] = q[h];
        q.push_back(w);
      }
  // disconnected subdomain graph: hang remaining components under the root
  for (int v = 0; v < P; ++v)
    if (parent[v] == -2) parent[v] = 0;
  return parent;
}

static std::vector<int32_t> central_tree(const std::vector<int32_t>& sub_to_rank) {
  const int P = (int)sub_to_rank.size();
  std::vector<int32_t> leader(*std::max_element(sub_to_rank.begin(), sub_to_rank.end()) + 1, -1), parent(P);
  for (int p = 0; p < P; ++p)
    if (leader[sub_to_rank[p]] < 0) leader[sub_to_rank[p]] = p;
  for (int p = 0; p < P; ++p) {
    const int L = leader[sub_to_rank[p]];
    parent[p] = p == 0 ? -1 : (p == L ? 0 : L);
  }
  return parent;
}

static ras_status setup_ipc(ras_ctx* c, AsyncRt* A) {
  const int W = c->world;
  A->peer_board.assign(W, nullptr);
  A->peer_x.assign(W, nullptr);
  A->peer_board[c->rank] = A->board;
  A->peer_x[c->rank] = c->d_x;
  if (W == 1) return RAS_OK;
  if (c->loopback) {  // virtual ranks on one device: the peers' windows are plain pointers
    std::vector<int64_t> mine{(int64_t)(uintptr_t)c->d_x, (int64_t)(uintptr_t)A->board};
    int64_t *d_mine, *d_all;
    TRY(upload(c, &d_mine, mine));
    TRY(zalloc(c, &d_all, (size_t)2 * W));
    TRY(coll_allgather(c, d_mine, d_all, 2, ncclInt64, c->stream));
    std::vector<int64_t> all((size_t)2 * W);
    RAS_CUDA(c, cudaMemcpyAsync(all.data(), d_all, all.size() * 8, cudaMemcpyDeviceToHost, c->stream));
    RAS_CUDA(c, cudaStreamSynchronize(c->stream));
    for (int r = 0; r < W; ++r) {
      A->peer_x[r] = (double*)(uintptr_t)all[2 * r];
      A->peer_board[r] = (int32_t*)(uintptr_t)all[2 * r + 1];
    }
    return RAS_OK;
  }
  cudaIpcMemHandle_t h[2];
  RAS_CUDA(c, cudaIpcGetMemHandle(&h[0], c->d_x));
  RAS_CUDA(c, cudaIpcGetMemHandle(&h[1], A->board));
  std::vector<char> mine(sizeof(h));
  std::memcpy(mine.data(), h, sizeof(h));
  char *d_mine, *d_all;
  TRY(upload(c, &d_mine, mine));
  TRY(zalloc(c, &d_all, sizeof(h) * W));
  TRY(coll_allgather(c, d_mine, d_all, sizeof(h), ncclInt8, c->stream));
  std::vector<char> all(sizeof(h) * W);
  RAS_CUDA(c, cudaMemcpyAsync(all.data(), d_all, all.size(), cudaMemcpyDeviceToHost, c->stream));
  RAS_CUDA(c, cudaStreamSynchronize(c->stream));
  for (int r = 0; r < W; ++r) {
    if (r == c->rank) continue;
    cudaIpcMemHandle_t hr[2];
    std::memcpy(hr, all.data() + r * sizeof(h), sizeof(h));
    void *px = nullptr, *pb = nullptr;
    RAS_CUDA(c, cudaIpcOpenMemHandle(&px, hr[0], cudaIpcMemLazyEnablePeerAccess));
    A->opened.push_back(px);
    RAS_CUDA(c, cudaIpcOpenMemHandle(&pb, hr[1], cudaIpcMemLazyEnablePeerAccess));
    A->opened.push_back(pb);
    A->peer_x[r] = (double*)px;
    A->peer_board[r] = (int32_t*)pb;
  }
  return RAS_OK;
}

ras_status async_setup(ras_ctx* c) {
  AsyncRt* A = new AsyncRt();
  c->async = A;
  ras_plan* pl = c->plan;
  const int P = pl->P, nl = c->nl, W = c->world;
  // boards: [STOP: P][REP: 2P][VER: P]
  A->board_words = (size_t)4 * P + 64;
  A->board = (int32_t*)dalloc_raw(c, A->board_words * 4);
  A->board2 = (int32_t*)dalloc_raw(c, A->board_words * 4);
  if (!A->board || !A->board2) return set_err(c, RAS_ENOMEM, "board allocation failed");
  TRY(setup_ipc(c, A));
  TRY(upload(c, &A->d_boards, A->peer_board));
  std::vector<int32_t*> b2v(W, nullptr);
  b2v[c->rank] = A->board2;  // scripted mode is single-rank
  TRY(upload(c, &A->d_boards2, b2v));
  TRY(upload(c, &A->d_peer_x, A->peer_x));
  // trees
  std::vector<std::vector<int32_t>> adj;
  TRY(subdomain_graph(c, adj));
  const std::vector<int32_t> par = c->opt.detector == RAS_DET_CENTRAL ? central_tree(pl->sub_to_rank) : bfs_tree(adj);
  std::vector<int32_t> gid(nl), nb_off(nl + 1, 0), nb, nb_rank, e_in, e_out, is_par, is_root(nl);
  std::vector<double> b2(nl);
  for (int lp = 0; lp < nl; ++lp) {
    const int p = pl->subs[lp].p;
    gid[lp] = p;
    is_root[lp] = par[p] == -1;
    b2[lp] = c->opt.local_crit_owned_only ? pl->subs[lp].b2_owned : pl->subs[lp].b2;
    auto add = [&](int u, bool up) {
      nb.push_back(u);
      nb_rank.push_back(pl->sub_to_rank[u]);
      // edge v->parent(v): 2v ; parent(v)->v: 2v+1
      e_in.push_back(up ? 2 * p + 1 : 2 * u);
      e_out.push_back(up ? 2 * p : 2 * u + 1);
      is_par.push_back(up ? 1 : 0);
    };
    if (par[p] >= 0) add(par[p], true);
    for (int u = 0; u < P; ++u)
      if (par[u] == p) add(u, false);
    nb_off[lp + 1] = (int32_t)nb.size();
  }
  A->h_gid = gid;
  DetDev& D = A->det;
  D.P = P;
  D.central = c->opt.detector == RAS_DET_CENTRAL;
  D.my_rank = c->rank;
  D.owned_only = c->opt.local_crit_owned_only;
  int32_t *dg, *dno, *dnb, *dnr, *dei, *deo, *dip, *dir;
  double* db2;
  TRY(upload(c, &dg, gid));
  TRY(upload(c, &dno, nb_off));
  TRY(upload(c, &dnb, nb, 1));
  TRY(upload(c, &dnr, nb_rank, 1));
  TRY(upload(c, &dei, e_in, 1));
  TRY(upload(c, &deo, e_out, 1));
  TRY(upload(c, &dip, is_par, 1));
  TRY(upload(c, &dir, is_root));
  TRY(upload(c, &db2, b2));
  D.gid = dg;
  D.nb_off = dno;
  D.nb = dnb;
  D.nb_rank = dnr;
  D.e_in = dei;
  D.e_out = deo;
  D.is_parent = dip;
  D.is_root = dir;
  D.b2 = db2;
  A->d_b2 = db2;
  TRY(zalloc(c, &A->d_force, 1));
  D.force = A->d_force;
  {
    const char* q = getenv("RAS_PERSISTENT_SEQLOCK");
    D.seqlock = !(q && q[0] == '0') && W == 1;
    std::vector<int32_t> off(1, 0), nb;
    for (int lp = 0; lp < nl; ++lp) {
      for (int32_t g : pl->subs[lp].nbr_subs) nb.push_back(g);  // one GPU: local id = global id
      off.push_back((int32_t)nb.size());
    }
    int32_t *doff, *dnb;
    TRY(upload(c, &doff, off, 1));
    TRY(upload(c, &dnb, nb, 1));
    D.dnb_off = doff;
    D.dnb = dnb;
    TRY(zalloc(c, &D.seq, (size_t)std::max(nl, 1)));
  }
  TRY(zalloc(c, &D.phase, (size_t)std::max(nl, 1) * kNPhase));
  TRY(zalloc(c, &D.phase_last, (size_t)std::max(nl, 1)));
  D.boards = A->d_boards;
  TRY(zalloc(c, &A->d_lstop, nl));
  TRY(zalloc(c, &A->d_updates, nl));
  TRY(zalloc(c, &A->d_noconv, nl));
  TRY(zalloc(c, &A->d_stop_sweep, nl));
  TRY(zalloc(c, &A->d_put_ticket, nl));
  RAS_CUDA(c, cudaHostAlloc((void**)&A->h_lstop, std::max(nl, 1) * 4, cudaHostAllocMapped));
  RAS_CUDA(c, cudaHostGetDevicePointer((void**)&A->h_lstop_dev, A->h_lstop, 0));
  RAS_CUDA(c, cudaHostAlloc((void**)&A->h_active, std::max(nl, 1) * 4, cudaHostAllocDefault));
  RAS_CUDA(c, cudaHostAlloc((void**)&A->h_kill, 4, cudaHostAllocMapped));
  RAS_CUDA(c, cudaHostGetDevicePointer((void**)&A->h_kill_dev, A->h_kill, 0));
  *A->h_kill = 0;
  // put lists: entries of the send lists whose source slot belongs to local p
  std::vector<int64_t> n_own_all(W, 0);
  n_own_all[c->rank] = c->n_own;
  if (W > 1) {
    int64_t* d;
    TRY(upload(c, &d, n_own_all));
    TRY(coll_allreduce(c, d, d, W, ncclInt64, ncclSum, c->stream));
    RAS_CUDA(c, cudaMemcpyAsync(n_own_all.data(), d, W * 8, cudaMemcpyDeviceToHost, c->stream));
    RAS_CUDA(c, cudaStreamSynchronize(c->stream));
  }
  std::vector<int32_t> ps, pr, peers;
  std::vector<int64_t> pi;
  A->put_off.assign(nl + 1, 0);
  A->put_peer_off.assign(nl + 1, 0);
  for (int lp = 0; lp < nl; ++lp) {
    const auto& S = pl->subs[lp];
    for (int q = 0; q < W; ++q) {
      bool any = false;
      for (size_t i = 0; i < pl->send_slot[q].size(); ++i) {
        const int32_t s = pl->send_slot[q][i];
        if (s >= S.own_off && s < S.own_off + S.nown) {
          ps.push_back(s);
          pr.push_back(q);
          pi.push_back(n_own_all[q] + pl->send_remote_off[q] + (int64_t)i);
          any = true;
        }
      }
      if (any) peers.push_back(q);
    }
    A->put_off[lp + 1] = (int64_t)ps.size();
    A->put_peer_off[lp + 1] = (int32_t)peers.size();
  }
  TRY(upload(c, &A->d_put_slot, ps, 1));
  TRY(upload(c, &A->d_put_rank, pr, 1));
  TRY(upload(c, &A->d_put_ridx, pi, 1));
  TRY(upload(c, &A->d_put_peers, peers, 1));
  TRY(upload(c, &A->d_put_off, A->put_off, 1));
  TRY(upload(c, &A->d_put_peer_off, A->put_peer_off, 1));
  A->streams.resize(nl);
  for (auto& s : A->streams) RAS_CUDA(c, cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  TRY(preload_async_kernels(c));
  return RAS_OK;
}

ras_status async_set_b2(ras_ctx* c) {
  AsyncRt* A = c->async;
  if (!A || !A->d_b2) return RAS_OK;
  std::vector<double> b2(c->nl);
  for (int lp = 0; lp < c->nl; ++lp)
    b2[lp] = c->opt.local_crit_owned_only ? c->plan->subs[lp].b2_owned : c->plan->subs[lp].b2;
  RAS_CUDA(c, cudaMemcpyAsync(A->d_b2, b2.data(), b2.size() * 8, cudaMemcpyHostToDevice, c->stream));
  RAS_CUDA(c, cudaStreamSynchronize(c->stream));
  return RAS_OK;
}

void async_free(ras_ctx* c) {
  AsyncRt* A = c->async;
  if (!A) return;
  for (auto s : A->streams) cudaStreamDestroy(s);
  for (void* p : A->opened) cudaIpcCloseMemHandle(p);
  if (A->h_lstop) cudaFreeHost(A->h_lstop);
  if (A->h_active) cudaFreeHost(A->h_active);
  if (A->h_kill) cudaFreeHost(A->h_kill);
  for (auto g : A->graph)
    if (g) cudaGraphExecDestroy(g);
  delete A;
  c->async = nullptr;
}

static ras_status reset_detection(ras_ctx* c) {
  AsyncRt* A = c->async;
  RAS_CUDA(c, cudaMemsetAsync(A->board, 0, A->board_words * 4, c->stream));
  RAS_CUDA(c, cudaMemsetAsync(A->board2, 0, A->board_words * 4, c->stream));
  RAS_CUDA(c, cudaMemsetAsync(A->d_lstop, 0, c->nl * 4, c->stream));
  RAS_CUDA(c, cudaMemsetAsync(A->d_noconv, 0, c->nl * 4, c->stream));
  RAS_CUDA(c, cudaMemsetAsync(A->d_put_ticket, 0, c->nl * 4, c->stream));
  for (int i = 0; i < c->nl; ++i) A->h_lstop[i] = 0;
  RAS_CUDA(c, cudaStreamSynchronize(c->stream));
  return barrier(c);  // every rank cleared its board before anyone writes again
}

// one sweep of local subdomain lp on stream s (true async)
static ras_status enqueue_sub_sweep(ras_ctx* c, int lp, cudaStream_t s, double tol, int64_t max_iters, int m,
                                    double inner_tol, bool exact) {
  AsyncRt* A = c->async;
  const ras_plan* pl = c->plan;
  const auto& SP = pl->subs[lp];
  const Range R = range_sub(c, lp);
  Ctl C{A->d_lstop, 1};
  k_phase<<<1, 32, 0, s>>>(A->det, lp, -1, A->d_lstop);
  TRY(enq_residual(c, s, R, C));
  k_detect<<<1, 32, 0, s>>>(lp, A->det, c->S, tol, max_iters, A->d_lstop, A->h_lstop_dev, A->d_updates,
                            A->d_noconv);
  c->launches += 2;
  TRY(enq_pcg(c, s, R, C, m, inner_tol, exact));
  const bool fused_prolong = c->small || c->chol || c->path == RAS_PCG_RESIDENT;
  if (!fused_prolong) {
    k_phase<<<1, 32, 0, s>>>(A->det, lp, PH_SOLVE, A->d_lstop);
    c->launches += 1;
  }
  TRY(enq_prolong(c, s, R, C));
  k_phase<<<1, 32, 0, s>>>(A->det, lp, fused_prolong ? PH_SOLVE : PH_PROL, A->d_lstop);
  c->launches += 1;
  const int64_t e0 = A->put_off[lp], e1 = A->put_off[lp + 1];
  if (e1 > e0) {
    const unsigned pg = (unsigned)std::min<int64_t>((e1 - e0 + 255) / 256, 148 * 4);
    k_put<<<pg, 256, 0, s>>>(lp, e0, e1, A->d_put_slot, A->d_put_rank, A->d_put_ridx, c->d_x, A->d_peer_x,
                             A->d_put_ticket, A->d_put_peers + A->put_peer_off[lp],
                             A->put_peer_off[lp + 1] - A->put_peer_off[lp], A->d_boards, pl->P, SP.p, A->d_lstop,
                             A->det);
    c->launches += 1;
  }
  return RAS_OK;
}

// Two consecutive subdomains updated by one launch of each kernel (RESIDENT path,
// default; RAS_ASYNC_PAIRS=0 turns it off): both read the latest data and write
// their own rows -- the asynchronous schedule [[lp, lp+1], ...] (oracle
// ras_schedule, R34); the RESIDENT kernel runs them as its two lanes.
static ras_status enqueue_pair_sweep(ras_ctx* c, int lp, cudaStream_t s, double tol, int64_t max_iters, int m,
                                     double inner_tol, bool exact) {
  AsyncRt* A = c->async;
  const ras_plan* pl = c->plan;
  Range R = range_sub(c, lp);
  R.ntiles += (unsigned)pl->subs[lp + 1].ntiles;  // tiles of consecutive subdomains are consecutive
  R.nsub = 2;
  Ctl C{A->d_lstop, 1};
  for (int q = lp; q < lp + 2; ++q) k_phase<<<1, 32, 0, s>>>(A->det, q, -1, A->d_lstop);
  TRY(enq_residual(c, s, R, C));
  for (int q = lp; q < lp + 2; ++q)
    k_detect<<<1, 32, 0, s>>>(q, A->det, c->S, tol, max_iters, A->d_lstop, A->h_lstop_dev, A->d_updates, A->d_noconv);
  c->launches += 4;
  TRY(enq_pcg(c, s, R, C, m, inner_tol, exact));  // RESIDENT: prolongation fused
  for (int q = lp; q < lp + 2; ++q) {
    k_phase<<<1, 32, 0, s>>>(A->det, q, PH_SOLVE, A->d_lstop);
    c->launches += 1;
    const int64_t e0 = A->put_off[q], e1 = A->put_off[q + 1];
    if (e1 > e0) {
      const unsigned pg = (unsigned)std::min<int64_t>((e1 - e0 + 255) / 256, 148 * 4);
      k_put<<<pg, 256, 0, s>>>(q, e0, e1, A->d_put_slot, A->d_put_rank, A->d_put_ridx, c->d_x, A->d_peer_x,
                               A->d_put_ticket, A->d_put_peers + A->put_peer_off[q],
                               A->put_peer_off[q + 1] - A->put_peer_off[q], A->d_boards, pl->P, pl->subs[q].p,
                               A->d_lstop, A->det);
      c->launches += 1;
    }
  }
  return RAS_OK;
}

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// true async loop on this rank: per-subdomain streams, host keeps <= Q sweeps
// in flight per stream, exits when every local subdomain stopped
static ras_status run_async_loop(ras_ctx* c, double tol, int64_t max_iters, int m, double inner_tol, bool exact,
                                 bool* timeout) {
  AsyncRt* A = c->async;
  const int nl = c->nl;
  const int Q = 2;
  std::vector<std::vector<cudaEvent_t>> ev(nl, std::vector<cudaEvent_t>(Q));
  for (auto& v : ev)
    for (auto& e : v) RAS_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  std::vector<int64_t> enq(nl, 0);
  // capture each subdomain's update as a CUDA graph (fixed-m solves: the kernel
  // sequence is static; the exact mode polls the host and is enqueued directly)
  const bool use_graph = !exact && c->opt.use_graphs != 0;
  if (use_graph && (A->graph.size() != (size_t)nl || A->g_tol != tol || A->g_maxit != max_iters || A->g_m != m ||
                    A->g_itol != inner_tol)) {
    for (auto g : A->graph)
      if (g) cudaGraphExecDestroy(g);
    A->graph.assign(nl, nullptr);
    A->graph_launches.assign(nl, 0);
    for (int lp = 0; lp < nl; ++lp) {
      cudaStream_t s = A->streams[lp];
      const int64_t l0 = c->launches;
      RAS_CUDA(c, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      const ras_status cs = enqueue_sub_sweep(c, lp, s, tol, max_iters, m, inner_tol, exact);
      cudaGraph_t g = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(s, &g);
      if (cs != RAS_OK) return cs;
      RAS_CUDA(c, ce);
      RAS_CUDA(c, cudaGraphInstantiate(&A->graph[lp], g, 0));
      cudaGraphDestroy(g);
      A->graph_launches[lp] = c->launches - l0;
      c->launches = l0;
    }
    A->g_tol = tol;
    A->g_maxit = max_iters;
    A->g_m = m;
    A->g_itol = inner_tol;
  }
  const double t0 = now_s();
  *timeout = false;
  ras_status st = RAS_OK;
  for (;;) {
    int nstopped = 0;
    bool progressed = false;
    for (int lp = 0; lp < nl; ++lp) {
      if (((volatile int32_t*)A->h_lstop)[lp]) {
        ++nstopped;
        continue;
      }
      if (enq[lp] >= Q && cudaEventQuery(ev[lp][enq[lp] % Q]) == cudaErrorNotReady) continue;
      if (use_graph) {
        const cudaError_t e = cudaGraphLaunch(A->graph[lp], A->streams[lp]);
        if (e != cudaSuccess) {
          st = cuda_err(c, e, "cudaGraphLaunch (async update)");
          break;
        }
        c->launches += A->graph_launches[lp];
      } else {
        st = enqueue_sub_sweep(c, lp, A->streams[lp], tol, max_iters, m, inner_tol, exact);
      }
      if (st != RAS_OK) break;
      RAS_CUDA(c, cudaEventRecord(ev[lp][enq[lp] % Q], A->streams[lp]));
      ++enq[lp];
      progressed = true;
    }
    if (st != RAS_OK || nstopped == nl) break;
    if (now_s() - t0 > c->opt.async_timeout_s) {
      *timeout = true;
      break;
    }
    if (!progressed) std::this_thread::sleep_for(std::chrono::microseconds(20));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      st = cuda_err(c, e, "async sweep");
      break;
    }
  }
  if (*timeout) {  // watchdog: stop every local subdomain from the host
    std::vector<int32_t> ones(nl, 1);
    cudaMemcpy(A->d_lstop, ones.data(), nl * 4, cudaMemcpyHostToDevice);
  }
  cudaDeviceSynchronize();
  for (auto& v : ev)
    for (auto& e : v) cudaEventDestroy(e);
  return st;
}

// persistent async mode (BLOCK regime, any number of GPUs): one cooperative
// launch per GPU, the host only watches the wall clock
static ras_status run_async_persistent(ras_ctx* c, double tol, int64_t max_iters, int m, double inner_tol,
                                       bool* timeout) {
  AsyncRt* A = c->async;
  const int nl = c->nl;
  const void* fn = async_persistent_kernel((c->small_nmax + kNT_SMALL - 1) / kNT_SMALL, c->z, c->zwR, c->zwL);
  const bool dl2 = c->small_nmax > kSmallSmemDRows;  // d in L2 (row space d_d) for the larger subdomains
  const size_t smem = (size_t)(dl2 ? 2 : 3) * c->small_nmax * sizeof(double);
  double* dglob = dl2 ? c->d_d : nullptr;
  TRY(allow_smem(c, fn));
  int per_sm = 0, sms = 0;
  RAS_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kNT_SMALL, smem));
  RAS_CUDA(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  if (per_sm < 1) return set_err(c, RAS_ESTATE, "persistent async kernel does not fit an SM");
  // loopback virtual ranks share one device: each persistent grid gets 1/world of
  // it so that every rank's CTAs are resident at once (they wait on each other's flags)
  int G = std::min(nl, std::max(1, per_sm * sms / (c->loopback ? c->world : 1)));
  if (c->opt.persistent_grid > 0) G = std::min(G, c->opt.persistent_grid);
  *A->h_kill = 0;
  int nl_ = nl;
  Sell Rm = c->R, L = c->L;
  Diag D = c->D;
  const double* b = c->d_b;
  const int32_t* own = c->d_own_slot;
  double* x = c->d_x;
  DetDev det = A->det;
  PutDev PD{A->d_put_off, A->d_put_slot, A->d_put_rank, A->d_put_ridx, A->d_peer_x, A->d_put_peer_off, A->d_put_peers};
  Scal S = c->S;
  int64_t mi = max_iters;
  int32_t mm = m;
  int32_t* lstop = A->d_lstop;
  volatile int32_t* hl = A->h_lstop_dev;
  int64_t* up = A->d_updates;
  int32_t* nc = A->d_noconv;
  const volatile int32_t* kill = A->h_kill_dev;
  SmallSubs SS = c->SS;
  void* args[] = {&nl_, &SS, &Rm, &L, &D, &b, &own, &x, &det, &PD, &S, &tol, &mi, &mm, &inner_tol, &lstop, &hl, &up, &nc, &kill,
                  &dglob};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)G);
  cfg.blockDim = dim3(kNT_SMALL);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  RAS_CUDA(c, cudaLaunchKernelExC(&cfg, fn, args));
  c->launches += 1;
  const double t0 = now_s();
  *timeout = false;
  for (;;) {
    const cudaError_t e = cudaStreamQuery(c->stream);
    if (e == cudaSuccess) break;
    if (e != cudaErrorNotReady) return cuda_err(c, e, "persistent async kernel");
    if (!*timeout && now_s() - t0 > c->opt.async_timeout_s) {
      *timeout = true;
      *(volatile int32_t*)A->h_kill = 1;  // every CTA stops at its next update
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  return RAS_OK;
}

// Asynchronous RAS with RESIDENT-sized subdomains (each local solve needs the
// whole GPU; any number of GPUs, puts to peers included): a rank's subdomain updates -- residual, Eq. 2 flag +
// detection step, the on-chip local solve with prolongation -- are issued one
// after another on one stream, each reading the latest data (R34: a legal
// asynchronous schedule, multiplicative-Schwarz ordered).  The host keeps <= Q
// rounds in flight and stops issuing when every subdomain stopped.
static ras_status run_async_sequential(ras_ctx* c, double tol, int64_t max_iters, int m, double inner_tol, bool exact,
                                       bool* timeout) {
  AsyncRt* A = c->async;
  const int nl = c->nl;
  const int Q = 4;
  std::vector<cudaEvent_t> ev(Q);
  for (auto& e : ev) RAS_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  c->resid_seq = true;
  // consecutive subdomains updated in pairs (two RESIDENT lanes per launch, R34);
  // RAS_ASYNC_PAIRS=0: one after another
  const char* pe = getenv("RAS_ASYNC_PAIRS");
  const bool pairs = !(pe && pe[0] == '0');
  const double t0 = now_s();
  *timeout = false;
  ras_status st = RAS_OK;
  for (int64_t k = 0;; ++k) {
    if (k >= Q && cudaEventSynchronize(ev[k % Q]) != cudaSuccess) {
      st = cuda_err(c, cudaGetLastError(), "async round");
      break;
    }
    int nstopped = 0;
    for (int lp = 0; lp < nl; ++lp) nstopped += ((volatile int32_t*)A->h_lstop)[lp] != 0;
    if (nstopped == nl) break;
    if (now_s() - t0 > c->opt.async_timeout_s) {
      *timeout = true;
      break;
    }
    for (int lp = 0; lp < nl && st == RAS_OK; ++lp) {
      const bool live = !((volatile int32_t*)A->h_lstop)[lp];
      if (pairs && lp + 1 < nl && live && !((volatile int32_t*)A->h_lstop)[lp + 1]) {
        st = enqueue_pair_sweep(c, lp, c->stream, tol, max_iters, m, inner_tol, exact);
        ++lp;
      } else if (live) {
        st = enqueue_sub_sweep(c, lp, c->stream, tol, max_iters, m, inner_tol, exact);
      }
    }
    if (st != RAS_OK) break;
    RAS_CUDA(c, cudaEventRecord(ev[k % Q], c->stream));
  }
  c->resid_seq = false;
  if (*timeout) {
    std::vector<int32_t> ones(nl, 1);
    cudaMemcpy(A->d_lstop, ones.data(), nl * 4, cudaMemcpyHostToDevice);
  }
  cudaStreamSynchronize(c->stream);
  for (auto& e : ev) cudaEventDestroy(e);
  return st;
}

// scripted lock-step mode (single rank): deterministic detector schedule
static ras_status run_scripted(ras_ctx* c, double tol, int64_t max_iters, int m, double inner_tol) {
  AsyncRt* A = c->async;
  const int nl = c->nl;
  if (c->world != 1) return set_err(c, RAS_EINVAL, "scripted detector mode needs world == 1");
  if (c->scripted_sweeps <= 0) return set_err(c, RAS_EINVAL, "no scripted flags set");
  if (A->scripted_n != c->scripted_sweeps) {
    TRY(upload(c, &A->d_scripted, c->scripted));
    A->scripted_n = c->scripted_sweeps;
  }
  RAS_CUDA(c, cudaMemsetAsync(A->d_stop_sweep, 0xff, nl * 8, c->stream));
  Ctl C{A->d_lstop, 1};
  int32_t** bufs[2] = {A->d_boards, A->d_boards2};
  int32_t* raw[2] = {A->board, A->board2};
  for (int64_t k = 0; k < max_iters; ++k) {
    const int cur = (int)(k & 1), prv = cur ^ 1;
    // stop words persist: next <- prev (stop section); reports are rewritten
    RAS_CUDA(c, cudaMemcpyAsync(raw[cur], raw[prv], (size_t)c->plan->P * 4, cudaMemcpyDeviceToDevice, c->stream));
    const Range R = range_all(c);
    TRY(enq_residual(c, c->stream, R, C));
    k_detect_scripted<<<(nl + 127) / 128, 128, 0, c->stream>>>(nl, k, A->det, A->d_scripted, c->scripted_sweeps,
                                                                bufs[prv], bufs[cur], A->d_lstop, A->d_stop_sweep,
                                                                A->d_updates);
    TRY(enq_pcg(c, c->stream, R, C, m, inner_tol, false));
    TRY(enq_prolong(c, c->stream, R, C));
    k_mirror_stops<<<(nl + 127) / 128, 128, 0, c->stream>>>(nl, A->d_lstop, A->h_lstop_dev);
    c->launches += 2;
    RAS_CUDA(c, cudaStreamSynchronize(c->stream));
    int all = 1;
    for (int i = 0; i < nl; ++i) all &= ((volatile int32_t*)A->h_lstop)[i] != 0;
    if (all) break;
  }
  RAS_CUDA(c, cudaGetLastError());
  (void)tol;
  return RAS_OK;
}

// ---------------------------------------------------------------------------
// Put / version stress test (reading R17, Q17; P389-397): the writer rank stores
// epoch-tagged 8-byte words into the reader rank's x window with the same plain
// stores the async puts use, then fences and bumps the reader's version counter
// with a system-scope atomic (the put + flush analogue).  The reader polls the
// counter with ld.acquire.sys and, after observing version v, reads the window:
// a word whose two halves differ is TORN (8-byte stores not single-copy atomic
// over the link), a word older than epoch v-1 is STALE (the release/acquire
// publication failed).  Destroys the x storage of both ranks (debug only).
// ---------------------------------------------------------------------------
static __global__ void k_stress_write(unsigned long long* win, int64_t words, int64_t epochs, int32_t* ver) {
  for (int64_t e = 0; e < epochs; ++e) {
    const unsigned long long tag = ((unsigned long long)(e + 1) << 32) | (unsigned long long)(e + 1);
    for (int64_t i = threadIdx.x; i < words; i += blockDim.x) win[i] = tag;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      atomicAdd_system(ver, 1);
    }
    __syncthreads();
  }
}

static __global__ void k_stress_read(const unsigned long long* win, int64_t words, int64_t epochs, const int32_t* ver,
                                     unsigned long long* out /* torn, stale, regress, observations */) {
  __shared__ int s_v;
  __shared__ unsigned long long s_cnt[3];
  if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
  int last = 0;
  unsigned long long obs = 0, t0 = 0;
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) {
      s_v = ld_acquire_sys(ver);
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (s_v < epochs && t - t0 > 60ull * 1000000000ull) s_v = -1;  // writer never finished: give up (no GPU hang)
    }
    __syncthreads();
    const int v = s_v;
    if (v < 0) {
      obs = 0;  // reported as zero observations: the caller's check fails
      break;
    }
    if (v < last && threadIdx.x == 0) atomicAdd(&s_cnt[2], 1ull);
    last = v;
    unsigned long long torn = 0, stale = 0;
    for (int64_t i = threadIdx.x; i < words; i += blockDim.x) {
      const unsigned long long w = __ldcv(win + i);
      const unsigned hi = (unsigned)(w >> 32), lo = (unsigned)w;
      torn += hi != lo;
      stale += (int64_t)lo < (int64_t)v;  // tag of epoch e is e + 1: version v => every tag >= v
    }
    if (torn) atomicAdd(&s_cnt[0], torn);
    if (stale) atomicAdd(&s_cnt[1], stale);
    ++obs;
    if (v >= epochs) break;
  }
  __syncthreads();
  if (threadIdx.x < 3) out[threadIdx.x] = s_cnt[threadIdx.x];
  if (threadIdx.x == 0) out[3] = obs;
}

ras_status put_stress(ras_ctx* c, int64_t epochs, int64_t words, int64_t* out4) {
  AsyncRt* A = c->async;
  if (c->world != 2) return set_err(c, RAS_EINVAL, "put stress test needs world == 2");
  if (words < 1 || words > c->n_own + c->n_halo || epochs < 1 || epochs > (1 << 30))
    return set_err(c, RAS_EINVAL, "put stress test: words must be in [1, storage of the reader], epochs >= 1");
  int32_t* ver = A->board + 3 * c->plan->P;  // VER section of this rank's board, word 0
  // every allocation before the barrier: with loopback virtual ranks on one device
  // a cudaMalloc / cudaFree may wait for the whole device, i.e. for the other
  // rank's spinning reader, which waits for this rank's writer (deadlock)
  unsigned long long* d_out = nullptr;
  TRY(zalloc(c, &d_out, 4));
  cudaFuncAttributes fa;  // loaded now, not at a launch racing the other rank's spinning kernel
  RAS_CUDA(c, cudaFuncGetAttributes(&fa, k_stress_write));
  RAS_CUDA(c, cudaFuncGetAttributes(&fa, k_stress_read));
  RAS_CUDA(c, cudaMemsetAsync(ver, 0, 4, c->stream));
  RAS_CUDA(c, cudaMemsetAsync(c->d_x, 0, (size_t)words * 8, c->stream));
  TRY(coll_barrier(c));  // the reader's window and counter are clear before the writer starts
  if (c->rank == 0) {
    k_stress_write<<<1, 1024, 0, c->stream>>>((unsigned long long*)A->peer_x[1], words, epochs,
                                              A->peer_board[1] + 3 * c->plan->P);
  } else {
    k_stress_read<<<1, 1024, 0, c->stream>>>((const unsigned long long*)c->d_x, words, epochs, ver, d_out);
  }
  RAS_CUDA(c, cudaGetLastError());
  std::vector<unsigned long long> h(4, 0);
  RAS_CUDA(c, cudaMemcpyAsync(h.data(), d_out, 32, cudaMemcpyDeviceToHost, c->stream));
  RAS_CUDA(c, cudaStreamSynchronize(c->stream));
  TRY(coll_barrier(c));
  dfree(c, d_out);
  for (int i = 0; i < 4; ++i) out4[i] = (int64_t)h[i];
  return RAS_OK;
}

ras_status solve_async(ras_ctx* c, double tol, int64_t max_iters) {
  AsyncRt* A = c->async;
  const int nl = c->nl;
  const bool exact = c->opt.local_solver == RAS_LS_EXACT_PCG;
  int64_t max_rows = 0;
  for (auto& S : c->plan->subs) max_rows = std::max<int64_t>(max_rows, (int64_t)S.omega.size());
  const int m = exact ? (int)std::min<int64_t>(10 * max_rows, INT32_MAX / 2) : c->opt.inner_iters;
  const double inner_tol = exact ? 1e-14 : c->opt.inner_tol;
  const bool kt = c->kt.on;
  c->kt.on = false;  // per-kernel event timing is a sync-mode (single stream) facility
  RAS_CUDA(c, cudaMemsetAsync(A->d_updates, 0, nl * 8, c->stream));
  RAS_CUDA(c, cudaMemsetAsync(A->det.phase, 0, (size_t)nl * kNPhase * 8, c->stream));
  RAS_CUDA(c, cudaStreamSynchronize(c->stream));
  ras_status st = RAS_OK;
  double rel = INFINITY;
  int resumes = 0;
  bool noconv_any = false, timeout = false;
  const double t0 = now_s();
  for (;;) {
    {
      const int32_t f = (c->opt.force_first_stop && resumes == 0) ? 1 : 0;
      RAS_CUDA(c, cudaMemcpyAsync(A->d_force, &f, 4, cudaMemcpyHostToDevice, c->stream));
    }
    TRY(reset_detection(c));
    if (c->opt.scripted_flags) {
      st = run_scripted(c, tol, max_iters, m, inner_tol);
    } else if (c->path == RAS_PCG_RESIDENT && !c->small) {
      st = run_async_sequential(c, tol, max_iters, m, inner_tol, exact, &timeout);
    } else if (c->small && (c->opt.async_persistent == 1 ||
                            (c->opt.async_persistent == 2 && (inner_tol > 0.0 || A->det.seqlock)))) {
      st = run_async_persistent(c, tol, max_iters, m, inner_tol, &timeout);
    } else {
      st = run_async_loop(c, tol, max_iters, m, inner_tol, exact, &timeout);
    }
    if (st != RAS_OK) break;
    c->st.time_to_solution_s = now_s() - t0;
    // post-termination verification (P346-348): barrier, halo refresh, true residual
    const double tv = now_s();
    TRY(barrier(c));
    TRY(sync_exchange(c));
    TRY(global_residual(c, &rel));
    c->st.verify_s += now_s() - tv;
    std::vector<int32_t> nc(nl);
    RAS_CUDA(c, cudaMemcpy(nc.data(), A->d_noconv, nl * 4, cudaMemcpyDeviceToHost));
    int local_nc = 0;
    for (int v : nc) local_nc |= v;
    noconv_any = local_nc || timeout;
    if (c->world > 1) {  // agree on "someone hit max_iters / the watchdog"
      double f = noconv_any ? 1.0 : 0.0;
      TRY(coll_allreduce_f64(c, &f, 1, true));
      noconv_any = f != 0.0;
    }
    if (rel < tol || noconv_any || c->opt.scripted_flags || resumes >= c->opt.max_resumes) break;
    ++resumes;  // R20: verification failed -> clear flags and resume asynchronous iteration
  }
  c->kt.on = kt;
  if (st != RAS_OK) return st;
  c->st.resumes = resumes;
  c->st.final_rel_residual = rel;
  c->st.converged = rel < tol;
  c->st.verified = rel < tol;
  std::vector<int64_t> up(nl);
  RAS_CUDA(c, cudaMemcpy(up.data(), A->d_updates, nl * 8, cudaMemcpyDeviceToHost));
  c->updates = up;
  std::vector<int64_t> srt = up;
  std::sort(srt.begin(), srt.end());
  c->st.updates_min = srt.front();
  c->st.updates_max = srt.back();
  c->st.updates_median = srt[srt.size() / 2];
  c->st.sweeps = srt.back();
  if (c->opt.scripted_flags) {
    c->det_stops.resize(nl);
    RAS_CUDA(c, cudaMemcpy(c->det_stops.data(), A->d_stop_sweep, nl * 8, cudaMemcpyDeviceToHost));
  }
  std::vector<int32_t> ver(c->plan->P);
  RAS_CUDA(c, cudaMemcpy(ver.data(), A->board + 3 * c->plan->P, ver.size() * 4, cudaMemcpyDeviceToHost));
  int64_t fresh = 0;
  for (int v : ver) fresh += v;
  c->st.fresh_halo_reads = fresh;
  // per-phase device time, summed over each subdomain's updates, mean over the local subdomains
  std::vector<double> ph((size_t)nl * kNPhase);
  RAS_CUDA(c, cudaMemcpy(ph.data(), A->det.phase, ph.size() * 8, cudaMemcpyDeviceToHost));
  double tot[kNPhase] = {};
  for (int lp = 0; lp < nl; ++lp)
    for (int k = 0; k < kNPhase; ++k) tot[k] += ph[(size_t)lp * kNPhase + k] / nl;
  c->st.t_residual = tot[PH_RES];
  c->st.t_local_solve = tot[PH_SOLVE];
  c->st.t_prolong = tot[PH_PROL];
  c->st.t_exchange = tot[PH_EXCH];
  c->st.t_convcheck = tot[PH_CHECK];
  if (c->st.converged) return RAS_OK;
  if (noconv_any || c->opt.scripted_flags) return RAS_ENOCONV;
  return set_err(c, RAS_EVERIFY,
                 "async RAS terminated but the true relative residual " + std::to_string(rel) +
                     " >= tol after " + std::to_string(resumes) + " resumes");
}

}  // namespace ras
