// sharded.cuh — Algorithm 1 row-sharded over R ranks, ONE persistent kernel per rank,
// ranks exchanging through peer memory (NVLink / NVSwitch P2P loads and stores), no NCCL.
//
// Decomposition (SURVEY §8(e) "banded" plan, which with full windows is the generic one):
//  * rank r owns the contiguous nnz-balanced rows [row0_r, row1_r) of A;
//  * its rows touch the column window W_r = [wlo_r, whi_r) (min / max column of its rows;
//    [0, n) for dense A);
//  * columns are OWNED by exactly one rank: [own_r, own_{r+1}), conformal to the row ranges
//    (rgdbek_plan_ownership): for banded A a column is owned by a rank whose window holds it,
//    so only the halo columns of neighbouring windows cross the link.
// One iteration (same arithmetic as Algorithm 1, reading R1; P-invariant because every
// random draw is indexed by GLOBAL row / column, reading R5):
//   pass T over the rank's rows -> window partials s_r = (A^(r))^T z^(r), v_r = (A^(r))^T xi^(r)
//   owner of column j: s_j = sum_{q : j in W_q} s_q[j]  (peer reads, rank order: the
//     reduce-scatter that replaces the paper's MPI_AllReduce of A^T z), keys of its
//     owned columns, level-1 histogram of its keys
//   exact global k_c-th key: histograms of every level summed over ranks, level-3 survivors
//     gathered from every rank, ranked; zeta, Z, x_k on owned columns
//   halo copy: zeta, x of the window's non-owned columns from their owners (peer reads)
//   pass N over the rank's rows (w = A zeta, A x_k), z update, row keys, global row selection
//     by the same distributed radix search, xi, X (fused into the next pass T for dense A)
// Global barriers: a two-level barrier — the rank's CTAs meet on the rank-local grid barrier;
// CTA 0 of each rank then publishes the rank's partials (scalars summed over its CTAs in CTA
// order, integer counters, histograms) into a double-buffered exchange block, signals every
// peer with a release store to the peer's flag word, waits for all peers' signals (acquire),
// sums the R published blocks in rank order into a rank-local combined block and releases its
// CTAs.  All ranks therefore take identical decisions from identical bits.
// The same kernel serves R real GPUs (one process per GPU, grid (G, 1), peers' blocks mapped
// by CUDA IPC) and R emulated ranks on one GPU (one cooperative launch of grid (G, R),
// blockIdx.y = rank, every CTA co-resident — B200_PROFILING.md: ranks that wait on one
// another must be one launch when they share a GPU).
#pragma once
#include "persistent.cuh"

namespace rg {

constexpr int MAXR = 8;               // ranks of a peer-memory shard group
constexpr int XSLOTS = 4;             // scalars published per barrier

struct __align__(128) XFlags {
  unsigned int arrive[2][MAXR];       // [round][source rank]: last barrier the source reached
  unsigned int pad[32 - 2 * MAXR];
};

struct __align__(16) XPub {           // one rank's contribution to one barrier
  double scal[XSLOTS];
  unsigned long long acc[2];          // [count, hash] of a block
  unsigned int nsurv, sflag;          // level-3 survivors of this rank; overflow flag
  unsigned int hist[NBINS];
  unsigned int hist2[NBINS];          // speculative level-2 histogram (predicted level-1 bucket)
  Cand surv[SURV_CAP];
};

struct __align__(16) XComb {          // the rank-local sum over ranks (read by all CTAs)
  double scal[XSLOTS];
  double rs[XSLOTS][MAXR];            // the published scalars rank by rank (Algorithm 2)
  unsigned long long acc[2];
  unsigned long long prefix;          // level-3 bucket prefix and count below it
  long long below;
  unsigned int nsurv, sflag;
  unsigned int hist[NBINS];
  unsigned int hist2[NBINS];
  Cand surv[MAXR * SURV_CAP];
};

// Everything a rank knows about the group (device copy per rank; the emulated launch
// holds R of them, indexed by blockIdx.y).
struct ShArgs {
  int R, rank;
  int sys, pad_;                      // 1: ranks on different GPUs (system-scope flags)
  long long own0, own1;               // owned columns of this rank
  long long wlo, whi;                 // this rank's column window
  long long ownb[MAXR + 1];           // owned-column boundaries of every rank
  long long plo[MAXR], phi[MAXR];     // every rank's window
  double* ps[MAXR];                   // peers' s (window partials, then owned sums)
  double* pv[MAXR];                   // peers' v
  double* pzeta[MAXR];                // peers' zeta (authoritative on their owned columns)
  double* px[MAXR];                   // peers' x
  unsigned long long* pkeys[MAXR];    // peers' column keys (Algorithm 2: U on the halo)
  XFlags* pflags[MAXR];               // peers' flag blocks (this rank writes arrive[.][rank])
  XPub* ppub[MAXR];                   // peers' publish blocks [2] (parity of the barrier)
  XComb* comb;                        // this rank's combined block
  GridBar* bar;                       // this rank's local grid barrier
};

// Flag words: system scope across GPUs (peers' memory over NVLink); an emulated group on
// one GPU (ShArgs::sys == 0) needs only device scope, measured ~30 % cheaper per exchange
// on the protocol (tools/sharded_probe.py, profiles/r2/sharded_probe_scope.jsonl).
__device__ __forceinline__ void st_release_x_u32(unsigned int* p, unsigned int v, int sys) {
  if (sys) asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
  else asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_x_u32(const unsigned int* p, int sys) {
  unsigned int v;
  if (sys) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Watchdog of the cross-rank waits: a rank that never arrives (a bug, or a peer process
// that died) traps the kernel after RG_XWAIT_NS instead of hanging the GPU.
#ifndef RG_XWAIT_NS
#define RG_XWAIT_NS 20000000000ull
#endif
__device__ __forceinline__ void x_watch(unsigned int& spins, unsigned long long& t0) {
  if ((++spins & 1023u) == 0u) {
    const unsigned long long t = gtimer();
    if (t0 == 0ull) t0 = t;
    else if (t - t0 > RG_XWAIT_NS) __trap();
  }
}

// Signal round `rd` of exchange number `g` to every rank, then wait until every rank has.
// Called by CTA 0 only, all threads.
__device__ __forceinline__ void x_flags(const ShArgs& x, int rd, unsigned int g) {
  if (x.sys) __threadfence_system();   // this CTA's publish writes before the signal
  else __threadfence();
  __syncthreads();
  if (threadIdx.x < x.R) st_release_x_u32(&x.pflags[threadIdx.x]->arrive[rd][x.rank], g, x.sys);
  if (threadIdx.x < x.R) {
    const unsigned int* f = &x.pflags[x.rank]->arrive[rd][threadIdx.x];
    unsigned int spins = 0u;
    unsigned long long t0 = 0ull;
    while ((int)(ld_acquire_x_u32(f, x.sys) - g) < 0) x_watch(spins, t0);
  }
  __syncthreads();
}

// What one global barrier exchanges.
struct XReq {
  int nslot;                          // scalars: bpart slots summed over the rank's CTAs
  int slot[XSLOTS];
  double direct;                      // nslot == -1: one direct value (prologue)
  unsigned long long* acc;            // rank-local [count, hash] to publish and zero (or null)
  unsigned int* hist;                 // rank-local histogram to publish and zero (or null)
  unsigned int* hist2;                // a second one (the speculative level-2 histogram)
  // level-3 survivors (second exchange round): the rank-local candidate list of the
  // selection side and the selection state (identical in every CTA)
  const Cand* cand;
  unsigned int* ncand;
  const PSel* ps;
};

__device__ __forceinline__ XReq xreq() {
  XReq q;
  q.nslot = 0;
  q.direct = 0.0;
  q.acc = nullptr; q.hist = nullptr; q.hist2 = nullptr; q.cand = nullptr; q.ncand = nullptr;
  q.ps = nullptr;
  return q;
}

// Global barrier over every CTA of every rank with the exchange described by q.
// bgen: the rank-local barrier generation (thread 0's copy); xg: exchange counter
// (identical in every CTA of every rank).  sh_u / sh_l: p_find_bucket scratch.
__device__ void xsync(const PArgs& a, const ShArgs& x, unsigned int& bgen, unsigned int& xg,
                      const XReq& q, unsigned int* sh_u, long long* sh_l) {
  __threadfence();
  __syncthreads();
  GridBar* gb = x.bar;
  const unsigned int myg = bgen;        // valid in thread 0
  xg += 1;
  const unsigned int par = xg & 1u;
  if (blockIdx.x != 0) {
    if (threadIdx.x == 0) {
      bgen = myg + 1u;
      atom_add_acqrel_u32(&gb->count, 1u);
      unsigned int spins = 0u;
      unsigned long long t0 = 0ull;
      while (ld_acquire_u32(&gb->gen) == myg) x_watch(spins, t0);
    }
    __syncthreads();
    return;
  }
  // ---- CTA 0: wait for the rank's other CTAs ----
  if (threadIdx.x == 0) {
    bgen = myg + 1u;
    unsigned int spins = 0u;
    unsigned long long t0 = 0ull;
    while (ld_acquire_u32(&gb->count) != gridDim.x - 1) x_watch(spins, t0);
    gb->count = 0u;
  }
  __syncthreads();
  // ---- publish (parity par): rank partials, counters, histogram ----
  XPub* mine = x.ppub[x.rank] + par;
  const int G = gridDim.x;
  if (q.nslot == -1) {
    if (threadIdx.x == 0) mine->scal[0] = q.direct;
  } else {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (w < q.nslot) {                  // warp w: the rank's sum of slot w over its CTAs
      double t = 0.0;
      for (int c = l; c < G; c += 32) t += __ldcg(a.bpart + q.slot[w] * G + c);
      t = warp_sum(t);
      if (l == 0) mine->scal[w] = t;
    }
  }
  if (q.acc && threadIdx.x < 2) {
    mine->acc[threadIdx.x] = __ldcg(q.acc + threadIdx.x);
    q.acc[threadIdx.x] = 0ull;
  }
  if (q.hist) {
    for (int i = threadIdx.x; i < NBINS; i += PT) {
      mine->hist[i] = __ldcg(q.hist + i);
      q.hist[i] = 0u;
    }
  }
  if (q.hist2) {
    for (int i = threadIdx.x; i < NBINS; i += PT) {
      mine->hist2[i] = __ldcg(q.hist2 + i);
      q.hist2[i] = 0u;
    }
  }
  x_flags(x, 0, xg);
  // ---- combine in rank order ----
  XComb* cb = x.comb;
  if (q.nslot != 0 && threadIdx.x < (q.nslot == -1 ? 1 : q.nslot)) {
    double t = 0.0;
    for (int r = 0; r < x.R; ++r) {
      const double v = __ldcv(&x.ppub[r][par].scal[threadIdx.x]);
      cb->rs[threadIdx.x][r] = v;
      t += v;
    }
    cb->scal[threadIdx.x] = t;
  }
  if (q.acc && threadIdx.x < 2) {
    unsigned long long t = 0ull;
    for (int r = 0; r < x.R; ++r) t += __ldcv(&x.ppub[r][par].acc[threadIdx.x]);
    cb->acc[threadIdx.x] = t;
  }
  if (q.hist) {
    for (int i = threadIdx.x; i < NBINS; i += PT) {
      unsigned int t = 0u;
      for (int r = 0; r < x.R; ++r) t += __ldcv(&x.ppub[r][par].hist[i]);
      cb->hist[i] = t;
    }
  }
  if (q.hist2) {
    for (int i = threadIdx.x; i < NBINS; i += PT) {
      unsigned int t = 0u;
      for (int r = 0; r < x.R; ++r) t += __ldcv(&x.ppub[r][par].hist2[i]);
      cb->hist2[i] = t;
    }
  }
  if (q.cand) {
    // level-3 bucket of the combined histogram, then this rank's survivors in it
    __syncthreads();
    int digit;
    long long below;
    p_find_bucket(cb->hist, q.ps->target - q.ps->below, sh_u, sh_l, digit, below);
    const unsigned long long pre3 = (q.ps->prefix << 12) | (unsigned long long)digit;
    __shared__ unsigned int ns;
    __shared__ int ovf;
    if (threadIdx.x == 0) { ns = 0u; ovf = 0; }
    __syncthreads();
    const unsigned int nc = __ldcg(q.ncand);
    if (nc > CAND_CAP) {
      if (threadIdx.x == 0) ovf = 1;
    } else {
      for (unsigned int c = threadIdx.x; c < nc; c += PT) {
        const Cand e = q.cand[c];
        if ((e.key >> L3_SHIFT) == pre3) {
          const unsigned int s = atomicAdd(&ns, 1u);
          if (s < SURV_CAP) mine->surv[s] = e; else ovf = 1;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      mine->nsurv = ns < SURV_CAP ? ns : SURV_CAP;
      mine->sflag = ovf;
      *q.ncand = 0u;
      cb->prefix = pre3;
      cb->below = q.ps->below + below;
    }
    x_flags(x, 1, xg);
    // every rank's survivors, concatenated in rank order (the rank is by (key, index))
    __shared__ unsigned int base[MAXR + 1];
    if (threadIdx.x == 0) {
      unsigned int t = 0u, f = 0u;
      for (int r = 0; r < x.R; ++r) {
        base[r] = t;
        t += __ldcv(&x.ppub[r][par].nsurv);
        f |= __ldcv(&x.ppub[r][par].sflag);
      }
      base[x.R] = t;
      cb->nsurv = t;
      cb->sflag = f;
    }
    __syncthreads();
    for (int r = 0; r < x.R; ++r) {
      const unsigned int c0 = base[r], cnt = base[r + 1] - base[r];
      for (unsigned int e = threadIdx.x; e < cnt; e += PT) cb->surv[c0 + e] = x.ppub[r][par].surv[e];
    }
  }
  // ---- release this rank's CTAs ----
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) st_release_u32(&gb->gen, myg + 1u);
  __syncthreads();
}

// Rank of the survivors in the combined block -> (tau, tie); every CTA, identical.
__device__ void x_rank_survivors(PSel* ps, const XComb* cb) {
  const int nf = (int)cb->nsurv;
  const long long need = ps->target - ps->below;
  for (int e = threadIdx.x; e < nf; e += PT) {
    const Cand me = cb->surv[e];
    long long rank = 0;
    for (int f = 0; f < nf; ++f) {
      const Cand o = cb->surv[f];
      rank += (o.key < me.key) || (o.key == me.key && o.idx < me.idx);
    }
    if (rank == need - 1) { ps->tau = me.key; ps->tie = me.idx; }
  }
  __syncthreads();
  if (threadIdx.x == 0) ps->mode = SEL_THRESH;
  __syncthreads();
}

// Distributed slow path (survivor or candidate overflow on some rank): the remaining key
// bits and then the index bits, one radix level per global barrier, over every rank's keys.
__device__ void x_sel_slow(PSel* ps, const unsigned long long* __restrict__ keys, long long N,
                           long long idx_base, unsigned int* gh_local, unsigned int* h,
                           const PArgs& a, const ShArgs& x, unsigned int& bgen, unsigned int& xg,
                           unsigned int* sh_u, long long* sh_l) {
  const int shifts[6] = {16, 4, 0, 20, 8, 0};
  const unsigned long long masks[6] = {0xFFF, 0xFFF, 0xF, 0xFFF, 0xFFF, 0xFF};
  unsigned long long kpre = ps->prefix;   // key >> 28
  int kshift = L3_SHIFT;
  unsigned long long ipre = 0;
  int ishift = 32;
  long long below = ps->below;
  const long long target = ps->target;
  for (int lv = 0; lv < 6; ++lv) {
    for (int i = threadIdx.x; i < NBINS; i += PT) h[i] = 0u;
    __syncthreads();
    const bool on_idx = lv >= 3;
    for (long long i = (long long)blockIdx.x * PT + threadIdx.x; i < N; i += (long long)gridDim.x * PT) {
      const unsigned long long key = keys[i];
      const unsigned long long gi = (unsigned long long)(idx_base + i);
      const bool in = on_idx ? (key == kpre && (ishift >= 32 || (gi >> ishift) == ipre))
                             : ((key >> kshift) == kpre);
      if (in) {
        const unsigned long long d = on_idx ? ((gi >> shifts[lv]) & masks[lv])
                                            : ((key >> shifts[lv]) & masks[lv]);
        atomicAdd(&h[d], 1u);
      }
    }
    __syncthreads();
    flush_hist<PT>(h, gh_local, NBINS);
    XReq q = xreq();
    q.hist = gh_local;
    xsync(a, x, bgen, xg, q, sh_u, sh_l);
    int digit;
    long long bl;
    p_find_bucket(x.comb->hist, target - below, sh_u, sh_l, digit, bl);
    below += bl;
    const int bits = (masks[lv] == 0xFFF) ? 12 : (masks[lv] == 0xFF ? 8 : 4);
    if (!on_idx) {
      kpre = (kpre << bits) | (unsigned long long)digit;
      kshift = shifts[lv];
    } else {
      ipre = (ishift >= 32) ? (unsigned long long)digit : ((ipre << bits) | (unsigned long long)digit);
      ishift = shifts[lv];
    }
  }
  if (threadIdx.x == 0) {
    ps->tau = kpre;
    ps->tie = (long long)ipre;
    ps->mode = SEL_THRESH;
    ps->slow |= 1;
  }
  __syncthreads();
}

// Exact global selection of the `kblock` smallest (key, index) over every rank's keys,
// given this rank's level-1 histogram (already accumulated in gh[0..NBINS)).
// `first` is extra payload of the first exchange (its scalars come back in first_out /
// first_rs); `gspec` is this rank's level-2 histogram of the keys whose level-1 digit is
// `pred` (-1 = no speculation), built while the keys were made: when the level-1 bucket
// is pred, the level-2 scan and its exchange are skipped.  digit_out = the resolved
// level-1 bucket (-1 when no radix search ran).  Levels 2 and 3 scan the rank's own keys;
// 2-3 global exchanges.
__device__ void x_select(PSel* ps, const unsigned long long* __restrict__ keys, long long N_local,
                         long long idx_base, long long N_global, long long kblock, unsigned int* gh,
                         Cand* cand, unsigned int* ncand, unsigned int* h, const PArgs& a,
                         const ShArgs& x, unsigned int& bgen, unsigned int& xg, unsigned int* sh_u,
                         long long* sh_l, XReq first, double* first_out, double* first_rs,
                         unsigned int* gspec, int pred, int& digit_out) {
  digit_out = -1;
  {
    XReq q = first;
    q.hist = gh;
    if (pred >= 0) q.hist2 = gspec;
    xsync(a, x, bgen, xg, q, sh_u, sh_l);
    if (first.nslot > 0) {
      if (first_out) *first_out = x.comb->scal[0];
      if (first_rs && threadIdx.x < x.R) first_rs[threadIdx.x] = x.comb->rs[0][threadIdx.x];
    }
  }
  p_sel_level1(ps, x.comb->hist, N_global, kblock, sh_u, sh_l);
  if (ps->mode != SEL_PENDING) return;          // identical in every CTA of every rank
  const int digit = (int)ps->prefix;            // the level-1 bucket
  if (pred >= 0 && digit == pred) {
    p_sel_level2(ps, x.comb->hist2, sh_u, sh_l);              // speculation hit
  } else {
    p_sel_scan<2>(ps, keys, N_local, idx_base, gh + NBINS, cand, ncand, h);
    XReq q = xreq();
    q.hist = gh + NBINS;
    xsync(a, x, bgen, xg, q, sh_u, sh_l);
    p_sel_level2(ps, x.comb->hist, sh_u, sh_l);
  }
  digit_out = digit;
  p_sel_scan<3>(ps, keys, N_local, idx_base, gh + 2 * NBINS, cand, ncand, h);
  {
    XReq q = xreq();
    q.hist = gh + 2 * NBINS;
    q.cand = cand; q.ncand = ncand; q.ps = ps;
    xsync(a, x, bgen, xg, q, sh_u, sh_l);
  }
  if (threadIdx.x == 0) { ps->prefix = x.comb->prefix; ps->below = x.comb->below; }
  __syncthreads();
  if (x.comb->sflag) {
    x_sel_slow(ps, keys, N_local, idx_base, gh + NBINS, h, a, x, bgen, xg, sh_u, sh_l);
    return;
  }
  x_rank_survivors(ps, x.comb);
}

// Rank-local exact selection (Algorithm 2's own rows): the single-GPU radix
// levels over this rank's keys, separated by the rank's grid barrier.  The histogram
// levels and the candidate count are zeroed by x_zero_local before their next use.
__device__ void x_select_local(PSel* ps, const unsigned long long* __restrict__ keys, long long N,
                               long long idx_base, long long kblock, unsigned int* gh, Cand* cand,
                               unsigned int* ncand, unsigned int* h, const ShArgs& x,
                               unsigned int& bgen, unsigned int* sh_u, long long* sh_l) {
  grid_sync(x.bar, bgen);                          // the rank's level-1 histogram is complete
  p_sel_level1(ps, gh, N, kblock, sh_u, sh_l);
  if (ps->mode != SEL_PENDING) return;
  p_sel_scan<2>(ps, keys, N, idx_base, gh + NBINS, cand, ncand, h);
  grid_sync(x.bar, bgen);
  p_sel_level2(ps, gh + NBINS, sh_u, sh_l);
  p_sel_scan<3>(ps, keys, N, idx_base, gh + 2 * NBINS, cand, ncand, h);
  grid_sync(x.bar, bgen);
  p_sel_level3(ps, gh + 2 * NBINS, cand, ncand, keys, N, idx_base, h, sh_u, sh_l);
}

__device__ void x_zero_local(unsigned int* gh, unsigned int* ncand) {
  for (int i = blockIdx.x * PT + threadIdx.x; i < 3 * NBINS; i += gridDim.x * PT) gh[i] = 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) *ncand = 0u;
}

// ---------------------------------------------------------------------------
// The sharded persistent kernel: Algorithm 1 (LAZY = false) or the paper's parallel
// Algorithm 2 over the R ranks as its processes (LAZY = true; reading R28: the global U
// from A^T z, local first-Krylov z-steps and own-row samples J^(p) of round(eta d_p) rows,
// the lazily averaged x += (1/R) sum_p (X_p / V_p) (A^(p))^T xi_p).
// Pseudoinverse-free update, random selection.
// ---------------------------------------------------------------------------
template <bool DENSE, bool LAZY>
__global__ void __launch_bounds__(PT, 1) k_sharded(const PArgs* __restrict__ pa,
                                                   const ShArgs* __restrict__ sa) {
  __shared__ __align__(16) unsigned int h[NBINS];
  __shared__ __align__(8) unsigned long long tbar[(PT / TG) * TRING];
  __shared__ double sh[PW];
  __shared__ unsigned int sh_u[4];
  __shared__ long long sh_l[40];
  __shared__ PSel ps;
  __shared__ PArgs a;
  __shared__ ShArgs x;
  __shared__ double lzX[MAXR], lzV[MAXR];        // Algorithm 2: every rank's X_p, V_p
  extern __shared__ __align__(16) double dyn[];
  if (threadIdx.x == 0) { a = pa[blockIdx.y]; x = sa[blockIdx.y]; }
  if (threadIdx.x < MAXR) { lzX[threadIdx.x] = 0.0; lzV[threadIdx.x] = 0.0; }
  __syncthreads();
  TileRing tring{tbar + (threadIdx.x / TG) * TRING, 0u};
  if (!DENSE) tile_rings_init(tbar);
  Scal* st = a.st;
  TraceRec* tr = a.tr;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  const int G = gridDim.x;
  double* bp = a.bpart;
  long long k = st->k;
  const long long k_begin = st->k_begin, k_end = st->k_end;
  const double tol = st->tol;
  const int stop_mode = st->stop_mode, has_ref = st->has_ref;
  const unsigned long long seed = st->seed;
  const double xsnorm2 = st->xsnorm2;
  const long long kc = st->kc, kr = LAZY ? a.lz_kr[0] : st->kr;
  int pending = st->pending;
  double X = st->X;
  long long kp_prev = st->kp_prev, kpp_prev = st->kpp_prev;
  const int n = a.n, m_loc = a.m_loc;
  const long long m_glob = st->m_global;
  const long long own0 = x.own0, nown = x.own1 - x.own0;
  unsigned int* hn = a.hist;
  unsigned int* hm = a.hist + 3 * NBINS;
  Cand* cn = a.cand;
  Cand* cm = a.cand + CAND_CAP;
  double* sown = LAZY ? a.lz_g : a.s;            // the owned columns' s = A^T z
  unsigned int* hspec = a.hist + 6 * NBINS;      // speculative level-2 histograms [2][NBINS]
  // speculative level-2 histograms: the predicted level-1 bucket is the last one
  // (identical in every CTA of every rank); -1 = no speculation
  int predU = -1, predJ = -1;
  unsigned int bgen = 0, xg = st->xgen;
  if (threadIdx.x == 0) bgen = ld_acquire_u32(&x.bar->gen);
  const XComb* cb = x.comb;
  // ---- prologue: ||b||^2 over ranks ----
  double bnorm2;
  {
    XReq q = xreq();
    q.nslot = -1;
    q.direct = st->bnorm2;             // this rank's ||b_r||^2
    xsync(a, x, bgen, xg, q, sh_u, sh_l);
    bnorm2 = cb->scal[0];
  }

  for (;;) {
    // ===== P1: pass T over the rank's rows: window partials s_r, v_r =====
    if constexpr (DENSE) {
      double Xp = 0.0;
      long long cnt = 0;
      unsigned long long hs = 0ull;
      if (a.capJ && pending)
        p_capture(a.capJ + ((k - 1) & 1) * (long long)m_loc, &ps, a.keys_m, a.row0,
                  blockIdx.x * PT + threadIdx.x, m_loc, G * PT);
      p_dense_passT(a, pending, dyn, nullptr, nullptr, &ps, &Xp, &cnt, &hs);
      if (pending) {
        cnt = warp_sum_ll(cnt);
        hs = warp_sum_u64(hs);
        if ((threadIdx.x & 31) == 0 && (cnt || hs)) {
          atomicAdd(&a.acc[2], (unsigned long long)cnt);
          atomicAdd(&a.acc[3], hs);
        }
        const double xb = pblock_sum(Xp, sh);
        if (threadIdx.x == 0) bp[SL_X * G + blockIdx.x] = xb;
      }
      grid_sync(x.bar, bgen);
      // the rank's column sums of its CTA partials (all n columns: the dense window)
      {
        constexpr int CW = 64, NG = PT / CW;
        double* red = dyn;
        const int cpb = (n + G - 1) / G;
        const int c0 = min(n, blockIdx.x * cpb), c1 = min(n, c0 + cpb);
        const int cl = threadIdx.x % CW, g = threadIdx.x / CW;
        for (int cbk = c0; cbk < c1; cbk += CW) {
          const int j = cbk + cl;
          double sj = 0.0, vj = 0.0;
          if (j < c1) {
            for (int p = g; p < G; p += NG) {
              const double* qq = a.part + (long long)p * 2 * n + j;
              sj += __ldcg(qq);
              if (pending) vj += __ldcg(qq + n);
            }
          }
          red[g * CW + cl] = sj;
          red[(NG + g) * CW + cl] = vj;
          __syncthreads();
          if (g == 0 && j < c1) {
            double ts = 0.0, tv = 0.0;
#pragma unroll
            for (int t = 0; t < NG; ++t) { ts += red[t * CW + cl]; tv += red[(NG + t) * CW + cl]; }
            a.s[j] = ts;
            a.v[j] = tv;
          }
          __syncthreads();
        }
      }
    } else {
      double d1 = 0.0, d2 = 0.0;
      const int g = threadIdx.x / TG;
      csr_tiles(blockIdx.x * (PT / TG) + g, G * (PT / TG), threadIdx.x % TG, 1 + g,
                reinterpret_cast<TileSmem*>(dyn) + g, tring, a.cp, a.ri, a.rv, a.tilesT,
                a.tilepT, a.ntilesT, a.z, a.xi, pending, nullptr, a.s, a.v, d1, d2, nullptr, 0,
                a.vecT);
      grid_sync(x.bar, bgen);
    }
    {
      // every rank's window partials are complete after this global barrier, which also
      // carries X, |J|, hash of the row step k-1 (dense: formed in this pass T; sparse:
      // in the row-mask sweep that ended the previous iteration)
      XReq q = xreq();
      q.nslot = 1; q.slot[0] = SL_X;
      q.acc = a.acc + 2;
      xsync(a, x, bgen, xg, q, sh_u, sh_l);
      if (pending) {
        X = cb->scal[0];
        if (LAZY && threadIdx.x < x.R) lzX[threadIdx.x] = cb->rs[0][threadIdx.x];
        const long long kppf = (long long)cb->acc[0];
        if (lead) {
          if (!LAZY && kppf != (ps.mode == SEL_NONE ? 0 : ps.target)) st->error |= 2;
          if (TraceRec* t = trace_at(tr, st, k - 1)) { t->kpp = kppf; t->hash_j = cb->acc[1]; t->X = X; }
        }
        kpp_prev = kppf;
      }
    }
    if constexpr (LAZY) x_zero_local(hm, a.ncand + 1);   // the rank's row selection is read

    // ===== P2: owned columns: s, v summed over the ranks whose window holds them;
    //           column keys, level-1 histogram (+ the speculative level-2 one), V partial =====
    unsigned int* h2 = reinterpret_cast<unsigned int*>(dyn);       // free between the passes
    for (int i = threadIdx.x; i < NBINS; i += PT) { h[i] = 0u; h2[i] = 0u; }
    __syncthreads();
    double Vp = 0.0;
    if constexpr (LAZY) {
      // V_p = ||(A^(p))^T xi_p||^2 over this rank's window (its own partial)
      if (pending)
        for (long long j = x.wlo + (long long)blockIdx.x * PT + threadIdx.x; j < x.whi; j += (long long)G * PT) {
          const double vj = a.v[j];
          Vp += vj * vj;
        }
    }
    for (long long jl = (long long)blockIdx.x * PT + threadIdx.x; jl < nown; jl += (long long)G * PT) {
      const long long j = own0 + jl;
      double sj = 0.0, vj = 0.0;
      for (int r = 0; r < x.R; ++r) {
        if (j >= x.plo[r] && j < x.phi[r]) {
          sj += __ldcv(x.ps[r] + j);
          if (!LAZY && pending) vj += __ldcv(x.pv[r] + j);
        }
      }
      sown[j] = sj;
      if constexpr (!LAZY) {
        a.v[j] = vj;
        if (pending) Vp += vj * vj;
      }
      const double gm = a.gamma[j];
      const double eps = gm > 0.0 ? __ddiv_rn(__dmul_rn(sj, sj), gm) : 0.0;
      const unsigned long long key = sel_key(eps, (unsigned long long)j, k, 0u, seed, 0);
      a.keys_n[j] = key;
      atomicAdd(&h[key >> L1_SHIFT], 1u);
      if ((int)(key >> L1_SHIFT) == predU) atomicAdd(&h2[(key >> L2_SHIFT) & 0xFFFull], 1u);
    }
    __syncthreads();
    flush_hist<PT>(h, hn, NBINS);
    if (predU >= 0) flush_hist<PT>(h2, hspec, NBINS);
    {
      const double vb = pblock_sum(Vp, sh);
      if (threadIdx.x == 0) bp[SL_V * G + blockIdx.x] = vb;
    }
    // ===== P3-P5: the global column selection U (its first exchange also carries V) =====
    __shared__ double Vsh;
    {
      XReq first = xreq();
      first.nslot = 1; first.slot[0] = SL_V;
      int d;
      x_select(&ps, a.keys_n + own0, nown, own0, n, kc, hn, cn, a.ncand, h, a, x, bgen, xg, sh_u,
               sh_l, first, threadIdx.x == 0 ? &Vsh : nullptr, LAZY ? lzV : nullptr, hspec, predU, d);
      predU = d;                                    // speculate: the bucket repeats
                                                    // (profiles/r2/sharded_probe_r2i_spec.jsonl)
    }
    __syncthreads();
    const double V = Vsh;
    const int do_x = pending && kpp_prev > 0 && V > 0.0;
    const double alpha_x = do_x ? __ddiv_rn(X, V) : 0.0;
    if (lead && pending) {
      if (TraceRec* t = trace_at(tr, st, k - 1)) t->V = V;
    }
    if (lead && ps.slow) st->selstat[1] += 1;
    // |U|, hash and Z on owned columns (Algorithm 1: zeta = s on U); x_k; ||x - x*||^2
    {
      double Zp = 0.0, Rp = 0.0;
      long long cnt = 0;
      unsigned long long hs = 0ull;
      for (long long jl = (long long)blockIdx.x * PT + threadIdx.x; jl < nown; jl += (long long)G * PT) {
        const long long j = own0 + jl;
        const double sj = sown[j];
        const bool sel = p_selected(&ps, a.keys_n[j], j);
        if (!LAZY) a.zeta[j] = sel ? sj : 0.0;
        if (sel) { Zp += sj * sj; cnt += 1; hs += splitmix64((unsigned long long)j); }
        double xj = a.x[j];
        if constexpr (LAZY) {
          // x_k = x_{k-1} + (1/R) sum_p (X_p / V_p) v_p, v_p over p's window
          if (pending) {
            double t = 0.0;
            for (int r = 0; r < x.R; ++r)
              if (lzX[r] > 0.0 && lzV[r] > 0.0 && j >= x.plo[r] && j < x.phi[r])
                t = __dadd_rn(t, __dmul_rn(__ddiv_rn(lzX[r], lzV[r]), __ldcv(x.pv[r] + j)));
            xj = __dadd_rn(xj, __ddiv_rn(t, (double)x.R));
            a.x[j] = xj;
          }
        } else {
          if (do_x) { xj = __dadd_rn(xj, __dmul_rn(alpha_x, a.v[j])); a.x[j] = xj; }
        }
        if (has_ref) { const double d = xj - a.xstar[j]; Rp += d * d; }
      }
      if (a.capU)
        p_capture(a.capU + (k & 1) * (long long)n + own0, &ps, a.keys_n + own0, own0,
                  blockIdx.x * PT + threadIdx.x, (int)nown, G * PT);
      cnt = warp_sum_ll(cnt);
      hs = warp_sum_u64(hs);
      if ((threadIdx.x & 31) == 0 && (cnt || hs)) {
        atomicAdd(&a.acc[0], (unsigned long long)cnt);
        atomicAdd(&a.acc[1], hs);
      }
      const double zb = pblock_sum(Zp, sh);
      const double rb = pblock_sum(Rp, sh);
      if (threadIdx.x == 0) { bp[SL_Z * G + blockIdx.x] = zb; bp[SL_R * G + blockIdx.x] = rb; }
    }
    pending = 0;
    double Z, relerr2;
    long long kp;
    {
      XReq q = xreq();
      q.nslot = 2; q.slot[0] = SL_Z; q.slot[1] = SL_R;
      q.acc = a.acc;
      xsync(a, x, bgen, xg, q, sh_u, sh_l);
      Z = cb->scal[0];
      relerr2 = cb->scal[1];
      kp = (long long)cb->acc[0];
      if (lead) {
        if (kp != (ps.mode == SEL_NONE ? 0 : ps.target)) st->error |= 1;
        if (TraceRec* t = trace_at(tr, st, k)) { t->k = k; t->kp = kp; t->hash_u = cb->acc[1]; if (!LAZY) t->Z = Z; }
      }
    }
    // ===== halo: the window's columns owned by other ranks =====
    double Zl = 0.0;                               // Algorithm 2: this rank's Z_p partial
    if constexpr (LAZY) {
      // zeta_p = (A^(p))^T z^(p) on U over the window; U on a halo column is
      // decided from its owner's key
      for (long long j = x.wlo + (long long)blockIdx.x * PT + threadIdx.x; j < x.whi; j += (long long)G * PT) {
        int o = x.rank;
        if (j < own0 || j >= x.own1)
          for (int r = 0; r < x.R; ++r) if (j >= x.ownb[r] && j < x.ownb[r + 1]) o = r;
        const unsigned long long key = o == x.rank ? a.keys_n[j] : __ldcv(x.pkeys[o] + j);
        if (o != x.rank) a.x[j] = __ldcv(x.px[o] + j);
        const double gj = a.s[j];
        const bool sel = p_selected(&ps, key, j);
        a.zeta[j] = sel ? gj : 0.0;
        if (sel) Zl += gj * gj;
      }
      const double zb = pblock_sum(Zl, sh);
      if (threadIdx.x == 0) bp[SL_MAXN * G + blockIdx.x] = zb;
    } else {
      for (int r = 0; r < x.R; ++r) {
        if (r == x.rank) continue;
        const long long lo = max(x.wlo, x.ownb[r]), hi = min(x.whi, x.ownb[r + 1]);
        for (long long j = lo + (long long)blockIdx.x * PT + threadIdx.x; j < hi; j += (long long)G * PT) {
          a.zeta[j] = __ldcv(x.pzeta[r] + j);
          a.x[j] = __ldcv(x.px[r] + j);
        }
      }
    }
    grid_sync(x.bar, bgen);
    const double Zr = LAZY ? slot_sum(bp, SL_MAXN, sh) : Z;

    // ===== P6: pass N over the rank's rows (w = A zeta, A x_k), W / ||b - A x||^2 =====
    {
      double Wp = 0.0, Yp = 0.0;
      if constexpr (DENSE) {
        p_dense_passN(a, dyn, Wp, Yp);
      } else {
        const int g = threadIdx.x / TG;
        csr_tiles(blockIdx.x * (PT / TG) + g, G * (PT / TG), threadIdx.x % TG, 1 + g,
                  reinterpret_cast<TileSmem*>(dyn) + g, tring, a.rp, a.ci, a.cv, a.tilesN,
                  a.tilepN, a.ntilesN, a.zeta, a.x, 1, a.b, a.w, a.ax, Wp, Yp, nullptr, 0, a.vecN,
                  RG_REV_N);
      }
      const double wb = pblock_sum(Wp, sh);
      const double yb = pblock_sum(Yp, sh);
      if (threadIdx.x == 0) { bp[SL_W * G + blockIdx.x] = wb; bp[SL_Y * G + blockIdx.x] = yb; }
    }
    double W, Y, Wr;
    {
      XReq q = xreq();
      q.nslot = LAZY ? 3 : 2; q.slot[0] = SL_W; q.slot[1] = SL_Y; q.slot[2] = SL_MAXN;
      xsync(a, x, bgen, xg, q, sh_u, sh_l);
      W = cb->scal[0];
      Y = cb->scal[1];
      Wr = LAZY ? cb->rs[0][x.rank] : W;
      if (LAZY) Z = cb->scal[2];                 // sum over ranks of Z_p (trace)
    }
    // ===== P8: stop test on x_k; z_{k+1}, r, row keys, level-1 histogram =====
    {
      const double rse = Y / bnorm2;
      const double rel = has_ref ? sqrt(relerr2 / xsnorm2) : __longlong_as_double(0x7FF8000000000000ll);
      int halt = 0, outcome = RGDBEK_MAX_ITER;
      if (k > k_begin) {
        if (stop_mode == RGDBEK_STOP_RSE && rse <= tol) { halt = 1; outcome = RGDBEK_CONVERGED; }
        else if (stop_mode == RGDBEK_STOP_REL_ERR && rel <= tol) { halt = 1; outcome = RGDBEK_CONVERGED; }
        else if (kp_prev == 0 && kpp_prev == 0) { halt = 1; outcome = RGDBEK_STALLED; }
      }
      if (!halt && (k > k_begin || k_end == k_begin) && k >= k_end) { halt = 1; outcome = RGDBEK_MAX_ITER; }
      if (lead) {
        if (TraceRec* t = trace_at(tr, st, k)) { t->W = W; if (LAZY) t->Z = Z; }
        if (k >= 1) { if (TraceRec* t = trace_at(tr, st, k - 1)) t->rse = rse; }
      }
      if (halt) {
        if (lead) {
          st->halted = 1; st->outcome = outcome; st->iters = k; st->rse_out = rse;
          st->relerr_out = rel; st->k = k; st->pending = 0; st->X = X;
          st->kp_prev = kp_prev; st->kpp_prev = kpp_prev;
          st->Z = Z; st->W = W; st->Y = Y; st->V = V; st->relerr2 = relerr2;
          st->npass += 2 * (k - k_begin + 1);
          st->xgen = xg;
          st->bnorm2_global = bnorm2;
        }
        return;
      }
    }
    unsigned int* h2m = reinterpret_cast<unsigned int*>(dyn);
    for (int i = threadIdx.x; i < NBINS; i += PT) { h[i] = 0u; h2m[i] = 0u; }
    __syncthreads();
    {
      const int doz = kp > 0 && Wr > 0.0;
      const double az = doz ? __ddiv_rn(Zr, Wr) : 0.0;
      for (int i = blockIdx.x * PT + threadIdx.x; i < m_loc; i += G * PT) {
        double zi = a.z[i];
        if (doz) { zi = __dsub_rn(zi, __dmul_rn(az, a.w[i])); a.z[i] = zi; }
        const double ri = __dsub_rn(__dsub_rn(a.b[i], zi), a.ax[i]);
        a.r[i] = ri;
        const double p = a.rho[i];
        const double eps = p > 0.0 ? __ddiv_rn(__dmul_rn(ri, ri), p) : 0.0;
        const unsigned long long key = sel_key(eps, (unsigned long long)(a.row0 + i), k, 1u, seed, 0);
        a.keys_m[i] = key;
        atomicAdd(&h[key >> L1_SHIFT], 1u);
        if (!LAZY && (int)(key >> L1_SHIFT) == predJ) atomicAdd(&h2m[(key >> L2_SHIFT) & 0xFFFull], 1u);
      }
    }
    __syncthreads();
    flush_hist<PT>(h, hm, NBINS);
    if (!LAZY && predJ >= 0) flush_hist<PT>(h2m, hspec + NBINS, NBINS);
    // ===== P9-P11: the row selection J (Algorithm 2: this rank's own rows) =====
    if constexpr (LAZY) {
      x_select_local(&ps, a.keys_m, m_loc, a.row0, kr, hm, cm, a.ncand + 1, h, x, bgen, sh_u, sh_l);
    } else {
      int d;
      x_select(&ps, a.keys_m, m_loc, a.row0, m_glob, kr, hm, cm, a.ncand + 1, h, a, x, bgen, xg,
               sh_u, sh_l, xreq(), nullptr, nullptr, hspec + NBINS, predJ, d);
      predJ = d;
    }
    if (lead && ps.slow) st->selstat[1] += 1;
    if constexpr (!DENSE) {
      // xi = r on J, X, |J|, hash (dense: formed in the next pass T)
      double Xp = 0.0;
      long long cnt = 0;
      unsigned long long hs = 0ull;
      for (int i = blockIdx.x * PT + threadIdx.x; i < m_loc; i += G * PT) {
        const long long gi = a.row0 + i;
        const double ri = a.r[i];
        const bool sel = p_selected(&ps, a.keys_m[i], gi);
        a.xi[i] = sel ? ri : 0.0;
        if (sel) { Xp += ri * ri; cnt += 1; hs += splitmix64((unsigned long long)gi); }
      }
      if (a.capJ)
        p_capture(a.capJ + (k & 1) * (long long)m_loc, &ps, a.keys_m, a.row0,
                  blockIdx.x * PT + threadIdx.x, m_loc, G * PT);
      cnt = warp_sum_ll(cnt);
      hs = warp_sum_u64(hs);
      if ((threadIdx.x & 31) == 0 && (cnt || hs)) {
        atomicAdd(&a.acc[2], (unsigned long long)cnt);
        atomicAdd(&a.acc[3], hs);
      }
      const double xb = pblock_sum(Xp, sh);
      if (threadIdx.x == 0) bp[SL_X * G + blockIdx.x] = xb;
      // X, |J|, hash are published by the next iteration's first global barrier
    }
    kp_prev = kp;
    pending = 1;
    k += 1;
    __syncthreads();
  }
}

}  // namespace rg
