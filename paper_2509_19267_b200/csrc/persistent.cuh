// persistent.cuh — the whole RGDBEK iteration loop as ONE persistent kernel.
//
// One CTA of PT threads per SM (or fewer for small problems; 1 CTA for C1),
// all co-resident, separated by a software grid barrier at the ~10 grid-wide
// dependencies of an iteration (pass T -> scores -> 3 selection levels ->
// mask -> pass N -> stop test + z update -> 3 levels -> mask).  Every global
// scalar (V, Z, W, ||b-Ax||^2, X, block sizes, radix buckets) is recomputed
// redundantly by every CTA from the same per-CTA partials in the same order,
// so all CTAs take identical decisions without a second barrier; CTA 0 alone
// writes the Scal state and the trace.  The host launches it once per
// rgdbek_solve / rgdbek_step call.
//
// Same method, same arithmetic and same reduction orders per launch geometry
// as the multi-kernel graph engine (kernels.cuh); tests run both.
#pragma once
#include "kernels.cuh"

namespace rg {

constexpr int PT = 1024;                  // threads per persistent CTA
constexpr int PW = PT / 32;
constexpr int ZCH = 1024;                 // rows of z / xi staged per chunk (pass T)
#ifndef RG_VEC_PREFETCH
#define RG_VEC_PREFETCH 1
#endif
#ifndef RG_VEC_PREFETCH2
#define RG_VEC_PREFETCH2 1      // mask sweeps (P5, P11) pipelined too: C2c +1 %, C3 +2 %, C4 -2 %
#endif
#ifndef RG_SCAN_VU
#define RG_SCAN_VU 6       // keys in flight per thread in the grid-wide level-2/3 scans (4: C3 -1.3 %)
#endif
#ifndef RG_FUSE_XI
#define RG_FUSE_XI 1      // dense: xi = r on J formed while pass T stages its rows (no P11 sweep)
#endif
#ifndef RG_SPEC_U
#define RG_SPEC_U 1       // sparse: speculative column level 2 built in pass T's key epilogue
#endif
constexpr int PN_RB = 256;                // max rows per batch (dense pass N)
constexpr int PN_QMAX = 8;                // max column chunks per row (dense pass N)
#ifndef RG_LOCAL_SEL_MAX
#define RG_LOCAL_SEL_MAX 32768
#endif
constexpr int LOCAL_SEL_MAX = RG_LOCAL_SEL_MAX;   // selections over <= this many keys run CTA-locally

struct GridBar {
  unsigned int count;
  unsigned int pad0[31];
  unsigned int gen;
  unsigned int pad1[31];
};

enum : int { SL_V = 0, SL_Z, SL_R, SL_W, SL_Y, SL_X, SL_MAXN, SL_MAXM, SL_NUM };
constexpr int LZ_MAX = 8;                  // Algorithm 2: at most 8 logical processes

struct PArgs {
  int dense, m_loc, n, vecN, vecT, Q, CH;
  long long row0, lda;
  const double* A;
  const long long* rp; const int* ci; const double* cv;
  const long long* cp; const int* ri; const double* rv;
  const double *b, *rho, *gamma, *xstar;
  double *x, *s, *v, *zeta, *z, *w, *ax, *r, *xi;
  unsigned long long *keys_n, *keys_m;
  double* part;                     // dense pass T partials [G][2][n]
  double* bpart;                    // [SL_NUM][G]
  unsigned int* hist;               // [2 sides][3 levels][NBINS]
  Cand* cand;                       // [2][CAND_CAP]
  unsigned long long* acc;          // [2 sides][count, hash]
  unsigned int* ncand;              // [2]
  Scal* st;
  TraceRec* tr;
  GridBar* bar;
  unsigned long long* ptime;        // optional per-phase device time (ns), [16]
  const int* tilesN; const int* tilesT;
  const long long* tilepN; const long long* tilepT;   // first nonzero of each tile
  int ntilesN, ntilesT;
  int greedy;                       // 1 = GDBEK threshold sets instead of sampling
  double eta;
  int pn_smem;                      // dense pass N: zeta / x staged in shared memory
  // optional block capture (rgdbek_set_capture): selection masks of U_k / J_k at
  // parity k & 1, [2][n] and [2][m_loc]; nullptr = off
  unsigned char* capU;
  unsigned char* capJ;
  int pt_rows;                      // dense pass T: one-sweep register-column form (opt-in)
  // Algorithm 2 (lazy averaging, P logical row processes; k_persistent<true, true>)
  int lzP, lzGp;                    // processes; CTAs per process (G = lzP * lzGp)
  long long lz_r0[LZ_MAX + 1];      // process row ranges [lz_r0[p], lz_r0[p + 1])
  long long lz_kr[LZ_MAX];          // per-process row block sizes round(eta d_p)
  double* lz_g;                     // [P][n] (A^(p))^T z^(p)
  double* lz_v;                     // [P][n] (A^(p))^T xi^(p)
  double* lz_zeta;                  // [P][n] zeta_p = g_p on U
  unsigned int* lz_hist;            // [P][NBINS] level-1 histograms of the row keys
  double* lz_slots;                 // [2 P][G]: per-CTA partials of V_p, Z_p
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Sense-free generation barrier: one acq_rel ticket per CTA, the last arriver
// resets the count and bumps the generation with a release store; the others
// spin on an acquire load (no full fences: the release/acquire pair orders
// every CTA's prior global writes before every CTA's later reads).
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned int atom_add_acqrel_u32(unsigned int* p, unsigned int v) {
  unsigned int old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// gen: thread 0's copy of the barrier generation (read once at kernel start).
// The ticket RMWs form a release sequence on `count`; the last arriver
// (acquire) publishes the next generation with a release store; waiters spin
// on an acquire load (which also invalidates the SM's L1, so read-only-path
// loads of vectors rewritten in earlier phases see the new values).
__device__ __forceinline__ void grid_sync(GridBar* gb, unsigned int& gen) {
  __syncthreads();
  if (gridDim.x == 1) return;
  if (threadIdx.x == 0) {
    const unsigned int g = gen++;
    const unsigned int t = atom_add_acqrel_u32(&gb->count, 1u);
    if (t == gridDim.x - 1) {
      gb->count = 0u;                       // ordered before the release below
      st_release_u32(&gb->gen, g + 1u);
    } else {
      while (ld_acquire_u32(&gb->gen) == g) { }
    }
  }
  __syncthreads();
}

// Block-wide sum of one double per thread, same tree in every CTA.
__device__ __forceinline__ double pblock_sum(double v, double* sh) {
  return block_sum<PT>(v, sh);
}

// Sum over the G per-CTA partials of one slot (identical in every CTA).
// Algorithm 2: P sums of per-CTA partials, out[p] = sum_c base[p * pstride + c]
// for c in [p * cstart, p * cstart + count); warp p sums, lanes strided, fixed
// tree (deterministic).  Per-process sums over the process's own CTAs use
// (pstride 0, cstart Gp, count Gp); sums over every CTA of a per-process
// quantity use (pstride G, cstart 0, count G).  out[] is shared memory, valid
// for every thread on return.
__device__ __forceinline__ void lz_sums(const double* base, int pstride, int cstart, int count,
                                        int P, double* out) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (w < P) {
    double t = 0.0;
    const double* q = base + (long long)w * pstride + (long long)w * cstart;
    for (int c = l; c < count; c += 32) t += __ldcg(q + c);
    t = warp_sum(t);
    if (l == 0) out[w] = t;
  }
  __syncthreads();
}

__device__ __forceinline__ double slot_sum(const double* bpart, int slot, double* sh) {
  double t = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += PT) t += __ldcg(bpart + slot * gridDim.x + i);
  return pblock_sum(t, sh);
}

// Block / grid maxima (greedy mode): fmax is order-independent, hence identical everywhere.
__device__ __forceinline__ double pblock_max(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = (threadIdx.x < 32 && l < PW) ? sh[l] : 0.0;
  if (threadIdx.x < 32) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
    if (l == 0) sh[0] = t;
  }
  __syncthreads();
  t = sh[0];
  __syncthreads();
  return t;
}
__device__ __forceinline__ double slot_max(const double* bpart, int slot, double* sh) {
  double t = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += PT) t = fmax(t, __ldcg(bpart + slot * gridDim.x + i));
  return pblock_max(t, sh);
}

// Bucket holding the need-th (1-based) count of a global histogram.  All
// threads return (digit, count strictly below).  Redundant in every CTA.
__device__ void p_find_bucket(const unsigned int* gh, long long need, unsigned int* sh_u,
                              long long* sh_l, int& digit, long long& below) {
  constexpr int PER = NBINS / PT;           // 4 bins per thread
  unsigned int loc[PER];
  long long mine = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    loc[i] = gh[threadIdx.x * PER + i];      // smem or global (after a grid barrier)
    mine += loc[i];
  }
  // inclusive warp scan, then scan of the warp totals
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long inc = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) sh_l[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    long long t = sh_l[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long u = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += u;
    }
    sh_l[lane] = t;                         // inclusive warp-total scan
  }
  __syncthreads();
  const long long base = inc - mine + (wid > 0 ? sh_l[wid - 1] : 0);
  if (base < need && need <= base + mine) {
    long long c = base;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      if (c + loc[i] >= need) {
        sh_u[0] = threadIdx.x * PER + i;
        sh_l[32] = c;
        break;
      }
      c += loc[i];
    }
  }
  __syncthreads();
  digit = (int)sh_u[0];
  below = sh_l[32];
  __syncthreads();
}

// Per-side selection state kept in shared memory (identical in all CTAs).
struct PSel {
  unsigned long long prefix, tau;
  long long below, target, npos, tie;
  int mode, slow;
  double thr;                  // greedy: select eps >= thr = eta * max eps
};

// GDBEK threshold set {i : eps_i >= eta * max eps} (>= per SPEC S:303).
__device__ __forceinline__ void p_sel_greedy(PSel* ps, double emax, double eta) {
  if (threadIdx.x == 0) {
    ps->mode = emax > 0.0 ? SEL_GREEDY : SEL_NONE;
    ps->thr = eta * emax;
    ps->target = -1;
    ps->slow = 0;
  }
  __syncthreads();
}

// Level-1 finalize: block size clamp and first bucket.
__device__ void p_sel_level1(PSel* ps, const unsigned int* gh, long long N, long long kblock,
                             unsigned int* sh_u, long long* sh_l) {
  const long long never = (long long)__ldcg(gh + (NBINS - 1));
  const long long npos = N - never;
  const long long target = kblock < npos ? kblock : npos;
  int mode = target == 0 ? SEL_NONE : (target == npos ? SEL_ALL : SEL_PENDING);
  int digit = 0;
  long long below = 0;
  if (mode == SEL_PENDING) p_find_bucket(gh, target, sh_u, sh_l, digit, below);
  if (threadIdx.x == 0) {
    ps->npos = npos; ps->target = target; ps->mode = mode; ps->slow = 0;
    ps->prefix = (unsigned long long)digit; ps->below = below;
    ps->tau = (mode == SEL_ALL) ? KEY_NEVER - 1ull : 0ull;
    ps->tie = (mode == SEL_ALL) ? 0x7FFFFFFFFFFFFFFFll : -1;
  }
  __syncthreads();
}

// Level 2/3 scan over the keys of the current bucket (grid-stride, all CTAs).
template <int LEVEL>
__device__ void p_sel_scan(const PSel* ps, const unsigned long long* __restrict__ keys, long long N,
                           long long idx_base, unsigned int* gh, Cand* cand, unsigned int* ncand,
                           unsigned int* h) {
  if (ps->mode != SEL_PENDING) return;
  for (int i = threadIdx.x; i < NBINS; i += PT) h[i] = 0u;
  __syncthreads();
  constexpr int SF = (LEVEL == 2) ? L1_SHIFT : L2_SHIFT;
  constexpr int SD = (LEVEL == 2) ? L2_SHIFT : L3_SHIFT;
  const unsigned long long pre = ps->prefix;
  const long long stride = (long long)gridDim.x * PT;
  constexpr int VU = RG_SCAN_VU;                // keys in flight per thread
  for (long long i0 = (long long)blockIdx.x * PT + threadIdx.x; i0 < N; i0 += VU * stride) {
    unsigned long long kv[VU];
#pragma unroll
    for (int e = 0; e < VU; ++e) {
      const long long i = i0 + e * stride;
      kv[e] = i < N ? keys[i] : KEY_NEVER;
    }
#pragma unroll
    for (int e = 0; e < VU; ++e) {
      const unsigned long long key = kv[e];
      if (i0 + e * stride < N && (key >> SF) == pre) {
        atomicAdd(&h[(key >> SD) & 0xFFFull], 1u);
        if (LEVEL == 3) {
          const unsigned int slot = atomicAdd(ncand, 1u);
          if (slot < CAND_CAP) cand[slot] = Cand{key, idx_base + i0 + e * stride};
        }
      }
    }
  }
  __syncthreads();
  flush_hist<PT>(h, gh, NBINS);
}

__device__ void p_sel_level2(PSel* ps, const unsigned int* gh, unsigned int* sh_u, long long* sh_l) {
  if (ps->mode != SEL_PENDING) return;
  int digit;
  long long below;
  p_find_bucket(gh, ps->target - ps->below, sh_u, sh_l, digit, below);
  if (threadIdx.x == 0) {
    ps->prefix = (ps->prefix << 12) | (unsigned long long)digit;
    ps->below += below;
  }
  __syncthreads();
}

// Slow path (candidate overflow): resolve the rest of the key and the tie index
// by radix levels over ALL keys, in this CTA alone (redundantly in every CTA).
__device__ void p_sel_slow(PSel* ps, const unsigned long long* __restrict__ keys, long long N,
                           long long idx_base, unsigned int* h, unsigned int* sh_u, long long* sh_l) {
  const int shifts[6] = {16, 4, 0, 20, 8, 0};
  const unsigned long long masks[6] = {0xFFF, 0xFFF, 0xF, 0xFFF, 0xFFF, 0xFF};
  unsigned long long kpre = ps->prefix;   // key >> 28
  int kshift = L3_SHIFT;
  unsigned long long ipre = 0;
  int ishift = 32;
  long long below = ps->below;
  const long long target = ps->target;
  for (int lv = 0; lv < 6; ++lv) {
    for (int q = threadIdx.x; q < NBINS; q += PT) h[q] = 0u;
    __syncthreads();
    const bool on_idx = lv >= 3;
    for (long long i = threadIdx.x; i < N; i += PT) {
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
    // bucket search on the smem histogram (copy through the helper's global-read path)
    constexpr int PER = NBINS / PT;
    long long mine = 0;
    for (int i = 0; i < PER; ++i) mine += h[threadIdx.x * PER + i];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    long long inc = mine;
    for (int o = 1; o < 32; o <<= 1) {
      const long long t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) sh_l[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      long long t = sh_l[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const long long u = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += u;
      }
      sh_l[lane] = t;
    }
    __syncthreads();
    const long long need = target - below;
    const long long base = inc - mine + (wid > 0 ? sh_l[wid - 1] : 0);
    if (base < need && need <= base + mine) {
      long long c = base;
      for (int i = 0; i < PER; ++i) {
        if (c + h[threadIdx.x * PER + i] >= need) {
          sh_u[0] = threadIdx.x * PER + i;
          sh_l[32] = c;
          break;
        }
        c += h[threadIdx.x * PER + i];
      }
    }
    __syncthreads();
    const unsigned long long dg = sh_u[0];
    below += sh_l[32];
    const int bits = (masks[lv] == 0xFFF) ? 12 : (masks[lv] == 0xFF ? 8 : 4);
    if (!on_idx) {
      kpre = (kpre << bits) | dg;
      kshift = shifts[lv];
    } else {
      ipre = (ishift >= 32) ? dg : ((ipre << bits) | dg);
      ishift = shifts[lv];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ps->tau = kpre;
    ps->tie = (long long)ipre;
    ps->mode = SEL_THRESH;
    ps->slow |= 1;               // counted by the kernel (rgdbek_selection_stats)
  }
  __syncthreads();
}

// Level-3 finalize + exact rank of the survivors -> (tau, tie).
__device__ void p_sel_level3(PSel* ps, const unsigned int* gh, const Cand* cand,
                             const unsigned int* ncand, const unsigned long long* keys, long long N,
                             long long idx_base, unsigned int* h, unsigned int* sh_u,
                             long long* sh_l) {
  if (ps->mode != SEL_PENDING) return;
  int digit;
  long long below;
  p_find_bucket(gh, ps->target - ps->below, sh_u, sh_l, digit, below);
  __shared__ int nf;
  if (threadIdx.x == 0) {
    ps->prefix = (ps->prefix << 12) | (unsigned long long)digit;
    ps->below += below;
    nf = 0;
  }
  __syncthreads();
  Cand* fc = reinterpret_cast<Cand*>(h);        // 16 KB = FINAL_CAP survivors
  const unsigned int nc = __ldcg(ncand);
  const unsigned long long pre3 = ps->prefix;
  if (nc <= CAND_CAP) {
    for (unsigned int c = threadIdx.x; c < nc; c += PT) {
      const Cand e = cand[c];
      if ((e.key >> L3_SHIFT) == pre3) {
        const int sl = atomicAdd(&nf, 1);
        if (sl < FINAL_CAP) fc[sl] = e;
      }
    }
  }
  __syncthreads();
  if (nc > CAND_CAP || nf > FINAL_CAP) {
    p_sel_slow(ps, keys, N, idx_base, h, sh_u, sh_l);
    return;
  }
  const long long need = ps->target - ps->below;
  for (int e = threadIdx.x; e < nf; e += PT) {
    const Cand me = fc[e];
    long long rank = 0;
    for (int f = 0; f < nf; ++f) {
      const Cand o = fc[f];
      rank += (o.key < me.key) || (o.key == me.key && o.idx < me.idx);
    }
    if (rank == need - 1) { ps->tau = me.key; ps->tie = me.idx; }
  }
  __syncthreads();
  if (threadIdx.x == 0) ps->mode = SEL_THRESH;
  __syncthreads();
}

// Local selection with the level-1 bucket's keys gathered into shared memory
// once (when they fit): levels 2, 3 and the survivor rank then run on the smem
// list instead of two more passes over all N keys in global memory.
#ifndef RG_LCAND_CAP
#define RG_LCAND_CAP 4096
#endif
constexpr int LCAND_CAP = RG_LCAND_CAP;
__device__ bool p_sel_local_smem(PSel* ps, const unsigned long long* __restrict__ keys,
                                 long long N, long long idx_base, const unsigned int* gh1,
                                 unsigned int* h, unsigned int* sh_u, long long* sh_l,
                                 Cand* cl, Cand* fc, unsigned long long* pt = nullptr) {
  if (ps->mode != SEL_PENDING) return true;
  // optional sub-phase timers (RGDBEK_PHASE_TIMING): pt[0..3] += gather, level 2,
  // level 3, final rank — read by thread 0 of CTA 0 only
  const bool tim = pt && blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long t0 = tim ? gtimer() : 0ull;
#define SUBT(i) if (tim) { const unsigned long long t1 = gtimer(); pt[i] += t1 - t0; t0 = t1; }
  const unsigned int c1 = __ldcg(gh1 + ps->prefix);
  if (c1 > (unsigned int)LCAND_CAP) return false;
  __shared__ int nc, nf;
  if (threadIdx.x == 0) { nc = 0; nf = 0; }
  __syncthreads();
  const unsigned long long pre1 = ps->prefix;
  for (long long i = threadIdx.x; i < N; i += PT) {
    const unsigned long long key = keys[i];
    if ((key >> L1_SHIFT) == pre1) {
      const int s = atomicAdd(&nc, 1);
      if (s < LCAND_CAP) cl[s] = Cand{key, idx_base + i};
    }
  }
  __syncthreads();
  SUBT(0);
  const int cnt = nc < LCAND_CAP ? nc : LCAND_CAP;
  for (int lv = 2; lv <= 3; ++lv) {
    const int sf = lv == 2 ? L1_SHIFT : L2_SHIFT;
    const int sd = lv == 2 ? L2_SHIFT : L3_SHIFT;
    for (int i = threadIdx.x; i < NBINS; i += PT) h[i] = 0u;
    __syncthreads();
    const unsigned long long pre = ps->prefix;
    for (int e = threadIdx.x; e < cnt; e += PT) {
      const unsigned long long key = cl[e].key;
      if ((key >> sf) == pre) atomicAdd(&h[(key >> sd) & 0xFFFull], 1u);
    }
    __syncthreads();
    int digit;
    long long below;
    p_find_bucket(h, ps->target - ps->below, sh_u, sh_l, digit, below);
    if (threadIdx.x == 0) {
      ps->prefix = (ps->prefix << 12) | (unsigned long long)digit;
      ps->below += below;
    }
    __syncthreads();
    SUBT(lv - 1);
  }
  const unsigned long long pre3 = ps->prefix;
  for (int e = threadIdx.x; e < cnt; e += PT) {
    const Cand c = cl[e];
    if ((c.key >> L3_SHIFT) == pre3) {
      const int s = atomicAdd(&nf, 1);
      if (s < FINAL_CAP) fc[s] = c;
    }
  }
  __syncthreads();
  const int nfin = nf;
  if (nfin > FINAL_CAP) {
    __syncthreads();
    p_sel_slow(ps, keys, N, idx_base, h, sh_u, sh_l);
    return true;
  }
  const long long need = ps->target - ps->below;
  for (int e = threadIdx.x; e < nfin; e += PT) {
    const Cand me = fc[e];
    long long rank = 0;
    for (int f = 0; f < nfin; ++f) {
      const Cand o = fc[f];
      rank += (o.key < me.key) || (o.key == me.key && o.idx < me.idx);
    }
    if (rank == need - 1) { ps->tau = me.key; ps->tie = me.idx; }
  }
  __syncthreads();
  if (threadIdx.x == 0) ps->mode = SEL_THRESH;
  __syncthreads();
  SUBT(3);
#undef SUBT
  return true;
}

// Small selections (N <= LOCAL_SEL_MAX): after the grid-wide level-1 bucket,
// every CTA resolves levels 2, 3 and the survivors by itself from all N keys
// (identical results everywhere), saving two grid barriers.
__device__ void p_sel_local(PSel* ps, const unsigned long long* __restrict__ keys, long long N,
                            long long idx_base, unsigned int* h, unsigned int* sh_u,
                            long long* sh_l) {
  if (ps->mode != SEL_PENDING) return;
  __shared__ int nfl;
  for (int lv = 2; lv <= 3; ++lv) {
    const int sf = lv == 2 ? L1_SHIFT : L2_SHIFT;
    const int sd = lv == 2 ? L2_SHIFT : L3_SHIFT;
    for (int i = threadIdx.x; i < NBINS; i += PT) h[i] = 0u;
    __syncthreads();
    const unsigned long long pre = ps->prefix;
    for (long long i = threadIdx.x; i < N; i += PT) {
      const unsigned long long key = keys[i];
      if ((key >> sf) == pre) atomicAdd(&h[(key >> sd) & 0xFFFull], 1u);
    }
    __syncthreads();
    int digit;
    long long below;
    p_find_bucket(h, ps->target - ps->below, sh_u, sh_l, digit, below);
    if (threadIdx.x == 0) {
      ps->prefix = (ps->prefix << 12) | (unsigned long long)digit;
      ps->below += below;
      nfl = 0;
    }
    __syncthreads();
  }
  Cand* fc = reinterpret_cast<Cand*>(h);
  const unsigned long long pre3 = ps->prefix;
  for (long long i = threadIdx.x; i < N; i += PT) {
    const unsigned long long key = keys[i];
    if ((key >> L3_SHIFT) == pre3) {
      const int sl = atomicAdd(&nfl, 1);
      if (sl < FINAL_CAP) fc[sl] = Cand{key, idx_base + i};
    }
  }
  __syncthreads();
  const int nf = nfl;
  if (nf > FINAL_CAP) {
    __syncthreads();
    p_sel_slow(ps, keys, N, idx_base, h, sh_u, sh_l);
    return;
  }
  const long long need = ps->target - ps->below;
  for (int e = threadIdx.x; e < nf; e += PT) {
    const Cand me = fc[e];
    long long rank = 0;
    for (int f = 0; f < nf; ++f) {
      const Cand o = fc[f];
      rank += (o.key < me.key) || (o.key == me.key && o.idx < me.idx);
    }
    if (rank == need - 1) { ps->tau = me.key; ps->tie = me.idx; }
  }
  __syncthreads();
  if (threadIdx.x == 0) ps->mode = SEL_THRESH;
  __syncthreads();
}

__device__ __forceinline__ bool p_selected(const PSel* ps, unsigned long long key, long long gidx) {
  if (ps->mode == SEL_THRESH) return key < ps->tau || (key == ps->tau && gidx <= ps->tie);
  if (ps->mode == SEL_GREEDY) return key != KEY_NEVER && __longlong_as_double((long long)key) >= ps->thr;
  if (ps->mode == SEL_ALL) return key != KEY_NEVER;
  return false;
}

// Block capture (rgdbek_set_capture; off in production): out[i] = [index i selected] for
// i = i0, i0 + stride, ... < i1.  Out of line, so its registers do not weigh on the
// callers' hot loops.
__device__ __noinline__ void p_capture(unsigned char* out, const PSel* ps,
                                       const unsigned long long* keys, long long base, int i0,
                                       int i1, int stride) {
  for (int i = i0; i < i1; i += stride) out[i] = p_selected(ps, keys[i], base + i) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// Dense pass T for this CTA's contiguous row range, all columns (column tiles
// of 2*PT): part[cta][0][j] = sum_i A_ij z_i, part[cta][1][j] = sum_i A_ij xi_i.
// ---------------------------------------------------------------------------

template <int KP>
__device__ void p_dense_passT_rows(const PArgs& a, int pending, double* zs, const double* in1,
                                   const double* in2);

// Optional fused row mask (psr != nullptr, RG_FUSE_XI): xi_i = r_i if row i is in
// the row block J (psr) else 0 is formed while the rows are staged, and this
// CTA's ||xi||^2, |J| and hash partials are returned (each row is staged by
// exactly one CTA, counted at the first column tile only).
__device__ void p_dense_passT(const PArgs& a, int pending, double* zs,
                              const double* in1 = nullptr, const double* in2 = nullptr,
                              const PSel* psr = nullptr, double* Xp = nullptr,
                              long long* cntp = nullptr, unsigned long long* hsp = nullptr) {
  if (!in1) in1 = a.z;
  if (!in2) in2 = a.xi;
  const int ntiles = (a.n + 2 * PT - 1) / (2 * PT);
  if (a.pt_rows) {                    // exact mode only (no fused row mask there)
    switch (ntiles) {
      case 1: p_dense_passT_rows<1>(a, pending, zs, in1, in2); return;
      case 2: p_dense_passT_rows<2>(a, pending, zs, in1, in2); return;
      case 3: p_dense_passT_rows<3>(a, pending, zs, in1, in2); return;
      default: break;
    }
  }
  const int G = gridDim.x, bb = blockIdx.x;
  const int rb = (int)((long long)a.m_loc * bb / G), re = (int)((long long)a.m_loc * (bb + 1) / G);
  double* out = a.part + (long long)bb * 2 * a.n;
  for (int t = 0; t < ntiles; ++t) {
    const int c = t * 2 * PT + 2 * threadIdx.x;
    double s0 = 0.0, s1 = 0.0, v0 = 0.0, v1 = 0.0;
    for (int rc = rb; rc < re; rc += ZCH) {
      const int rows = min(ZCH, re - rc);
      __syncthreads();
      for (int i = threadIdx.x; i < rows; i += PT) {
        zs[i] = in1[rc + i];
        if (psr) {
          double xv = 0.0;
          if (pending) {
            const long long gi = a.row0 + rc + i;
            if (p_selected(psr, a.keys_m[rc + i], gi)) {
              xv = a.r[rc + i];
              if (t == 0) { *Xp += xv * xv; *cntp += 1; *hsp += splitmix64((unsigned long long)gi); }
            }
          }
          zs[ZCH + i] = xv;
        } else {
          zs[ZCH + i] = pending ? in2[rc + i] : 0.0;
        }
      }
      __syncthreads();
      const double* p = a.A + (long long)rc * a.lda + c;
      if (c + 1 < a.n) {
#pragma unroll 8
        for (int i = 0; i < rows; ++i) {
          const double2 av = ld_stream2(p + (long long)i * a.lda);
          const double zi = zs[i], xv = zs[ZCH + i];
          s0 = fma(av.x, zi, s0);
          s1 = fma(av.y, zi, s1);
          v0 = fma(av.x, xv, v0);
          v1 = fma(av.y, xv, v1);
        }
      } else if (c < a.n) {
        for (int i = 0; i < rows; ++i) {
          const double av = ld_stream(p + (long long)i * a.lda);
          s0 = fma(av, zs[i], s0);
          v0 = fma(av, zs[ZCH + i], v0);
        }
      }
    }
    if (c + 1 < a.n) {
      out[c] = s0; out[c + 1] = s1;
      out[a.n + c] = v0; out[a.n + c + 1] = v1;
    } else if (c < a.n) {
      out[c] = s0;
      out[a.n + c] = v0;
    }
  }
}

// Dense pass T in ONE sweep over the CTA's rows: thread t accumulates the column
// pairs 2t + 2*PT*k (k < KP) in registers (no per-tile re-staging of z / xi and
// no sweep with a partly idle block).
template <int KP>
__device__ void p_dense_passT_rows(const PArgs& a, int pending, double* zs, const double* in1,
                                   const double* in2) {
  const int G = gridDim.x, bb = blockIdx.x;
  const int rb = (int)((long long)a.m_loc * bb / G), re = (int)((long long)a.m_loc * (bb + 1) / G);
  const int n = a.n;
  double* out = a.part + (long long)bb * 2 * n;
  double acc[KP][4];
#pragma unroll
  for (int k = 0; k < KP; ++k) { acc[k][0] = acc[k][1] = acc[k][2] = acc[k][3] = 0.0; }
  for (int rc = rb; rc < re; rc += ZCH) {
    const int rows = min(ZCH, re - rc);
    __syncthreads();
    for (int i = threadIdx.x; i < rows; i += PT) {
      zs[i] = in1[rc + i];
      zs[ZCH + i] = pending ? in2[rc + i] : 0.0;
    }
    __syncthreads();
    const double* p = a.A + (long long)rc * a.lda + 2 * threadIdx.x;
#pragma unroll 2
    for (int i = 0; i < rows; ++i) {
      const double zi = zs[i], xv = zs[ZCH + i];
      const double* pr = p + (long long)i * a.lda;
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const int c = 2 * threadIdx.x + 2 * PT * k;
        if (c + 1 < n) {
          const double2 av = ld_stream2(pr + 2 * PT * k);
          acc[k][0] = fma(av.x, zi, acc[k][0]);
          acc[k][1] = fma(av.y, zi, acc[k][1]);
          acc[k][2] = fma(av.x, xv, acc[k][2]);
          acc[k][3] = fma(av.y, xv, acc[k][3]);
        } else if (c < n) {
          const double av = ld_stream(pr + 2 * PT * k);
          acc[k][0] = fma(av, zi, acc[k][0]);
          acc[k][2] = fma(av, xv, acc[k][2]);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    const int c = 2 * threadIdx.x + 2 * PT * k;
    if (c + 1 < n) {
      out[c] = acc[k][0]; out[c + 1] = acc[k][1];
      out[n + c] = acc[k][2]; out[n + c + 1] = acc[k][3];
    } else if (c < n) {
      out[c] = acc[k][0];
      out[n + c] = acc[k][2];
    }
  }
}

// ---------------------------------------------------------------------------
// Dense pass N for this CTA's rows, in batches of PN_RB rows: warp-units of
// (1 row) x (column chunk of CH), partials in smem, summed in chunk order.
// Returns this thread's contributions to W and ||b - Ax||^2.
// ---------------------------------------------------------------------------
__device__ void p_dense_passN(const PArgs& a, double* np, double& Wp, double& Yp,
                              const double* in1 = nullptr, const double* in2 = nullptr,
                              double* out1 = nullptr, double* out2 = nullptr,
                              const double* bvec = nullptr, bool use_b = true) {
  if (!in1) in1 = a.zeta;
  if (!in2) in2 = a.x;
  if (!out1) out1 = a.w;
  if (!out2) out2 = a.ax;
  if (!bvec && use_b) bvec = a.b;
  const int G = gridDim.x, bb = blockIdx.x;
  const int rb = (int)((long long)a.m_loc * bb / G), re = (int)((long long)a.m_loc * (bb + 1) / G);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int Q = a.Q, CH = a.CH, n = a.n;
  // stage the two input vectors in shared memory (LDS instead of L1 loads in
  // the streaming loop, so the only long-latency loads in flight are A's)
  const double* v1s = in1;
  const double* v2s = in2;
  if (a.pn_smem) {
    double* zs = np + PN_RB * PN_QMAX * 2;
    for (int c = threadIdx.x * 2; c < n; c += 2 * PT) {
      if (c + 1 < n) {
        *reinterpret_cast<double2*>(zs + c) = *reinterpret_cast<const double2*>(in1 + c);
        *reinterpret_cast<double2*>(zs + a.lda + c) = *reinterpret_cast<const double2*>(in2 + c);
      } else {
        zs[c] = in1[c];
        zs[a.lda + c] = in2[c];
      }
    }
    __syncthreads();
    v1s = zs;
    v2s = zs + a.lda;
  }
  const int nbatch = (re - rb + PN_RB - 1) / PN_RB;             // evenly sized batches
  const int per = nbatch ? (re - rb + nbatch - 1) / nbatch : 0;
  // rows bottom-up (batches and row pairs in reverse): pass T just streamed this
  // CTA's rows top-down, so the rows it read last are still in L2 when pass N
  // starts; the next pass T (top-down) then meets the rows pass N read last
  for (int bt = nbatch - 1; bt >= 0; --bt) {
    const int r0 = rb + (RG_REV_N ? bt : nbatch - 1 - bt) * per;
    const int rows = min(per, re - r0);
    const int npairs = (rows + 1) >> 1;
    const int units = npairs * Q;                                // 2 rows x 1 chunk per unit
    for (int u = wid; u < units; u += PW) {
      const int up = u / Q, q = u - up * Q;
      const int rp = RG_REV_N ? npairs - 1 - up : up;
      const int rr = 2 * rp;
      const bool two = rr + 1 < rows;
      const int c0 = q * CH, c1 = min(n, c0 + CH);
      const int c1e = c0 + ((c1 - c0) & ~1);
      const double* a0 = a.A + (long long)(r0 + rr) * a.lda;
      const double* a1 = two ? a0 + a.lda : a0;
      double w0 = 0.0, x0 = 0.0, w1 = 0.0, x1 = 0.0;
      int c = c0 + lane * 2;
      // batches of 4 column groups: all 8 A loads issued before any use
      for (; c + 192 < c1e; c += 256) {
        double2 va[4], vb[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          va[g] = ld_stream2(a0 + c + 64 * g);
          vb[g] = two ? ld_stream2(a1 + c + 64 * g) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const double2 zc = *reinterpret_cast<const double2*>(v1s + c + 64 * g);
          const double2 xc = *reinterpret_cast<const double2*>(v2s + c + 64 * g);
          w0 = fma(va[g].x, zc.x, w0); w0 = fma(va[g].y, zc.y, w0);
          x0 = fma(va[g].x, xc.x, x0); x0 = fma(va[g].y, xc.y, x0);
          w1 = fma(vb[g].x, zc.x, w1); w1 = fma(vb[g].y, zc.y, w1);
          x1 = fma(vb[g].x, xc.x, x1); x1 = fma(vb[g].y, xc.y, x1);
        }
      }
      for (; c < c1e; c += 64) {
        const double2 zc = *reinterpret_cast<const double2*>(v1s + c);
        const double2 xc = *reinterpret_cast<const double2*>(v2s + c);
        const double2 v0 = ld_stream2(a0 + c);
        const double2 v1 = two ? ld_stream2(a1 + c) : make_double2(0.0, 0.0);
        w0 = fma(v0.x, zc.x, w0); w0 = fma(v0.y, zc.y, w0);
        x0 = fma(v0.x, xc.x, x0); x0 = fma(v0.y, xc.y, x0);
        w1 = fma(v1.x, zc.x, w1); w1 = fma(v1.y, zc.y, w1);
        x1 = fma(v1.x, xc.x, x1); x1 = fma(v1.y, xc.y, x1);
      }
      if (c1e < c1 && lane == 0) {
        const double v0 = ld_stream(a0 + c1e);
        w0 = fma(v0, in1[c1e], w0);
        x0 = fma(v0, in2[c1e], x0);
        if (two) {
          const double v1 = ld_stream(a1 + c1e);
          w1 = fma(v1, in1[c1e], w1);
          x1 = fma(v1, in2[c1e], x1);
        }
      }
      w0 = warp_sum(w0); x0 = warp_sum(x0);
      w1 = warp_sum(w1); x1 = warp_sum(x1);
      if (lane == 0) {
        np[(rr * PN_QMAX + q) * 2] = w0; np[(rr * PN_QMAX + q) * 2 + 1] = x0;
        if (two) { np[((rr + 1) * PN_QMAX + q) * 2] = w1; np[((rr + 1) * PN_QMAX + q) * 2 + 1] = x1; }
      }
    }
    __syncthreads();
    if (threadIdx.x < rows) {
      const int rr = threadIdx.x, i = r0 + rr;
      double tw = 0.0, tx = 0.0;
      for (int q = 0; q < Q; ++q) { tw += np[(rr * PN_QMAX + q) * 2]; tx += np[(rr * PN_QMAX + q) * 2 + 1]; }
      out1[i] = tw;
      out2[i] = tx;
      Wp += tw * tw;
      if (bvec) {
        const double y = bvec[i] - tx;
        Yp += y * y;
      } else {
        Yp += tx * tx;
      }
    }
    __syncthreads();
  }
}

// CSR / CSC dual SpMV over all CTAs' warps (VEC lanes per row).
template <int VEC>
__device__ void p_csr_dual(const long long* __restrict__ ptr, const int* __restrict__ idx,
                           const double* __restrict__ val, int nrows,
                           const double* __restrict__ in1, const double* __restrict__ in2,
                           int use2, const double* __restrict__ b, double* __restrict__ out1,
                           double* __restrict__ out2, double& Wp, double& Yp) {
  constexpr int SPW = 32 / VEC;
  const int lane = threadIdx.x & (VEC - 1);
  const int sub = (threadIdx.x & 31) / VEC;
  const int gw = (blockIdx.x * PT + threadIdx.x) >> 5;
  const int nw = (gridDim.x * PT) >> 5;
  for (int base = gw * SPW; base < nrows; base += nw * SPW) {
    const int row = base + sub;
    const bool valid = row < nrows;
    double a1 = 0.0, a2 = 0.0;
    if (valid) {
      const long long p0 = ptr[row], p1 = ptr[row + 1];
      for (long long p = p0 + lane; p < p1; p += VEC) {
        const double av = ld_stream(val + p);
        const int c = __ldg(idx + p);
        a1 = fma(av, __ldg(in1 + c), a1);
        if (use2) a2 = fma(av, __ldg(in2 + c), a2);
      }
    }
#pragma unroll
    for (int o = VEC / 2; o > 0; o >>= 1) {
      a1 += __shfl_xor_sync(0xffffffffu, a1, o, VEC);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o, VEC);
    }
    if (lane == 0 && valid) {
      out1[row] = a1;
      out2[row] = a2;
      if (b) {
        const double y = b[row] - a2;
        Wp += a1 * a1;
        Yp += y * y;
      }
    }
  }
}

template <int VEC>
__device__ __forceinline__ void p_csr_dispatch_dummy() {}

__device__ void p_csr(int vec, const long long* ptr, const int* idx, const double* val, int nrows,
                      const double* in1, const double* in2, int use2, const double* b,
                      double* o1, double* o2, double& Wp, double& Yp) {
  switch (vec) {
    case 2: p_csr_dual<2>(ptr, idx, val, nrows, in1, in2, use2, b, o1, o2, Wp, Yp); break;
    case 4: p_csr_dual<4>(ptr, idx, val, nrows, in1, in2, use2, b, o1, o2, Wp, Yp); break;
    case 8: p_csr_dual<8>(ptr, idx, val, nrows, in1, in2, use2, b, o1, o2, Wp, Yp); break;
    case 16: p_csr_dual<16>(ptr, idx, val, nrows, in1, in2, use2, b, o1, o2, Wp, Yp); break;
    default: p_csr_dual<32>(ptr, idx, val, nrows, in1, in2, use2, b, o1, o2, Wp, Yp); break;
  }
}

// Zero this CTA's slice of one side's histograms / accumulators.
__device__ void p_zero_side(const PArgs& a, int side) {
  unsigned int* h = a.hist + side * 3 * NBINS;
  for (int i = blockIdx.x * PT + threadIdx.x; i < 3 * NBINS; i += gridDim.x * PT) h[i] = 0u;
  unsigned int* hs = a.hist + (6 + side) * NBINS;               // the speculative level 2
  for (int i = blockIdx.x * PT + threadIdx.x; i < NBINS; i += gridDim.x * PT) hs[i] = 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.acc[2 * side] = 0ull;
    a.acc[2 * side + 1] = 0ull;
    a.ncand[side] = 0u;
  }
}


// ---------------------------------------------------------------------------
// The persistent kernel.
// ---------------------------------------------------------------------------
// DENSE selects the pass kernels at compile time: each instantiation carries
// only its own pass code, so the register allocation (64 per thread at 1024
// threads) is not shared between the dense and the sparse paths.
template <bool DENSE, bool LAZY = false>
__global__ void __launch_bounds__(PT, 1) k_persistent(PArgs a) {
  __shared__ __align__(16) unsigned int h[NBINS];
  __shared__ __align__(8) unsigned long long tbar[(PT / TG) * TRING];
  __shared__ double sh[PW];
  __shared__ unsigned int sh_u[4];
  __shared__ long long sh_l[40];
  __shared__ PSel ps;
  __shared__ double lzs[4][LZ_MAX];      // Algorithm 2: per-process V, X, Z, W
  extern __shared__ __align__(16) double dyn[];
  TileRing tring{tbar + (threadIdx.x / TG) * TRING, 0u};
  if (!DENSE) tile_rings_init(tbar);
  Scal* st = a.st;
  TraceRec* tr = a.tr;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  const int G = gridDim.x;
  double* bp = a.bpart;
  // ---- call state (identical in every CTA) ----
  long long k = st->k;
  const long long k_begin = st->k_begin, k_end = st->k_end;
  const double tol = st->tol;
  const int stop_mode = st->stop_mode, has_ref = st->has_ref;
  const unsigned long long seed = st->seed;
  const double bnorm2 = st->bnorm2, xsnorm2 = st->xsnorm2;
  const long long kc = st->kc, kr = st->kr;
  int pending = st->pending;
  double X = st->X;
  long long kp_prev = st->kp_prev, kpp_prev = st->kpp_prev;
  const int n = a.n, m_loc = a.m_loc;
  unsigned int* hn = a.hist;                    // n-side levels 1..3
  unsigned int* hm = a.hist + 3 * NBINS;        // m-side levels 1..3
  Cand* cn = a.cand;
  Cand* cm = a.cand + CAND_CAP;
  unsigned long long t_last = 0;
  unsigned int bgen = 0;
  int predJ = -1;                               // speculative row level 2 (sparse, see P8)
  int predU = -1;                               // speculative column level 2 (sparse, pass T)
  if (threadIdx.x == 0) bgen = ld_acquire_u32(&a.bar->gen);
#define PH(i)                                                        \
  if (a.ptime && lead) {                                             \
    const unsigned long long t_ = gtimer();                          \
    if (t_last) a.ptime[i] += t_ - t_last;                           \
    t_last = t_;                                                     \
  }
  PH(0);

  for (;;) {
    // ===== P1: pass T  (s_k = A^T z_k, v_{k-1} = A^T xi_{k-1}) =====
    // Sparse: the column scores, keys, level-1 histogram and V partial are fused
    // into the tile epilogue, so the separate P2 phase (and its barrier) vanishes.
    double Vp = 0.0, Emax = 0.0;
    if constexpr (DENSE) {
      if constexpr (RG_FUSE_XI) {
        // pass T forms xi_{k-1} from r and the row selection still in `ps`, and
        // publishes ||xi||^2, |J| and hash partials (replaces the P11 sweep)
        double Xp = 0.0;
        long long cnt = 0;
        unsigned long long hs = 0ull;
        if (a.capJ && pending)                  // J_{k-1} from the row selection still in ps
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
      } else {
        p_dense_passT(a, pending, dyn);
      }
      grid_sync(a.bar, bgen);
      PH(1);
      if constexpr (RG_FUSE_XI) {
        // the row step k-1's |J|, hash and X (read by every CTA before the P2
        // barrier; the m-side counters are zeroed after it, in P3)
        if (pending) {
          X = slot_sum(bp, SL_X, sh);
          const long long kppf = (long long)__ldcg(&a.acc[2]);
          const unsigned long long hashJ = __ldcg(&a.acc[3]);
          if (lead) {
            if (!a.greedy && !LAZY && kppf != (ps.mode == SEL_NONE ? 0 : ps.target)) st->error |= 2;
            if (TraceRec* t = trace_at(tr, st, k - 1)) { t->kpp = kppf; t->hash_j = hashJ; t->X = X; }
          }
          kpp_prev = kppf;
        }
      } else {
        p_zero_side(a, 1);                      // m-side buffers: consumed in P9..P12
      }
      if constexpr (LAZY) {
        for (int i = blockIdx.x * PT + threadIdx.x; i < a.lzP * NBINS; i += G * PT) a.lz_hist[i] = 0u;
      }

      // ===== P2 (dense): s, v = sum of the CTA partials; V; keys; level-1 histogram =====
      for (int i = threadIdx.x; i < NBINS; i += PT) h[i] = 0u;
      __syncthreads();
      // CTA b owns columns [c0, c1); thread (c = tid % 64, g = tid / 64) sums the
      // partials p = g, g + 16, ... of column c0 + chunk + c (coalesced across c),
      // then the 16 group sums are added in group order (deterministic) and one
      // thread per column makes its key — all columns of a CTA in parallel.
      if constexpr (LAZY) {
        // Algorithm 2: g_p = (A^(p))^T z^(p), v_p = (A^(p))^T xi^(p) from the CTA
        // partials of process p (its CTAs, in order); s = sum_p g_p (process order)
        const int cpb = (n + G - 1) / G;
        const int c0 = min(n, blockIdx.x * cpb), c1 = min(n, c0 + cpb);
        const int nc = c1 - c0, P = a.lzP, Gp = a.lzGp;
        double* gS = dyn;                         // [P][cpb]
        double* vS = dyn + P * cpb;               // [P][cpb]
        for (int it = threadIdx.x; it < P * nc; it += PT) {
          const int pp = it / nc, jl = it - pp * nc, j = c0 + jl;
          double gs = 0.0, vs = 0.0;
          for (int c = pp * Gp; c < (pp + 1) * Gp; ++c) {
            const double* q = a.part + (long long)c * 2 * n + j;
            gs += __ldcg(q);
            if (pending) vs += __ldcg(q + n);
          }
          gS[pp * cpb + jl] = gs;
          vS[pp * cpb + jl] = vs;
          a.lz_g[(long long)pp * n + j] = gs;
          a.lz_v[(long long)pp * n + j] = vs;
        }
        __syncthreads();
        for (int jl = threadIdx.x; jl < nc; jl += PT) {     // any number of columns per CTA
          const int j = c0 + jl;
          double ts = 0.0;
          for (int pp = 0; pp < P; ++pp) ts += gS[pp * cpb + jl];
          a.s[j] = ts;
          const double gm = a.gamma[j];
          const double eps = gm > 0.0 ? __ddiv_rn(__dmul_rn(ts, ts), gm) : 0.0;
          const unsigned long long key = sel_key(eps, (unsigned long long)j, k, 0u, seed, 0);
          a.keys_n[j] = key;
          atomicAdd(&h[key >> L1_SHIFT], 1u);
        }
        {                                         // V_p partial of this CTA's columns: warp p,
          const int w = threadIdx.x >> 5, l = threadIdx.x & 31;   // lanes strided, fixed tree
          if (w < P) {
            double t = 0.0;
            for (int jl = l; jl < nc; jl += 32) t += vS[w * cpb + jl] * vS[w * cpb + jl];
            t = warp_sum(t);
            if (l == 0) a.lz_slots[(long long)w * G + blockIdx.x] = t;
          }
        }
      } else {
        constexpr int CW = 64, NG = PT / CW;
        double* red = dyn;                        // [2][NG][CW]
        const int cpb = (n + G - 1) / G;
        const int c0 = min(n, blockIdx.x * cpb), c1 = min(n, c0 + cpb);
        const int cl = threadIdx.x % CW, g = threadIdx.x / CW;
        for (int cb = c0; cb < c1; cb += CW) {
          const int j = cb + cl;
          double sj = 0.0, vj = 0.0;
          if (j < c1) {
            double ps[10], pv[10];
#pragma unroll
            for (int t = 0; t < 10; ++t) {
              const int p = g + NG * t;
              const double* q = a.part + (long long)p * 2 * n + j;
              ps[t] = p < G ? __ldcg(q) : 0.0;
              pv[t] = (p < G && pending) ? __ldcg(q + n) : 0.0;
            }
#pragma unroll
            for (int t = 0; t < 10; ++t) { sj += ps[t]; vj += pv[t]; }
            for (int p = g + NG * 10; p < G; p += NG) {       // G > 160 (not on B200)
              const double* q = a.part + (long long)p * 2 * n + j;
              sj += __ldcg(q);
              if (pending) vj += __ldcg(q + n);
            }
          }
          red[g * CW + cl] = sj;
          red[(NG + g) * CW + cl] = vj;
          __syncthreads();
          if (g == 0 && j < c1) {
            double ts = 0.0, tv = 0.0;
#pragma unroll
            for (int q = 0; q < NG; ++q) { ts += red[q * CW + cl]; tv += red[(NG + q) * CW + cl]; }
            a.s[j] = ts;
            a.v[j] = tv;
            if (pending) Vp += tv * tv;
            const double gm = a.gamma[j];
            const double eps = gm > 0.0 ? __ddiv_rn(__dmul_rn(ts, ts), gm) : 0.0;
            Emax = fmax(Emax, eps);
            const unsigned long long key = sel_key(eps, (unsigned long long)j, k, 0u, seed, a.greedy);
            a.keys_n[j] = key;
            atomicAdd(&h[key >> L1_SHIFT], 1u);
          }
          __syncthreads();
        }
      }
      __syncthreads();
      PH(11);
      flush_hist<PT>(h, hn, NBINS);
      {
        const double vb = pblock_sum(Vp, sh);
        const double eb = pblock_max(Emax, sh);
        if (threadIdx.x == 0) { bp[SL_V * G + blockIdx.x] = vb; bp[SL_MAXN * G + blockIdx.x] = eb; }
      }
      PH(12);
      grid_sync(a.bar, bgen);
      PH(2);
    } else {
      for (int i = threadIdx.x; i < NBINS; i += PT) h[i] = 0u;
      __syncthreads();
      // speculative column level 2: the keys in the last iteration's level-1 bucket are
      // counted by their level-2 digit as they are made (global atomics; zeroed in P8)
      const ColKeyEpi ep{a.gamma, a.keys_n, h, k, seed, pending, a.greedy,
                         (RG_SPEC_U && predU >= 0) ? a.hist + 6 * NBINS : nullptr, predU};
      const int g = threadIdx.x / TG;
      csr_tiles(blockIdx.x * (PT / TG) + g, G * (PT / TG), threadIdx.x % TG, 1 + g,
                reinterpret_cast<TileSmem*>(dyn) + g, tring, a.cp, a.ri, a.rv, a.tilesT,
                a.tilepT, a.ntilesT,
                a.z, a.xi, pending, nullptr, a.s, a.v, Vp, Emax, &ep, 0, a.vecT);
      __syncthreads();
      flush_hist<PT>(h, hn, NBINS);
      {
        const double vb = pblock_sum(Vp, sh);
        const double eb = pblock_max(Emax, sh);
        if (threadIdx.x == 0) { bp[SL_V * G + blockIdx.x] = vb; bp[SL_MAXN * G + blockIdx.x] = eb; }
      }
      grid_sync(a.bar, bgen);
      PH(1);
      p_zero_side(a, 1);                        // m-side buffers: consumed in P9..P12
    }

    // ===== P3: V, alpha_x; level-1 bucket (U); level-2 scan =====
    if constexpr (DENSE && RG_FUSE_XI) p_zero_side(a, 1);   // every CTA read acc[2..3] before P2's barrier
    double V;
    if constexpr (LAZY) {
      // per-process V_p (over every CTA's columns) and X_p (the process's rows,
      // last iteration's P11 partials); V = sum_p V_p for the trace
      lz_sums(a.lz_slots, G, 0, G, a.lzP, lzs[0]);
      lz_sums(bp + SL_X * G, 0, a.lzGp, a.lzGp, a.lzP, lzs[1]);
      V = 0.0;
      for (int pp = 0; pp < a.lzP; ++pp) V += lzs[0][pp];
    } else {
      V = slot_sum(bp, SL_V, sh);
    }
    const int do_x = pending && kpp_prev > 0 && V > 0.0;
    const double alpha_x = do_x ? __ddiv_rn(X, V) : 0.0;
    if (lead && pending) {
      if (TraceRec* t = trace_at(tr, st, k - 1)) t->V = V;
    }
    if (a.greedy) {
      p_sel_greedy(&ps, slot_max(bp, SL_MAXN, sh), a.eta);
    } else if (n <= LOCAL_SEL_MAX) {
      p_sel_level1(&ps, hn, n, kc, sh_u, sh_l);
      PH(13);
      if (!p_sel_local_smem(&ps, a.keys_n, n, 0, hn, h, sh_u, sh_l, reinterpret_cast<Cand*>(dyn),
                            reinterpret_cast<Cand*>(dyn) + LCAND_CAP)) {
        if (a.ptime && lead) a.ptime[16] += 1;
        if (lead) st->selstat[0] += 1;
        p_sel_local(&ps, a.keys_n, n, 0, h, sh_u, sh_l);
      }
      PH(14);
    } else {
      p_sel_level1(&ps, hn, n, kc, sh_u, sh_l);
      const int dU = ps.mode == SEL_PENDING ? (int)ps.prefix : -1;  // identical in every CTA
      if (!DENSE && !LAZY && RG_SPEC_U && dU >= 0 && dU == predU) {
        // speculation hit: pass T built the level-2 histogram (no scan, no barrier)
        p_sel_level2(&ps, a.hist + 6 * NBINS, sh_u, sh_l);
      } else {
        p_sel_scan<2>(&ps, a.keys_n, n, 0, hn + NBINS, cn, a.ncand, h);
        grid_sync(a.bar, bgen);
        PH(3);
        // ===== P4: level-2 bucket; level-3 scan + candidates =====
        p_sel_level2(&ps, hn + NBINS, sh_u, sh_l);
      }
      if (!DENSE && !LAZY) predU = dU;
      p_sel_scan<3>(&ps, a.keys_n, n, 0, hn + 2 * NBINS, cn, a.ncand, h);
      grid_sync(a.bar, bgen);
      PH(4);
      // ===== P5: exact threshold =====
      p_sel_level3(&ps, hn + 2 * NBINS, cn, a.ncand, a.keys_n, n, 0, h, sh_u, sh_l);
    }
    if (lead && ps.slow) st->selstat[1] += 1;            // column selection took the slow path
    // ===== P5: zeta, Z, |U|, hash; x_k = x_{k-1} + alpha_x v =====
    if constexpr (LAZY) {
      // Algorithm 2: zeta_p = g_p on U (every process), Z_p partials; the lazily
      // averaged x_k = x_{k-1} + (sum_p (X_p / V_p) v_p) / P
      const int P = a.lzP;
      double Zl[LZ_MAX];
      for (int pp = 0; pp < LZ_MAX; ++pp) Zl[pp] = 0.0;
      double Rp = 0.0;
      long long cnt = 0;
      unsigned long long hs = 0ull;
      for (int j = blockIdx.x * PT + threadIdx.x; j < n; j += G * PT) {
        const bool sel = p_selected(&ps, a.keys_n[j], j);
        double t = 0.0;
#pragma unroll
        for (int pp = 0; pp < LZ_MAX; ++pp) {
          if (pp < P) {
            const double g = a.lz_g[(long long)pp * n + j];
            a.lz_zeta[(long long)pp * n + j] = sel ? g : 0.0;
            if (sel) Zl[pp] += g * g;
            const double Xq = lzs[1][pp], Vq = lzs[0][pp];
            if (pending && Xq > 0.0 && Vq > 0.0)
              t = __dadd_rn(t, __dmul_rn(__ddiv_rn(Xq, Vq), a.lz_v[(long long)pp * n + j]));
          }
        }
        if (sel) { cnt += 1; hs += splitmix64((unsigned long long)j); }
        double xj = a.x[j];
        if (pending) { xj = __dadd_rn(xj, __ddiv_rn(t, (double)P)); a.x[j] = xj; }
        if (has_ref) { const double d = xj - a.xstar[j]; Rp += d * d; }
      }
      cnt = warp_sum_ll(cnt);
      hs = warp_sum_u64(hs);
      if ((threadIdx.x & 31) == 0 && (cnt || hs)) {
        atomicAdd(&a.acc[0], (unsigned long long)cnt);
        atomicAdd(&a.acc[1], hs);
      }
      for (int pp = 0; pp < P; ++pp) {
        const double zb = pblock_sum(Zl[pp], sh);
        if (threadIdx.x == 0) a.lz_slots[(long long)(P + pp) * G + blockIdx.x] = zb;
      }
      const double rb = pblock_sum(Rp, sh);
      if (threadIdx.x == 0) { bp[SL_Z * G + blockIdx.x] = 0.0; bp[SL_R * G + blockIdx.x] = rb; }
    } else {
      double Zp = 0.0, Rp = 0.0;
      long long cnt = 0;
      unsigned long long hs = 0ull;
#if RG_VEC_PREFETCH2
      const int stride = G * PT;
      const int j0 = blockIdx.x * PT + threadIdx.x;
      double ns = 0.0, nx = 0.0, nv = 0.0, nxs = 0.0;
      unsigned long long nk = 0ull;
      if (j0 < n) {
        ns = a.s[j0]; nk = a.keys_n[j0]; nx = a.x[j0];
        nv = do_x ? a.v[j0] : 0.0; nxs = has_ref ? a.xstar[j0] : 0.0;
      }
      for (int j = j0; j < n; j += stride) {
        const double sj = ns, vj = nv, xsj = nxs;
        const unsigned long long kj = nk;
        double xj = nx;
        if (j + stride < n) {
          const int q = j + stride;
          ns = a.s[q]; nk = a.keys_n[q]; nx = a.x[q];
          nv = do_x ? a.v[q] : 0.0; nxs = has_ref ? a.xstar[q] : 0.0;
        }
        const bool sel = p_selected(&ps, kj, j);
        a.zeta[j] = sel ? sj : 0.0;
        if (sel) { Zp += sj * sj; cnt += 1; hs += splitmix64((unsigned long long)j); }
        if (do_x) { xj = __dadd_rn(xj, __dmul_rn(alpha_x, vj)); a.x[j] = xj; }
        if (has_ref) { const double d = xj - xsj; Rp += d * d; }
      }
#else
      for (int j = blockIdx.x * PT + threadIdx.x; j < n; j += G * PT) {
        const double sj = a.s[j];
        const bool sel = p_selected(&ps, a.keys_n[j], j);
        a.zeta[j] = sel ? sj : 0.0;
        if (sel) { Zp += sj * sj; cnt += 1; hs += splitmix64((unsigned long long)j); }
        double xj = a.x[j];
        if (do_x) { xj = __dadd_rn(xj, __dmul_rn(alpha_x, a.v[j])); a.x[j] = xj; }
        if (has_ref) { const double d = xj - a.xstar[j]; Rp += d * d; }
      }
#endif
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
    if (a.capU)                                   // block capture (off in production)
      p_capture(a.capU + (k & 1) * (long long)n, &ps, a.keys_n, 0, blockIdx.x * PT + threadIdx.x, n,
                G * PT);
    pending = 0;
    grid_sync(a.bar, bgen);
    PH(5);

    // ===== P6: Z, |U|; pass N (w = A zeta, A x_k) with W / ||b - Ax||^2 partials =====
    double Z;
    if constexpr (LAZY) {
      lz_sums(a.lz_slots + (long long)a.lzP * G, G, 0, G, a.lzP, lzs[2]);   // Z_p
      Z = 0.0;
      for (int pp = 0; pp < a.lzP; ++pp) Z += lzs[2][pp];
    } else {
      Z = slot_sum(bp, SL_Z, sh);
    }
    const double relerr2 = slot_sum(bp, SL_R, sh);
    const long long kp = (long long)__ldcg(&a.acc[0]);
    const unsigned long long hashU = __ldcg(&a.acc[1]);
    if (lead) {
      if (!a.greedy && kp != (ps.mode == SEL_NONE ? 0 : ps.target)) st->error |= 1;
      if (TraceRec* t = trace_at(tr, st, k)) { t->k = k; t->kp = kp; t->hash_u = hashU; t->Z = Z; }
    }
    {
      double Wp = 0.0, Yp = 0.0;
      if constexpr (LAZY) {                       // w = A^(p) zeta_p on this CTA's process
        p_dense_passN(a, dyn, Wp, Yp, a.lz_zeta + (long long)(blockIdx.x / a.lzGp) * n);
      } else if constexpr (DENSE) {
        p_dense_passN(a, dyn, Wp, Yp);
      } else {
        const int g = threadIdx.x / TG;
        csr_tiles(blockIdx.x * (PT / TG) + g, G * (PT / TG), threadIdx.x % TG, 1 + g,
                  reinterpret_cast<TileSmem*>(dyn) + g, tring, a.rp, a.ci, a.cv, a.tilesN,
                  a.tilepN, a.ntilesN,
                  a.zeta, a.x, 1, a.b, a.w, a.ax, Wp, Yp, nullptr, 0, a.vecN, RG_REV_N);
      }
      const double wb = pblock_sum(Wp, sh);
      const double yb = pblock_sum(Yp, sh);
      if (threadIdx.x == 0) { bp[SL_W * G + blockIdx.x] = wb; bp[SL_Y * G + blockIdx.x] = yb; }
    }
    grid_sync(a.bar, bgen);
    PH(6);

    // ===== P8: stop test on x_k; z_{k+1}, r, row scores and keys, level-1 histogram =====
    double W;
    if constexpr (LAZY) {                         // W_p over the process's own CTAs
      lz_sums(bp + SL_W * G, 0, a.lzGp, a.lzGp, a.lzP, lzs[3]);
      W = 0.0;
      for (int pp = 0; pp < a.lzP; ++pp) W += lzs[3][pp];
    } else {
      W = slot_sum(bp, SL_W, sh);
    }
    const double Y = slot_sum(bp, SL_Y, sh);
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
        if (TraceRec* t = trace_at(tr, st, k)) t->W = W;
        if (k >= 1) { if (TraceRec* t = trace_at(tr, st, k - 1)) t->rse = rse; }
      }
      if (halt) {
        p_zero_side(a, 0);
        if (lead) {
          st->halted = 1; st->outcome = outcome; st->iters = k; st->rse_out = rse;
          st->relerr_out = rel; st->k = k; st->pending = 0; st->X = X;
          st->kp_prev = kp_prev; st->kpp_prev = kpp_prev;
          st->Z = Z; st->W = W; st->Y = Y; st->V = V; st->relerr2 = relerr2;
          st->npass += 2 * (k - k_begin + 1);
        }
        return;
      }
    }
    // sparse, grid-wide row selection: a speculative level-2 histogram of the keys in the
    // predicted level-1 bucket (the last iteration's), in the free tile memory
    constexpr bool SPEC = !DENSE && !LAZY;
    unsigned int* h2 = reinterpret_cast<unsigned int*>(dyn);
    for (int i = threadIdx.x; i < NBINS; i += PT) {
      h[i] = 0u;
      if (SPEC) h2[i] = 0u;
    }
    __syncthreads();
    double EmaxM = 0.0;
    {
      // Algorithm 2: the local z-step of this CTA's process, alpha = Z_p / W_p
      const int lzp = LAZY ? (int)(blockIdx.x / a.lzGp) : 0;
      const double Zs = LAZY ? lzs[2][lzp] : Z, Ws = LAZY ? lzs[3][lzp] : W;
      const int doz = kp > 0 && Ws > 0.0;
      const double az = doz ? __ddiv_rn(Zs, Ws) : 0.0;
      // rows of this sweep: grid-stride over all rows, or (Algorithm 2) this
      // CTA's own contiguous rows, which lie in its process
      const int m_end = LAZY ? (int)((long long)m_loc * (blockIdx.x + 1) / G) : m_loc;
#if RG_VEC_PREFETCH
      // software-pipelined: the next element's five inputs are in flight while
      // this element's key (Philox + log + two divisions) is computed
      const int stride = LAZY ? PT : G * PT;
      int i0 = LAZY ? (int)((long long)m_loc * blockIdx.x / G) + threadIdx.x
                    : blockIdx.x * PT + threadIdx.x;
      double nz = 0.0, nw = 0.0, nb = 0.0, nax = 0.0, nrho = 0.0;
      if (i0 < m_end) {
        nz = a.z[i0]; nw = doz ? a.w[i0] : 0.0; nb = a.b[i0]; nax = a.ax[i0]; nrho = a.rho[i0];
      }
      for (int i = i0; i < m_end; i += stride) {
        double zi = nz;
        const double wi = nw, bi = nb, axi = nax, p = nrho;
        if (i + stride < m_end) {
          const int j = i + stride;
          nz = a.z[j]; nw = doz ? a.w[j] : 0.0; nb = a.b[j]; nax = a.ax[j]; nrho = a.rho[j];
        }
        if (doz) { zi = __dsub_rn(zi, __dmul_rn(az, wi)); a.z[i] = zi; }
        const double ri = __dsub_rn(__dsub_rn(bi, zi), axi);
        a.r[i] = ri;
#else
      static_assert(!LAZY || RG_VEC_PREFETCH, "Algorithm 2 uses the pipelined row sweep");
      for (int i = blockIdx.x * PT + threadIdx.x; i < m_loc; i += G * PT) {
        double zi = a.z[i];
        if (doz) { zi = __dsub_rn(zi, __dmul_rn(az, a.w[i])); a.z[i] = zi; }
        const double ri = __dsub_rn(__dsub_rn(a.b[i], zi), a.ax[i]);
        a.r[i] = ri;
        const double p = a.rho[i];
#endif
        const double eps = p > 0.0 ? __ddiv_rn(__dmul_rn(ri, ri), p) : 0.0;
        EmaxM = fmax(EmaxM, eps);
        const unsigned long long key = sel_key(eps, (unsigned long long)(a.row0 + i), k, 1u, seed, a.greedy);
        a.keys_m[i] = key;
        atomicAdd(&h[key >> L1_SHIFT], 1u);
        if (SPEC && (int)(key >> L1_SHIFT) == predJ) atomicAdd(&h2[(key >> L2_SHIFT) & 0xFFFull], 1u);
      }
    }
    __syncthreads();
    if (SPEC && predJ >= 0) flush_hist<PT>(h2, a.hist + 7 * NBINS, NBINS);
    if constexpr (LAZY) {
      flush_hist<PT>(h, a.lz_hist + (long long)(blockIdx.x / a.lzGp) * NBINS, NBINS);
    } else {
      flush_hist<PT>(h, hm, NBINS);
    }
    {
      const double eb = pblock_max(EmaxM, sh);
      if (threadIdx.x == 0) bp[SL_MAXM * G + blockIdx.x] = eb;
    }
    p_zero_side(a, 0);                          // n-side buffers: consumed in P3..P6
    grid_sync(a.bar, bgen);
    PH(7);

    // ===== P9: level-1 bucket (J); level-2 scan =====
    if constexpr (LAZY) {
      // Algorithm 2: each process samples round(eta d_p) of its own rows;
      // every CTA resolves its process's selection locally (d_p <= LOCAL_SEL_MAX)
      const int pp = (int)(blockIdx.x / a.lzGp);
      const long long r0p = a.lz_r0[pp], dp = a.lz_r0[pp + 1] - r0p;
      const unsigned int* hp = a.lz_hist + (long long)pp * NBINS;
      p_sel_level1(&ps, hp, dp, a.lz_kr[pp], sh_u, sh_l);
      if (!p_sel_local_smem(&ps, a.keys_m + r0p, dp, a.row0 + r0p, hp, h, sh_u, sh_l,
                            reinterpret_cast<Cand*>(dyn), reinterpret_cast<Cand*>(dyn) + LCAND_CAP))
        p_sel_local(&ps, a.keys_m + r0p, dp, a.row0 + r0p, h, sh_u, sh_l);
    } else if (a.greedy) {
      p_sel_greedy(&ps, slot_max(bp, SL_MAXM, sh), a.eta);
    } else if (m_loc <= LOCAL_SEL_MAX) {
      p_sel_level1(&ps, hm, m_loc, kr, sh_u, sh_l);
      if (!p_sel_local_smem(&ps, a.keys_m, m_loc, a.row0, hm, h, sh_u, sh_l,
                            reinterpret_cast<Cand*>(dyn), reinterpret_cast<Cand*>(dyn) + LCAND_CAP,
                            a.ptime ? a.ptime + 18 : nullptr)) {
        if (a.ptime && lead) a.ptime[17] += 1;
        if (lead) st->selstat[0] += 1;
        p_sel_local(&ps, a.keys_m, m_loc, a.row0, h, sh_u, sh_l);
      }
      PH(15);
    } else {
      p_sel_level1(&ps, hm, m_loc, kr, sh_u, sh_l);
      const int d = ps.mode == SEL_PENDING ? (int)ps.prefix : -1;   // identical in every CTA
      if (SPEC && d >= 0 && d == predJ) {
        // speculation hit: the level-2 histogram was built with the keys (no scan, no barrier)
        p_sel_level2(&ps, a.hist + 7 * NBINS, sh_u, sh_l);
      } else {
        p_sel_scan<2>(&ps, a.keys_m, m_loc, a.row0, hm + NBINS, cm, a.ncand + 1, h);
        grid_sync(a.bar, bgen);
        PH(8);
        // ===== P10: level-2 bucket; level-3 scan + candidates =====
        p_sel_level2(&ps, hm + NBINS, sh_u, sh_l);
      }
      if (SPEC) predJ = d;
      p_sel_scan<3>(&ps, a.keys_m, m_loc, a.row0, hm + 2 * NBINS, cm, a.ncand + 1, h);
      grid_sync(a.bar, bgen);
      PH(9);
      // ===== P11: exact threshold =====
      p_sel_level3(&ps, hm + 2 * NBINS, cm, a.ncand + 1, a.keys_m, m_loc, a.row0, h, sh_u, sh_l);
    }
    if (lead && ps.slow) st->selstat[1] += 1;            // row selection took the slow path
    // ===== P11: xi = r on J, X, |J|, hash (dense: fused into the next pass T) =====
    if constexpr (!(DENSE && RG_FUSE_XI)) {
      double Xp = 0.0;
      long long cnt = 0;
      unsigned long long hs = 0ull;
#if RG_VEC_PREFETCH2
      // software-pipelined: the next element's key and residual are in flight
      const int stride = LAZY ? PT : G * PT;
      const int i0 = LAZY ? (int)((long long)m_loc * blockIdx.x / G) + threadIdx.x
                          : blockIdx.x * PT + threadIdx.x;
      const int i_end = LAZY ? (int)((long long)m_loc * (blockIdx.x + 1) / G) : m_loc;
      unsigned long long nk = 0ull;
      double nr = 0.0;
      if (i0 < i_end) { nk = a.keys_m[i0]; nr = a.r[i0]; }
      for (int i = i0; i < i_end; i += stride) {
        const unsigned long long ki = nk;
        const double ri = nr;
        if (i + stride < i_end) { nk = a.keys_m[i + stride]; nr = a.r[i + stride]; }
        const long long gi = a.row0 + i;
        const bool sel = p_selected(&ps, ki, gi);
        a.xi[i] = sel ? ri : 0.0;
        if (sel) { Xp += ri * ri; cnt += 1; hs += splitmix64((unsigned long long)gi); }
      }
#else
      const int i_beg = LAZY ? (int)((long long)m_loc * blockIdx.x / G) + threadIdx.x
                             : blockIdx.x * PT + threadIdx.x;
      const int i_end = LAZY ? (int)((long long)m_loc * (blockIdx.x + 1) / G) : m_loc;
      for (int i = i_beg; i < i_end; i += (LAZY ? PT : G * PT)) {
        const long long gi = a.row0 + i;
        const bool sel = p_selected(&ps, a.keys_m[i], gi);
        const double ri = a.r[i];
        a.xi[i] = sel ? ri : 0.0;
        if (sel) { Xp += ri * ri; cnt += 1; hs += splitmix64((unsigned long long)gi); }
      }
#endif
      cnt = warp_sum_ll(cnt);
      hs = warp_sum_u64(hs);
      if ((threadIdx.x & 31) == 0 && (cnt || hs)) {
        atomicAdd(&a.acc[2], (unsigned long long)cnt);
        atomicAdd(&a.acc[3], hs);
      }
      const double xb = pblock_sum(Xp, sh);
      if (threadIdx.x == 0) bp[SL_X * G + blockIdx.x] = xb;
      if (a.capJ)                                 // block capture (off in production)
        p_capture(a.capJ + (k & 1) * (long long)m_loc, &ps, a.keys_m, a.row0,
                  LAZY ? (int)((long long)m_loc * blockIdx.x / G) + threadIdx.x : blockIdx.x * PT + threadIdx.x,
                  LAZY ? (int)((long long)m_loc * (blockIdx.x + 1) / G) : m_loc, LAZY ? PT : G * PT);
      grid_sync(a.bar, bgen);
    }
    PH(10);

    // ===== P12: X, |J|; bookkeeping; k++ =====
    if constexpr (!(DENSE && RG_FUSE_XI)) {
      X = slot_sum(bp, SL_X, sh);
      const long long kpp = (long long)__ldcg(&a.acc[2]);
      const unsigned long long hashJ = __ldcg(&a.acc[3]);
      if (lead) {
        if (!a.greedy && !LAZY && kpp != (ps.mode == SEL_NONE ? 0 : ps.target)) st->error |= 2;
        if (TraceRec* t = trace_at(tr, st, k)) { t->kpp = kpp; t->hash_j = hashJ; t->X = X; }
      }
      kpp_prev = kpp;
    }
    kp_prev = kp;
    pending = 1;
    k += 1;
    PH(0);
    __syncthreads();
  }
#undef PH
}

}  // namespace rg
