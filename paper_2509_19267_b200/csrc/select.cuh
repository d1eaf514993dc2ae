// select.cuh — exact k-th smallest (key, index) selection on the device.
//
// Realises "select n*eta columns / m*eta rows using probability P" (P:116,
// P:121; readings R3/R4) as: U = the k' indices with the smallest
// (kappa, index) pairs.  The threshold (tau, tie) is found by a 3-level MSD
// radix search over the 64-bit key bits (level 1 fused into the kernel that
// produces the keys), then an exact rank among the few survivors.
// Result: select j iff (key_j, j) <= (tau, tie) lexicographically.
#pragma once
#include "common.cuh"

namespace rg {

// Smem histogram flush: add the nonzero bins to the global histogram.
template <int NT>
__device__ __forceinline__ void flush_hist(const unsigned int* sh, unsigned int* gh, int nb) {
  for (int b = threadIdx.x; b < nb; b += NT) {
    const unsigned int c = sh[b];
    if (c) atomicAdd(gh + b, c);
  }
}

// Find the bucket holding the need-th (1-based) key in the global histogram;
// updates ss->prefix / ss->below and zeroes the histogram.  One block.
template <int NT>
__device__ void finalize_level(SelState* ss, unsigned int* gh, int shift_digit) {
  constexpr int PER = NBINS / NT;
  __shared__ long long ex[NT];
  unsigned int loc[PER];
  long long mine = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    loc[i] = __ldcg(gh + threadIdx.x * PER + i);
    mine += loc[i];
  }
  ex[threadIdx.x] = mine;
  __syncthreads();
  // inclusive scan (Hillis-Steele) over NT partial counts
  for (int o = 1; o < NT; o <<= 1) {
    long long t = (threadIdx.x >= o) ? ex[threadIdx.x - o] : 0;
    __syncthreads();
    ex[threadIdx.x] += t;
    __syncthreads();
  }
  const long long need = ss->target - ss->below;
  const long long base = ex[threadIdx.x] - mine;
  if (base < need && need <= base + mine) {
    long long c = base;
    for (int i = 0; i < PER; ++i) {
      if (c + loc[i] >= need) {
        const unsigned long long digit = (unsigned long long)(threadIdx.x * PER + i);
        ss->prefix = (shift_digit == L1_SHIFT) ? digit : ((ss->prefix << 12) | digit);
        ss->below += c;
        break;
      }
      c += loc[i];
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < PER; ++i) gh[threadIdx.x * PER + i] = 0u;
  __syncthreads();
}

// Level-1 finalize, run by the last block of the key-producing kernel.
// k_block is the unclamped block size (k_c or k_r).
template <int NT>
__device__ void finalize_level1(SelState* ss, unsigned int* gh, long long N, long long k_block) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long never = (long long)__ldcg(gh + (NBINS - 1));
    ss->npos = N - never;
    ss->target = k_block < ss->npos ? k_block : ss->npos;
    ss->below = 0;
    ss->prefix = 0;
    ss->ncand = 0u;
    ss->slow = 0;
    ss->tie = -1;
    if (ss->target == 0) {
      ss->mode = SEL_NONE;
      ss->tau = 0ull;
    } else if (ss->target == ss->npos) {
      ss->mode = SEL_ALL;                // every positive score: all keys != NEVER
      ss->tau = KEY_NEVER - 1ull;
      ss->tie = 0x7FFFFFFFFFFFFFFFll;
    } else {
      ss->mode = SEL_PENDING;
    }
  }
  __syncthreads();
  if (ss->mode == SEL_PENDING) {
    finalize_level<NT>(ss, gh, L1_SHIFT);
  } else {
    for (int b = threadIdx.x; b < NBINS; b += NT) gh[b] = 0u;
  }
}

// Speculative level 2 of the graph engine, decided by the last block of the key kernel
// right after finalize_level1: a hit when the new level-1 bucket is the predicted digit
// (the key kernel counted that bucket's keys into `spec` by level-2 digit); a miss zeroes
// `spec` for the next build.  The prediction becomes the new bucket.
template <int NT>
__device__ void spec_decide(SelState* ss, int* pred, unsigned int* spec) {
  __shared__ int hit;
  if (threadIdx.x == 0) {
    hit = ss->mode == SEL_PENDING && (long long)ss->prefix == (long long)*pred;
    ss->spec_hit = hit ? 1u : 0u;
    *pred = ss->mode == SEL_PENDING ? (int)ss->prefix : -1;
  }
  __syncthreads();
  if (!hit)
    for (int b = threadIdx.x; b < NBINS; b += NT) spec[b] = 0u;
}

// Level 2 / 3 pass over all keys of the bucket resolved so far.  spec (level 2 only, or
// nullptr): the speculative level-2 histogram — on a hit the scan is skipped.
template <int NT, int LEVEL>
__global__ void __launch_bounds__(NT) k_select_pass(const unsigned long long* __restrict__ keys,
                                                    long long N, long long idx_base, Scal* st,
                                                    int which, unsigned int* gh, Cand* cand,
                                                    unsigned int* spec = nullptr) {
  if (st->halted) return;
  SelState* ss = which ? &st->selm : &st->seln;
  if (ss->mode != SEL_PENDING) return;
  if (LEVEL == 2 && spec && ss->spec_hit) {
    if (!last_block(&st->counters[C_SEL2N + (which ? (C_SEL2M - C_SEL2N) : 0)])) return;
    finalize_level<NT>(ss, spec, L2_SHIFT);   // zeroes spec for the next build
    return;
  }
  __shared__ __align__(16) unsigned int h[NBINS];
  for (int b = threadIdx.x; b < NBINS; b += NT) h[b] = 0u;
  __syncthreads();
  constexpr int SF = (LEVEL == 2) ? L1_SHIFT : L2_SHIFT;
  constexpr int SD = (LEVEL == 2) ? L2_SHIFT : L3_SHIFT;
  const unsigned long long pre = ss->prefix;
  const long long stride = (long long)gridDim.x * NT;
  // SCAN_U keys in flight per thread (independent loads), visited in the same order
  constexpr int SCAN_U = 4;
  for (long long i0 = (long long)blockIdx.x * NT + threadIdx.x; i0 < N; i0 += SCAN_U * stride) {
    unsigned long long kk[SCAN_U];
#pragma unroll
    for (int u = 0; u < SCAN_U; ++u) kk[u] = i0 + u * stride < N ? keys[i0 + u * stride] : 0ull;
#pragma unroll
    for (int u = 0; u < SCAN_U; ++u) {
      const long long i = i0 + u * stride;
      const unsigned long long key = kk[u];
      if (i < N && (key >> SF) == pre) {
        atomicAdd(&h[(key >> SD) & 0xFFFull], 1u);
        if (LEVEL == 3 && !(which && st->dist)) {
          const unsigned int slot = atomicAdd(&ss->ncand, 1u);
          if (slot < CAND_CAP) cand[slot] = Cand{key, idx_base + i};
        }
      }
    }
  }
  __syncthreads();
  flush_hist<NT>(h, gh, NBINS);
  if (which && st->dist) return;             // sharded rows: allreduce, then k_sel_fin
  if (!last_block(&st->counters[(LEVEL == 2 ? C_SEL2N : C_SEL3N) + (which ? (C_SEL2M - C_SEL2N) : 0)]))
    return;
  finalize_level<NT>(ss, gh, SD);
  if (LEVEL != 3) return;
  // ---- exact rank among the survivors (key >> 28 == prefix) ----
  __shared__ int nf;
  Cand* fc = reinterpret_cast<Cand*>(h);      // 16 KB = FINAL_CAP candidates
  if (threadIdx.x == 0) nf = 0;
  __syncthreads();
  const unsigned int nc = __ldcg(&ss->ncand);
  const unsigned long long pre3 = ss->prefix;
  if (nc <= CAND_CAP) {
    for (unsigned int c = threadIdx.x; c < nc; c += NT) {
      const Cand e = cand[c];
      if ((e.key >> L3_SHIFT) == pre3) {
        const int s = atomicAdd(&nf, 1);
        if (s < FINAL_CAP) fc[s] = e;
      }
    }
  }
  __syncthreads();
  if (nc > CAND_CAP || nf > FINAL_CAP) {
    if (threadIdx.x == 0) ss->slow = 1;
    return;
  }
  const long long need = ss->target - ss->below;     // 1-based rank inside the survivors
  for (int e = threadIdx.x; e < nf; e += NT) {
    const Cand me = fc[e];
    long long rank = 0;
    for (int f = 0; f < nf; ++f) {
      const Cand o = fc[f];
      rank += (o.key < me.key) || (o.key == me.key && o.idx < me.idx);
    }
    if (rank == need - 1) {
      ss->tau = me.key;
      ss->tie = me.idx;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ss->mode = SEL_THRESH;
    ss->ncand = 0u;
  }
}

// Slow path (candidate overflow; practically only with massive exact ties):
// one block resolves the remaining key bits and then the tie index by radix
// levels over ALL keys.  Exact, O(levels * N) on a single SM.
template <int NT>
__global__ void __launch_bounds__(NT) k_select_slow(const unsigned long long* __restrict__ keys,
                                                    long long N, long long idx_base, Scal* st,
                                                    int which) {
  if (st->halted) return;
  SelState* ss = which ? &st->selm : &st->seln;
  if (ss->mode != SEL_PENDING || !ss->slow) return;
  __shared__ __align__(16) unsigned int h[NBINS];
  __shared__ long long ex[NT];
  __shared__ unsigned long long sel_digit;
  __shared__ long long sel_below;
  // levels over key bits [27:16], [15:4], [3:0]; then index bits [31:20], [19:8], [7:0]
  const int shifts[6] = {16, 4, 0, 20, 8, 0};
  const unsigned long long masks[6] = {0xFFF, 0xFFF, 0xF, 0xFFF, 0xFFF, 0xFF};
  unsigned long long kpre = ss->prefix;   // key >> 28
  int kshift = L3_SHIFT;
  unsigned long long ipre = 0;
  int ishift = 32;
  long long below = ss->below;
  const long long target = ss->target;
  for (int lv = 0; lv < 6; ++lv) {
    for (int b = threadIdx.x; b < NBINS; b += NT) h[b] = 0u;
    __syncthreads();
    const bool on_idx = lv >= 3;
    for (long long i = threadIdx.x; i < N; i += NT) {
      const unsigned long long key = keys[i];
      const unsigned long long gi = (unsigned long long)(idx_base + i);
      bool in = on_idx ? (key == kpre && (ishift >= 32 ? true : (gi >> ishift) == ipre))
                       : ((key >> kshift) == kpre);
      if (in) {
        const unsigned long long d = on_idx ? ((gi >> shifts[lv]) & masks[lv])
                                            : ((key >> shifts[lv]) & masks[lv]);
        atomicAdd(&h[d], 1u);
      }
    }
    __syncthreads();
    constexpr int PER = NBINS / NT;
    long long mine = 0;
    for (int i = 0; i < PER; ++i) mine += h[threadIdx.x * PER + i];
    ex[threadIdx.x] = mine;
    __syncthreads();
    for (int o = 1; o < NT; o <<= 1) {
      long long t = (threadIdx.x >= o) ? ex[threadIdx.x - o] : 0;
      __syncthreads();
      ex[threadIdx.x] += t;
      __syncthreads();
    }
    const long long need = target - below;
    const long long base = ex[threadIdx.x] - mine;
    if (base < need && need <= base + mine) {
      long long c = base;
      for (int i = 0; i < PER; ++i) {
        if (c + h[threadIdx.x * PER + i] >= need) {
          sel_digit = (unsigned long long)(threadIdx.x * PER + i);
          sel_below = c;
          break;
        }
        c += h[threadIdx.x * PER + i];
      }
    }
    __syncthreads();
    below += sel_below;
    const int bits = (masks[lv] == 0xFFF) ? 12 : (masks[lv] == 0xFF ? 8 : 4);
    if (!on_idx) {
      kpre = (kpre << bits) | sel_digit;
      kshift = shifts[lv];
    } else {
      ipre = (ishift >= 32) ? sel_digit : ((ipre << bits) | sel_digit);
      ishift = shifts[lv];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ss->tau = kpre;
    ss->tie = (long long)ipre;
    ss->mode = SEL_THRESH;
    ss->slow = 0;
    ss->ncand = 0u;
    st->selstat[2] += 1;
  }
}

// ---- row-sharded (multi-GPU) selection of J: finalize after each histogram
// allreduce; the level-3 survivors of every rank are allgathered and ranked.
template <int NT>
__global__ void __launch_bounds__(NT) k_sel_fin(Scal* st, unsigned int* gh, int level) {
  if (st->halted) return;
  SelState* ss = &st->selm;
  if (level == 1) {
    finalize_level1<NT>(ss, gh, st->m_global, st->kr);
    return;
  }
  if (ss->mode != SEL_PENDING) return;
  finalize_level<NT>(ss, gh, level == 2 ? L2_SHIFT : L3_SHIFT);
}

// Local keys in the level-3 bucket -> surv[1..], surv[0] = {count, overflow}.
template <int NT>
__global__ void __launch_bounds__(NT) k_collect_surv(const unsigned long long* __restrict__ keys,
                                                     long long N, long long idx_base, Scal* st,
                                                     Cand* surv) {
  if (st->halted) return;
  const SelState& ss = st->selm;
  if (ss.mode != SEL_PENDING) return;
  const unsigned long long pre3 = ss.prefix;
  for (long long i = (long long)blockIdx.x * NT + threadIdx.x; i < N; i += (long long)gridDim.x * NT) {
    const unsigned long long key = keys[i];
    if ((key >> L3_SHIFT) == pre3) {
      const unsigned int sl = atomicAdd(&st->nsurv, 1u);
      if (sl < SURV_CAP) surv[1 + sl] = Cand{key, idx_base + i};
      else st->surv_over = 1u;
    }
  }
  if (!last_block(&st->counters[C_SURV])) return;
  if (threadIdx.x == 0) {
    const unsigned int c = __ldcg(&st->nsurv);
    surv[0] = Cand{(unsigned long long)(c < SURV_CAP ? c : SURV_CAP), (long long)__ldcg(&st->surv_over)};
    st->nsurv = 0u;
    st->surv_over = 0u;
  }
}

// Rank the survivors of all ranks (identical on every rank) -> (tau, tie).
template <int NT>
__global__ void __launch_bounds__(NT) k_rank_surv(Scal* st, const Cand* __restrict__ all, int P) {
  if (st->halted) return;
  SelState* ss = &st->selm;
  if (ss->mode != SEL_PENDING) return;
  __shared__ Cand fc[8 * SURV_CAP];
  __shared__ int nf;
  if (threadIdx.x == 0) nf = 0;
  __syncthreads();
  for (int r = 0; r < P; ++r) {
    const Cand* blk = all + (long long)r * (SURV_CAP + 1);
    const int c = (int)blk[0].key;
    if (blk[0].idx && threadIdx.x == 0) st->error |= 4;     // survivor overflow on a rank
    for (int e = threadIdx.x; e < c; e += NT) {
      const int sl = atomicAdd(&nf, 1);
      if (sl < 8 * SURV_CAP) fc[sl] = blk[1 + e];
    }
  }
  __syncthreads();
  const int cnt = nf < 8 * SURV_CAP ? nf : 8 * SURV_CAP;
  const long long need = ss->target - ss->below;
  for (int e = threadIdx.x; e < cnt; e += NT) {
    const Cand me = fc[e];
    long long rank = 0;
    for (int f = 0; f < cnt; ++f) {
      const Cand o = fc[f];
      rank += (o.key < me.key) || (o.key == me.key && o.idx < me.idx);
    }
    if (rank == need - 1) { ss->tau = me.key; ss->tie = me.idx; }
  }
  __syncthreads();
  if (threadIdx.x == 0) ss->mode = SEL_THRESH;
}

__device__ __forceinline__ bool is_selected(const SelState& ss, unsigned long long key, long long gidx) {
  if (ss.mode == SEL_THRESH) return key < ss.tau || (key == ss.tau && gidx <= ss.tie);
  if (ss.mode == SEL_ALL) return key != KEY_NEVER;
  return false;
}

}  // namespace rg
