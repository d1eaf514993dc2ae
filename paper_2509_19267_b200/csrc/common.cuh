// common.cuh — device-side state, Philox sampler and reduction helpers.
//
// Philox4x32-10 is re-stated here from the SC'11 definition (Salmon et al.);
// it shares no code with the oracle (oracle/philox.py).  Layout (R5):
//   ctr = (index, k mod 2^32, step, k >> 32), key = (seed mod 2^32, seed >> 32)
// U01 (R6): u = (w >> 12) * 2^-52 + 2^-53, w = (o1 << 32) | o0.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/rgdbek.h"

namespace rg {

// ---------------------------------------------------------------------------
// Keys.  kappa = -ln(u)/eps is positive, so its IEEE bits order like uint64.
// eps == 0 (never selectable, reading R6) maps to all-ones, above +inf.
// ---------------------------------------------------------------------------
constexpr unsigned long long KEY_NEVER = 0xFFFFFFFFFFFFFFFFull;

// Selection modes (SelState::mode)
enum : int { SEL_NONE = 0, SEL_ALL = 1, SEL_THRESH = 2, SEL_PENDING = 3, SEL_GREEDY = 4 };

// Radix levels of the exact k-th key search: L1 = key >> 52 (sign+exponent,
// 4096 bins, fused into the key-producing kernel), L2 = bits [51:40],
// L3 = bits [39:28] (+ candidate list), final = rank among the survivors.
constexpr int L1_SHIFT = 52, L2_SHIFT = 40, L3_SHIFT = 28;
constexpr int NBINS = 4096;
// Candidate capacities of the exact selection.  The -D overrides exist only for the
// selection-stress test build (tests/test_gpu_selection_paths.py), which shrinks them
// so that every overflow / slow path of select.cuh and persistent.cuh runs.
#ifndef RG_CAND_CAP
#define RG_CAND_CAP (1u << 16)
#endif
#ifndef RG_FINAL_CAP
#define RG_FINAL_CAP 1024
#endif
constexpr unsigned int CAND_CAP = RG_CAND_CAP;
constexpr int FINAL_CAP = RG_FINAL_CAP;

struct Cand { unsigned long long key; long long idx; };

struct SelState {
  unsigned long long prefix;   // key >> shift of the resolved bucket
  long long below;             // # keys strictly below the bucket
  long long target;            // block size k' after the clamp
  long long npos;              // # positive scores
  unsigned long long tau;      // threshold key: select (key, idx) <= (tau, tie)
  long long tie;
  int mode;
  int slow;                    // candidate overflow -> single-block slow path
  unsigned int ncand;
  unsigned int spec_hit;       // graph engine: level-1 bucket == the predicted digit
};

// Last-block counters
enum : int { C_NSIDE = 0, C_SEL2N, C_SEL3N, C_MASKN, C_PASSN, C_MSIDE, C_SEL2M, C_SEL3M,
             C_MASKM, C_SURV, C_NUM };

struct Scal {
  // call control
  long long k, k_begin, k_end;
  double tol;
  int stop_mode, halted, outcome, pending;
  unsigned long long seed;
  int has_ref, do_x, error, pad0;
  // iteration scalars
  double X, V, Z, W, Y, alpha_x, relerr2;
  long long kp, kpp, kp_prev, kpp_prev, kc, kr;
  unsigned long long hashU, hashJ;
  long long cnt_acc;           // integer accumulators (atomics, deterministic)
  unsigned long long hash_acc;
  double bnorm2, xsnorm2;
  long long iters;
  double rse_out, relerr_out;
  long long trace_cap;
  SelState seln, selm;
  unsigned int counters[C_NUM];
  // multi-GPU (row-sharded, graph engine): rank-local partials that are
  // allreduced in place by NCCL between kernels
  int dist, pad1;
  long long m_global;
  double wy[2];                  // [W_p, ||b_p - A_p x||^2]
  unsigned long long jacc[2];    // [|J_p|, hash(J_p)]
  unsigned int nsurv, surv_over; // local survivors of the level-3 bucket
  long long npass;               // full passes over A since the last reset (exact mode)
  // selection path counters since create (rgdbek_selection_stats): [0] CTA-local
  // selections whose level-1 bucket overflowed the shared-memory list, [1] selections
  // resolved by the persistent slow path, [2] by the graph engine's k_select_slow
  long long selstat[4];
  // peer-memory sharded engine (sharded.cuh): exchange counter (identical on every rank,
  // persists across launches with the flag words) and the combined ||b||^2
  unsigned int xgen, pad3;
  double bnorm2_global;
  double abytes;                 // exact mode: algorithmic bytes of A read since the last reset
  // graph engine: level-1 digit predicted for each side's next selection (the last one's);
  // the key kernel counts that bucket's keys by level-2 digit (speculative level 2)
  int spec_pred[2];
};

constexpr int SURV_CAP = 256;    // per-rank survivors exchanged by allgather

// Read-only / streaming global loads
__device__ __forceinline__ double2 ld_stream2(const double* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ double ld_stream(const double* p) {
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}

// ---------------------------------------------------------------------------
// Philox4x32-10
// ---------------------------------------------------------------------------
__device__ __forceinline__ void philox4x32_10(uint32_t& c0, uint32_t& c1, uint32_t& c2,
                                              uint32_t& c3, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += W0; k1 += W1; }
    const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
    const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
}

__device__ __forceinline__ double u01(uint32_t o0, uint32_t o1) {
  const unsigned long long w = ((unsigned long long)o1 << 32) | o0;
  return __dadd_rn(__dmul_rn((double)(w >> 12), 0x1p-52), 0x1p-53);
}

// key bits of kappa = -ln(u(seed,k,step,gidx)) / eps   (reading R3)
__device__ __forceinline__ unsigned long long make_key(double eps, unsigned long long gidx,
                                                       long long k, uint32_t step,
                                                       unsigned long long seed) {
  if (!(eps > 0.0)) return KEY_NEVER;
  uint32_t c0 = (uint32_t)gidx, c1 = (uint32_t)(unsigned long long)k, c2 = step,
           c3 = (uint32_t)((unsigned long long)k >> 32);
  philox4x32_10(c0, c1, c2, c3, (uint32_t)seed, (uint32_t)(seed >> 32));
  const double u = u01(c0, c1);
  const double kappa = __ddiv_rn(-log(u), eps);
  return (unsigned long long)__double_as_longlong(kappa);
}

// Selection key of one score: the Philox exponential key (RGDBEK) or, in
// the greedy GDBEK mode, the score's own bits.
__device__ __forceinline__ unsigned long long sel_key(double eps, unsigned long long gidx,
                                                      long long k, uint32_t step,
                                                      unsigned long long seed, int greedy) {
  if (greedy) return eps > 0.0 ? (unsigned long long)__double_as_longlong(eps) : KEY_NEVER;
  return make_key(eps, gidx, k, step, seed);
}

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// ---------------------------------------------------------------------------
// Deterministic block reductions (fixed tree for a fixed blockDim)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum of one double per thread over the block; result valid in all threads.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh /* >= NT/32 */) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = (l < NT / 32) ? sh[l] : 0.0;
    t = warp_sum(t);
    if (l == 0) sh[0] = t;
  }
  __syncthreads();
  t = sh[0];
  __syncthreads();
  return t;
}

// Last-block-done detection.  Every thread fences its own global writes first.
__device__ __forceinline__ bool last_block(unsigned int* counter) {
  __shared__ int is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int nb = gridDim.x * gridDim.y * gridDim.z;
    const unsigned int t = atomicAdd(counter, 1u);
    is_last = (t == nb - 1);
    if (is_last) *counter = 0u;
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last != 0;
}

// Sum of `count` doubles written by other blocks (fixed order: deterministic).
template <int NT>
__device__ __forceinline__ double reduce_partials(const double* part, int count, double* sh) {
  double v = 0.0;
  for (int i = threadIdx.x; i < count; i += NT) v += __ldcg(part + i);
  return block_sum<NT>(v, sh);
}

// ---------------------------------------------------------------------------
// mbarrier + bulk-copy (TMA, cp.async.bulk) helpers, CTA scope.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile("{\n .reg .pred p;\n WAIT_%=:\n"
               " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra WAIT_%=;\n}" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Weak (L1-cached, coherent after the grid barrier's acquire) load of a vector
// that other CTAs rewrite during a persistent launch: never the .nc path.
__device__ __forceinline__ double ld_weak(const double* p) {
  double v;
  asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

}  // namespace rg
