// csr_tiles.cuh — CSR (or CSC) dual SpMV by nnz tiles ("CSR-stream").
//
// A sparse pass computes o1 = A in1 and o2 = A in2 over rows (pass N: A zeta,
// A x; pass T over the CSC: A^T z, A^T xi).  Short rows (5-41 nnz here) make
// a row-per-thread or sub-warp-per-row loop a chain of three dependent memory
// round trips per row (row pointer -> value/index -> gathered vector), so
// each warp keeps almost nothing in flight.  Instead a worker group of TG
// threads takes a tile of consecutive rows holding <= TILE_NNZ nonzeros:
//   1. stage the tile's row pointers in shared memory;
//   2. stream its values and indices with fully coalesced loads (every thread
//      ~8 independent loads in flight) and store the products val*in1[idx],
//      val*in2[idx] in shared memory;
//   3. sum each row's products in order (deterministic) from shared memory.
// A row longer than TILE_NNZ is a tile by itself, reduced across the group.
// Tiles are precomputed at create (greedy on the row pointer).
#pragma once
#include "common.cuh"

namespace rg {

constexpr int TG = 128;              // threads per worker group
constexpr int TILE_NNZ = 1024;       // 8 nonzeros per thread, in two sub-rounds of 4
constexpr int TILE_ROWS = 256;

struct TileSmem {
  double p1[TILE_NNZ];
  double p2[TILE_NNZ];
  long long rp[TILE_ROWS + 1];
  double red[2 * (TG / 32)];
};

// Barrier over this worker group's TG threads (named barrier id >= 1).
__device__ __forceinline__ void group_bar(int id) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(TG) : "memory");
}

// Optional fused epilogue of pass T (persistent engine): column scores
// eps_j = s_j^2 / gamma_j, Philox keys and the level-1 histogram, and the
// V = ||v||^2 partial, computed as each column sum is produced (the ALU work of
// the keys overlaps the pass's memory traffic, and s, v are not re-read).
struct ColKeyEpi {
  const double* gamma;
  unsigned long long* keys;
  unsigned int* hist;      // shared-memory level-1 histogram of this CTA
  long long k;
  unsigned long long seed;
  int pending;
  int greedy;
};

__device__ __forceinline__ void colkey_epilogue(const ColKeyEpi* ep, int j, double sj, double vj,
                                                double& Vp, double& Emax) {
  if (ep->pending) Vp += vj * vj;
  const double g = ep->gamma[j];
  const double eps = g > 0.0 ? __ddiv_rn(__dmul_rn(sj, sj), g) : 0.0;
  Emax = fmax(Emax, eps);
  const unsigned long long key = sel_key(eps, (unsigned long long)j, ep->k, 0u, ep->seed, ep->greedy);
  ep->keys[j] = key;
  atomicAdd(&ep->hist[key >> L1_SHIFT], 1u);
}

__device__ void csr_tiles(int gid, int ngroups, int lt, int bar_id, TileSmem* sm,
                          const long long* __restrict__ ptr, const int* __restrict__ idx,
                          const double* __restrict__ val, const int* __restrict__ tiles,
                          int ntiles, const double* __restrict__ in1,
                          const double* __restrict__ in2, int use2,
                          const double* __restrict__ b, double* __restrict__ o1,
                          double* __restrict__ o2, double& Wp, double& Yp,
                          const ColKeyEpi* ep = nullptr, int acc1 = 0, int vec = 1) {
  for (int t = gid; t < ntiles; t += ngroups) {
    const int r0 = tiles[t], r1 = tiles[t + 1];
    const int nr = r1 - r0;
    for (int i = lt; i <= nr; i += TG) sm->rp[i] = ptr[r0 + i];
    group_bar(bar_id);
    const long long p0 = sm->rp[0], p1 = sm->rp[nr];
    if (p1 - p0 > TILE_NNZ) {                      // one long row: group-wide reduction
      double a1 = 0.0, a2 = 0.0;
      for (long long p = p0 + lt; p < p1; p += TG) {
        const double a = ld_stream(val + p);
        const int c = __ldg(idx + p);
        a1 = fma(a, __ldg(in1 + c), a1);
        if (use2) a2 = fma(a, __ldg(in2 + c), a2);
      }
      a1 = warp_sum(a1);
      a2 = warp_sum(a2);
      if ((lt & 31) == 0) { sm->red[2 * (lt >> 5)] = a1; sm->red[2 * (lt >> 5) + 1] = a2; }
      group_bar(bar_id);
      if (lt == 0) {
        double s1 = 0.0, s2 = 0.0;
        for (int q = 0; q < TG / 32; ++q) { s1 += sm->red[2 * q]; s2 += sm->red[2 * q + 1]; }
        o1[r0] = s1;
        o2[r0] = s2;
        if (b) {
          const double y = b[r0] - s2;
          Wp += s1 * s1;
          Yp += y * y;
        }
        if (ep) colkey_epilogue(ep, r0, s1, s2, Wp, Yp);
        if (acc1) Wp += s1 * s1;
      }
      group_bar(bar_id);
      continue;
    }
    const int nz = (int)(p1 - p0);
    // sub-rounds of SUB entries per thread, each in two phases (all values /
    // indices first, then all gathers), so SUB independent chains are in flight
    constexpr int SUB = 4;
    for (int e0 = 0; e0 < TILE_NNZ / TG; e0 += SUB) {
      double av[SUB], g1[SUB], g2[SUB];
      int ci[SUB];
#pragma unroll
      for (int e = 0; e < SUB; ++e) {
        const int q = lt + (e0 + e) * TG;
        av[e] = 0.0; ci[e] = 0;
        if (q < nz) { av[e] = ld_stream(val + p0 + q); ci[e] = __ldg(idx + p0 + q); }
      }
#pragma unroll
      for (int e = 0; e < SUB; ++e) {
        const int q = lt + (e0 + e) * TG;
        g1[e] = 0.0; g2[e] = 0.0;
        if (q < nz) {
          g1[e] = __ldg(in1 + ci[e]);
          if (use2) g2[e] = __ldg(in2 + ci[e]);
        }
      }
#pragma unroll
      for (int e = 0; e < SUB; ++e) {
        const int q = lt + (e0 + e) * TG;
        if (q < nz) { sm->p1[q] = av[e] * g1[e]; sm->p2[q] = av[e] * g2[e]; }
      }
      if (lt + (e0 + SUB) * TG >= nz) break;
    }
    group_bar(bar_id);
    // row sums: vec lanes per row (power of two, chosen from the mean row length),
    // strided partial sums then a fixed shuffle tree — deterministic; loop
    // bounds are warp-uniform so the shuffles are well defined
    const int lane = lt & 31, lw = lt >> 5;
    const int spw = 32 / vec, sub = lane / vec, sl = lane & (vec - 1);
    for (int base = lw * spw; base < nr; base += (TG / 32) * spw) {
      const int r = base + sub;
      const bool valid = r < nr;
      double s1 = 0.0, s2 = 0.0;
      if (valid) {
        const int q0 = (int)(sm->rp[r] - p0), q1 = (int)(sm->rp[r + 1] - p0);
        for (int q = q0 + sl; q < q1; q += vec) { s1 += sm->p1[q]; s2 += sm->p2[q]; }
      }
      for (int o = vec >> 1; o > 0; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o, vec);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o, vec);
      }
      if (valid && sl == 0) {
        o1[r0 + r] = s1;
        o2[r0 + r] = s2;
        if (b) {
          const double y = b[r0 + r] - s2;
          Wp += s1 * s1;
          Yp += y * y;
        }
        if (ep) colkey_epilogue(ep, r0 + r, s1, s2, Wp, Yp);
        if (acc1) Wp += s1 * s1;
      }
    }
    group_bar(bar_id);
  }
}

}  // namespace rg
