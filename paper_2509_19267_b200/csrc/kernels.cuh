// kernels.cuh — the per-iteration kernels of the fused RGDBEK schedule.
//
// Iteration body k (Alg. 1 P:112-123 with the two A-passes of
// consecutive half-steps fused):
//   pass T   : s_k = A^T z_k  and  v_{k-1} = A^T xi_{k-1}
//   n-side   : V = ||v||^2, alpha_x; eps^z = s^2/gamma; keys; L1 histogram
//   select U : levels 2,3 (+slow path)
//   mask n   : zeta = s on U, Z; x_k = x_{k-1} + alpha_x v; ||x-x*||^2
//   pass N   : w = A zeta, (A x_k); W, ||b - A x_k||^2 -> stop test
//   m-side   : z_{k+1} = z_k - (Z/W) w; r = (b - z_{k+1}) - A x_k; eps^x; keys
//   select J, mask m : xi = r on J, X
//   tail     : k++, WHILE-node condition
#pragma once
#include "select.cuh"
#include "csr_tiles.cuh"

namespace rg {

constexpr int NT = 256;          // threads per block of the vector kernels
constexpr int MAXBLK = 2048;     // cap on blocks of kernels that write per-block partials

struct TraceRec {                // == rgdbek_trace_record
  long long k, kp;
  unsigned long long hash_u;
  double Z, W;
  long long kpp;
  unsigned long long hash_j;
  double X, V, rse;
};

__device__ __forceinline__ TraceRec* trace_at(TraceRec* tr, const Scal* st, long long k) {
  if (st->trace_cap <= 0 || k < 0) return nullptr;
  return tr + (k % st->trace_cap);
}

// ---------------------------------------------------------------------------
// Dense pass T: partial column sums over a panel of rows (deterministic 2-stage).
// part[p][0][j] = sum_{i in panel p} A_ij z_i,  part[p][1][j] = sum A_ij xi_i.
// Block = TPB threads x 2 columns (one 16-byte load per row), panel = R rows.
// ---------------------------------------------------------------------------
template <int TPB>
__global__ void __launch_bounds__(TPB) k_dense_passT(const double* __restrict__ A, long long lda,
                                                    int m_loc, int n, int R,
                                                    const double* __restrict__ z,
                                                    const double* __restrict__ xi,
                                                    double* __restrict__ part, const Scal* st) {
  if (st->halted) return;
  extern __shared__ double shv[];              // [R] z, [R] xi
  const int panel = blockIdx.y;
  const int r0 = panel * R;
  const int rows = min(R, m_loc - r0);
  const int pending = st->pending;
  for (int i = threadIdx.x; i < rows; i += TPB) {
    shv[i] = z[r0 + i];
    shv[R + i] = pending ? xi[r0 + i] : 0.0;
  }
  __syncthreads();
  const int c = (blockIdx.x * TPB + threadIdx.x) * 2;
  if (c >= n) return;
  double s0 = 0.0, s1 = 0.0, v0 = 0.0, v1 = 0.0;
  const double* p = A + (long long)r0 * lda + c;
  if (c + 1 < n) {
#pragma unroll 8
    for (int i = 0; i < rows; ++i) {
      const double2 a = ld_stream2(p + (long long)i * lda);
      const double zi = shv[i], xv = shv[R + i];
      s0 = fma(a.x, zi, s0);
      s1 = fma(a.y, zi, s1);
      v0 = fma(a.x, xv, v0);
      v1 = fma(a.y, xv, v1);
    }
    double* o = part + (long long)panel * 2 * n;
    o[c] = s0; o[c + 1] = s1;
    o[n + c] = v0; o[n + c + 1] = v1;
  } else {
    for (int i = 0; i < rows; ++i) {
      const double a = ld_stream(p + (long long)i * lda);
      s0 = fma(a, shv[i], s0);
      v0 = fma(a, shv[R + i], v0);
    }
    double* o = part + (long long)panel * 2 * n;
    o[c] = s0;
    o[n + c] = v0;
  }
}

// ---------------------------------------------------------------------------
// Dense pass N: partial dots of (ROWS rows) x (one chunk of CH columns) per
// warp-unit, units dealt round-robin to all resident warps (~20 each, so the
// per-warp work is balanced to a few %).  The streaming loop has no barrier,
// fence or atomic (a __threadfence per unit invalidates L1 — CCTL.IVALL — and
// with it the cached zeta/x).  k_dense_reduceN adds the Q chunk partials in
// chunk order (deterministic) and forms w, A x, W, ||b - A x||^2.
// ---------------------------------------------------------------------------
__device__ void passN_finish(Scal* st, TraceRec* tr, double* bpart, int nblk, double* sh);

template <int ROWS>
__global__ void __launch_bounds__(NT) k_dense_passN(const double* __restrict__ A, long long lda,
                                                   int m_loc, int n, int CH, int Q,
                                                   const double* __restrict__ zeta,
                                                   const double* __restrict__ x,
                                                   double* __restrict__ npart, const Scal* st) {
  if (st->halted) return;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * NT + threadIdx.x) >> 5;
  const int nw = (gridDim.x * NT) >> 5;
  const int groups = (m_loc + ROWS - 1) / ROWS;
  const int units = groups * Q;
  for (int u = gw; u < units; u += nw) {
    const int g = u / Q, q = u - g * Q;
    const int r0 = g * ROWS;
    const int nr = min(ROWS, m_loc - r0);
    const int c0 = q * CH;
    const int c1 = min(n, c0 + CH);
    const int c1e = c0 + ((c1 - c0) & ~1);
    double sw[ROWS], sx[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) { sw[r] = 0.0; sx[r] = 0.0; }
    const double* arow = A + (long long)r0 * lda;
#pragma unroll 4
    for (int c = c0 + lane * 2; c < c1e; c += 64) {
      const double2 zc = __ldg(reinterpret_cast<const double2*>(zeta + c));
      const double2 xc = __ldg(reinterpret_cast<const double2*>(x + c));
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        if (r < nr) {
          const double2 a = ld_stream2(arow + (long long)r * lda + c);
          sw[r] = fma(a.x, zc.x, sw[r]); sw[r] = fma(a.y, zc.y, sw[r]);
          sx[r] = fma(a.x, xc.x, sx[r]); sx[r] = fma(a.y, xc.y, sx[r]);
        }
      }
    }
    if (c1e < c1 && lane == 0) {                 // odd tail column (odd n, last chunk)
      for (int r = 0; r < nr; ++r) {
        const double a = ld_stream(arow + (long long)r * lda + c1e);
        sw[r] = fma(a, zeta[c1e], sw[r]);
        sx[r] = fma(a, x[c1e], sx[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < ROWS; ++r) { sw[r] = warp_sum(sw[r]); sx[r] = warp_sum(sx[r]); }
    if (lane < 2 * nr) {
      // lane 2r holds row r's A.zeta partial, lane 2r+1 its A.x partial
      double val = 0.0;
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        if (lane == 2 * r) val = sw[r];
        if (lane == 2 * r + 1) val = sx[r];
      }
      npart[((long long)q * m_loc + r0) * 2 + lane] = val;
    }
  }
}

// Second stage of dense pass N: w_i, (A x)_i = sum over chunks in order;
// W = ||w||^2 and ||b - A x||^2 -> stop test on x_k (last block).
__global__ void __launch_bounds__(NT) k_dense_reduceN(const double* __restrict__ npart, int Q,
                                                     int m_loc, const double* __restrict__ b,
                                                     double* __restrict__ w,
                                                     double* __restrict__ ax, Scal* st,
                                                     TraceRec* tr, double* bpart) {
  if (st->halted) return;
  __shared__ double sh[NT / 32];
  double Wp = 0.0, Yp = 0.0;
  for (int i = blockIdx.x * NT + threadIdx.x; i < m_loc; i += gridDim.x * NT) {
    double tw = 0.0, tx = 0.0;
    for (int q = 0; q < Q; ++q) {
      const double2 p = __ldcg(reinterpret_cast<const double2*>(npart + ((long long)q * m_loc + i) * 2));
      tw += p.x;
      tx += p.y;
    }
    w[i] = tw;
    ax[i] = tx;
    const double y = b[i] - tx;
    Wp += tw * tw;
    Yp += y * y;
  }
  const double Wb = block_sum<NT>(Wp, sh);
  const double Yb = block_sum<NT>(Yp, sh);
  if (threadIdx.x == 0) { bpart[blockIdx.x] = Wb; bpart[MAXBLK + blockIdx.x] = Yb; }
  if (!last_block(&st->counters[C_PASSN])) return;
  passN_finish(st, tr, bpart, gridDim.x, sh);
}

// ---------------------------------------------------------------------------
// CSR dual SpMV, VEC lanes per row.  MODE 0 = pass N (A zeta, A x, with the
// W / ||b-Ax||^2 epilogue), MODE 1 = pass T over the transposed copy (CSC) or
// the CSR of a symmetric A (s = A^T z, v = A^T xi).
// ---------------------------------------------------------------------------
template <int VEC, int MODE>
__global__ void __launch_bounds__(NT) k_csr_dual(const long long* __restrict__ ptr,
                                                const int* __restrict__ idx,
                                                const double* __restrict__ val, int nrows,
                                                const double* __restrict__ in1,
                                                const double* __restrict__ in2,
                                                const double* __restrict__ b,
                                                double* __restrict__ out1, double* __restrict__ out2,
                                                Scal* st, TraceRec* tr, double* bpart) {
  if (st->halted) return;
  __shared__ double sh[NT / 32];
  constexpr int SPW = 32 / VEC;                       // rows per warp per sweep
  const int lane = threadIdx.x & (VEC - 1);
  const int sub = (threadIdx.x & 31) / VEC;
  const int gw = (blockIdx.x * NT + threadIdx.x) >> 5;
  const int nw = (gridDim.x * NT) >> 5;
  const int use2 = (MODE == 1) ? st->pending : 1;
  double Wp = 0.0, Yp = 0.0;
  for (int base = gw * SPW; base < nrows; base += nw * SPW) {   // warp-uniform trip count
    const int row = base + sub;
    const bool valid = row < nrows;
    double a1 = 0.0, a2 = 0.0;
    if (valid) {
      const long long p0 = ptr[row], p1 = ptr[row + 1];
      for (long long p = p0 + lane; p < p1; p += VEC) {
        const double a = ld_stream(val + p);
        const int c = __ldg(idx + p);
        a1 = fma(a, __ldg(in1 + c), a1);
        if (use2) a2 = fma(a, __ldg(in2 + c), a2);
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
      if (MODE == 0) {
        const double y = b[row] - a2;
        Wp += a1 * a1;
        Yp += y * y;
      }
    }
  }
  if (MODE == 1) return;
  const double Wb = block_sum<NT>(Wp, sh);
  const double Yb = block_sum<NT>(Yp, sh);
  if (threadIdx.x == 0) { bpart[blockIdx.x] = Wb; bpart[MAXBLK + blockIdx.x] = Yb; }
  if (!last_block(&st->counters[C_PASSN])) return;
  passN_finish(st, tr, bpart, gridDim.x, sh);
}

// Tiled CSR/CSC dual SpMV (csr_tiles.cuh), one 256-thread block = one worker
// group.  MODE 0 = pass N with the W / ||b - Ax||^2 epilogue, MODE 1 = pass T.
__device__ void passN_finish(Scal* st, TraceRec* tr, double* bpart, int nblk, double* sh);

template <int MODE>
__global__ void __launch_bounds__(NT) k_csr_tiles(const long long* __restrict__ ptr,
                                                 const int* __restrict__ idx,
                                                 const double* __restrict__ val,
                                                 const int* __restrict__ tiles,
                                                 const long long* __restrict__ tilep, int ntiles,
                                                 const double* in1, const double* in2,
                                                 const double* __restrict__ b,
                                                 double* __restrict__ o1, double* __restrict__ o2,
                                                 Scal* st, TraceRec* tr, double* bpart,
                                                 int vec) {
  if (st->halted) return;
  constexpr int GPB = NT / TG;                    // worker groups per block
  extern __shared__ __align__(16) unsigned char tsm_raw[];
  const int g = threadIdx.x / TG;
  TileSmemT<GRAPH_TBUF>* sm = reinterpret_cast<TileSmemT<GRAPH_TBUF>*>(tsm_raw) + g;
  __shared__ double sh[NT / 32];
  __shared__ __align__(8) unsigned long long tbar[GPB * 2 * GRAPH_TBUF];
  tile_rings_init<GRAPH_TBUF>(tbar);
  TileRing ring{tbar + g * 2 * GRAPH_TBUF, 0u};
  const int use2 = (MODE == 1) ? st->pending : 1;
  double Wp = 0.0, Yp = 0.0;
  csr_tiles<GRAPH_TBUF>(blockIdx.x * GPB + g, gridDim.x * GPB, threadIdx.x % TG, 1 + g, sm, ring, ptr, idx,
            val, tiles, tilep, ntiles, in1, in2, use2, MODE == 0 ? b : nullptr, o1, o2, Wp, Yp,
            nullptr, 0, vec, MODE == 0 ? RG_REV_N : 0);
  if (MODE == 1) return;
  const double Wb = block_sum<NT>(Wp, sh);
  const double Yb = block_sum<NT>(Yp, sh);
  if (threadIdx.x == 0) { bpart[blockIdx.x] = Wb; bpart[MAXBLK + blockIdx.x] = Yb; }
  if (!last_block(&st->counters[C_PASSN])) return;
  passN_finish(st, tr, bpart, gridDim.x, sh);
}

// Stop test on x_k (reading R12), given the global W and ||b - A x_k||^2.
__device__ void passN_decide(Scal* st, TraceRec* tr, double W, double Y) {
  st->W = W;
  st->Y = Y;
  const long long k = st->k;
  const double rse = Y / st->bnorm2;
  const double rel = st->has_ref ? sqrt(st->relerr2 / st->xsnorm2) : __longlong_as_double(0x7FF8000000000000ll);
  if (TraceRec* t = trace_at(tr, st, k)) t->W = W;
  if (k >= 1) {
    if (TraceRec* t = trace_at(tr, st, k - 1)) t->rse = rse;
  }
  int halt = 0, outcome = RGDBEK_MAX_ITER;
  if (k > st->k_begin) {
    if (st->stop_mode == RGDBEK_STOP_RSE && rse <= st->tol) { halt = 1; outcome = RGDBEK_CONVERGED; }
    else if (st->stop_mode == RGDBEK_STOP_REL_ERR && rel <= st->tol) { halt = 1; outcome = RGDBEK_CONVERGED; }
    else if (st->kp_prev == 0 && st->kpp_prev == 0) { halt = 1; outcome = RGDBEK_STALLED; }
  }
  if (!halt && (k > st->k_begin || st->k_end == st->k_begin) && k >= st->k_end) {
    halt = 1; outcome = RGDBEK_MAX_ITER;
  }
  if (halt) {
    st->halted = 1;
    st->outcome = outcome;
    st->iters = k;
    st->rse_out = rse;
    st->relerr_out = rel;
  }
}

// Run by the last block of pass N: single GPU -> stop test now; row-sharded ->
// publish this rank's partials for the NCCL allreduce (k_passN_decide follows).
__device__ void passN_finish(Scal* st, TraceRec* tr, double* bpart, int nblk, double* sh) {
  const double W = reduce_partials<NT>(bpart, nblk, sh);
  const double Y = reduce_partials<NT>(bpart + MAXBLK, nblk, sh);
  if (threadIdx.x != 0) return;
  if (st->dist) {
    st->wy[0] = W;
    st->wy[1] = Y;
    return;
  }
  passN_decide(st, tr, W, Y);
}

__global__ void k_passN_decide(Scal* st, TraceRec* tr) {
  if (st->halted) return;
  passN_decide(st, tr, st->wy[0], st->wy[1]);
}

// ---------------------------------------------------------------------------
// n-side: finish s, v (sum of dense panel partials, or read them), V and
// alpha_x, column scores eps^z_j = s_j^2/gamma_j, keys, L1 histogram.
// ---------------------------------------------------------------------------
// Dense pass T second stage: s_j = sum_p part[p][0][j], v_j likewise, in a
// fixed order (8 panel groups per column, then the 8 group sums in order).
__global__ void __launch_bounds__(NT) k_dense_reduceT(const double* __restrict__ part, int P, int n,
                                                     double* __restrict__ s,
                                                     double* __restrict__ v, const Scal* st) {
  if (st->halted) return;
  __shared__ double rs[8][33], rv[8][33];
  const int c = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + c;
  const int pending = st->pending;
  double a = 0.0, bb = 0.0;
  if (j < n) {
    for (int p = g; p < P; p += 8) {
      const double* q = part + (long long)p * 2 * n + j;
      a += __ldcg(q);
      if (pending) bb += __ldcg(q + n);
    }
  }
  rs[g][c] = a;
  rv[g][c] = bb;
  __syncthreads();
  if (g == 0 && j < n) {
    double ta = 0.0, tb = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) { ta += rs[q][c]; tb += rv[q][c]; }
    s[j] = ta;
    v[j] = tb;
  }
}

__global__ void __launch_bounds__(NT) k_nside(int n, const double* __restrict__ s,
                                             const double* __restrict__ v,
                                             const double* __restrict__ xslot,
                                             const double* __restrict__ gamma,
                                             unsigned long long* __restrict__ keys, Scal* st,
                                             TraceRec* tr, unsigned int* gh, double* bpart,
                                             unsigned int* spec) {
  if (st->halted) return;
  __shared__ __align__(16) unsigned int h[NBINS];
  __shared__ double sh[NT / 32];
  const int pred = st->spec_pred[0];
  for (int b = threadIdx.x; b < NBINS; b += NT) h[b] = 0u;
  __syncthreads();
  const int pending = st->pending;
  const long long k = st->k;
  const unsigned long long seed = st->seed;
  double Vp = 0.0;
  for (int j = blockIdx.x * NT + threadIdx.x; j < n; j += gridDim.x * NT) {
    const double sj = s[j];
    if (pending) {
      const double vj = v[j];
      Vp += vj * vj;
    }
    const double g = gamma[j];
    const double eps = g > 0.0 ? __ddiv_rn(__dmul_rn(sj, sj), g) : 0.0;
    const unsigned long long key = make_key(eps, (unsigned long long)j, k, 0u, seed);
    keys[j] = key;
    atomicAdd(&h[key >> L1_SHIFT], 1u);
    if ((int)(key >> L1_SHIFT) == pred) atomicAdd(&spec[(key >> L2_SHIFT) & 0xFFFull], 1u);
  }
  __syncthreads();
  flush_hist<NT>(h, gh, NBINS);
  const double Vb = block_sum<NT>(Vp, sh);
  if (threadIdx.x == 0) bpart[blockIdx.x] = Vb;
  if (!last_block(&st->counters[C_NSIDE])) return;
  const double V = reduce_partials<NT>(bpart, gridDim.x, sh);
  if (threadIdx.x == 0) {
    st->V = V;
    const int dox = pending && st->kpp_prev > 0 && V > 0.0;
    st->do_x = dox;
    const double X = *xslot;                 // global ||xi||^2 (allreduced when sharded)
    st->X = X;
    st->alpha_x = dox ? __ddiv_rn(X, V) : 0.0;
    if (pending) {
      if (TraceRec* t = trace_at(tr, st, k - 1)) { t->V = V; t->X = X; }
    }
  }
  finalize_level1<NT>(&st->seln, gh, n, st->kc);
  spec_decide<NT>(&st->seln, &st->spec_pred[0], spec);
}

// ---------------------------------------------------------------------------
// mask n: zeta = s on U; Z, |U|, hash(U); x_k = x_{k-1} + alpha_x v; ||x - x*||^2
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) k_mask_n(const unsigned long long* __restrict__ keys,
                                              const double* __restrict__ s,
                                              const double* __restrict__ v,
                                              double* __restrict__ zeta, double* __restrict__ x,
                                              const double* __restrict__ xstar,
                                              unsigned char* __restrict__ selmask, int n, Scal* st,
                                              TraceRec* tr, double* bpart) {
  if (st->halted) return;
  __shared__ double sh[NT / 32];
  const SelState ss = st->seln;
  const int dox = st->do_x, has_ref = st->has_ref;
  if (selmask) selmask += (st->k & 1) * (long long)n;          // parity of k (get_blocks)
  const double ax = st->alpha_x;
  double Zp = 0.0, Rp = 0.0;
  long long cnt = 0;
  unsigned long long hs = 0ull;
  for (int j = blockIdx.x * NT + threadIdx.x; j < n; j += gridDim.x * NT) {
    const double sj = s[j];
    const bool sel = is_selected(ss, keys[j], j);
    zeta[j] = sel ? sj : 0.0;
    if (sel) {
      Zp += sj * sj;
      cnt += 1;
      hs += splitmix64((unsigned long long)j);
    }
    if (selmask) selmask[j] = sel ? 1 : 0;
    double xj = x[j];
    if (dox) {
      xj = __dadd_rn(xj, __dmul_rn(ax, v[j]));
      x[j] = xj;
    }
    if (has_ref) {
      const double d = xj - xstar[j];
      Rp += d * d;
    }
  }
  cnt = warp_sum_ll(cnt);
  hs = warp_sum_u64(hs);
  if ((threadIdx.x & 31) == 0 && (cnt || hs)) {
    atomicAdd((unsigned long long*)&st->cnt_acc, (unsigned long long)cnt);
    atomicAdd(&st->hash_acc, hs);
  }
  const double Zb = block_sum<NT>(Zp, sh);
  const double Rb = block_sum<NT>(Rp, sh);
  if (threadIdx.x == 0) { bpart[blockIdx.x] = Zb; bpart[MAXBLK + blockIdx.x] = Rb; }
  if (!last_block(&st->counters[C_MASKN])) return;
  const double Z = reduce_partials<NT>(bpart, gridDim.x, sh);
  const double R = reduce_partials<NT>(bpart + MAXBLK, gridDim.x, sh);
  if (threadIdx.x == 0) {
    const long long kp = __ldcg(&st->cnt_acc);
    const unsigned long long hu = __ldcg(&st->hash_acc);
    st->cnt_acc = 0;
    st->hash_acc = 0ull;
    if (kp != (ss.mode == SEL_NONE ? 0 : ss.target)) st->error |= 1;
    st->Z = Z;
    st->kp = kp;
    st->hashU = hu;
    st->relerr2 = R;
    st->pending = 0;
    if (TraceRec* t = trace_at(tr, st, st->k)) {
      t->k = st->k; t->kp = kp; t->hash_u = hu; t->Z = Z;
    }
  }
}

// ---------------------------------------------------------------------------
// m-side: z_{k+1} = z_k - (Z/W) w (reading R1); r = (b - z_{k+1}) - A x_k
// (reading R8); eps^x = r^2 / rho; keys; L1 histogram.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) k_mside(int m_loc, long long row0, double* __restrict__ z,
                                             const double* __restrict__ w,
                                             const double* __restrict__ ax,
                                             const double* __restrict__ b,
                                             const double* __restrict__ rho,
                                             double* __restrict__ r,
                                             unsigned long long* __restrict__ keys, Scal* st,
                                             unsigned int* gh, unsigned int* spec) {
  if (st->halted) return;
  __shared__ __align__(16) unsigned int h[NBINS];
  const int pred = spec ? st->spec_pred[1] : -2;   // no speculation when sharded (spec null)
  for (int q = threadIdx.x; q < NBINS; q += NT) h[q] = 0u;
  __syncthreads();
  const int doz = st->kp > 0 && st->W > 0.0;
  const double az = doz ? __ddiv_rn(st->Z, st->W) : 0.0;
  const long long k = st->k;
  const unsigned long long seed = st->seed;
  for (int i = blockIdx.x * NT + threadIdx.x; i < m_loc; i += gridDim.x * NT) {
    double zi = z[i];
    if (doz) {
      zi = __dsub_rn(zi, __dmul_rn(az, w[i]));
      z[i] = zi;
    }
    const double ri = __dsub_rn(__dsub_rn(b[i], zi), ax[i]);
    r[i] = ri;
    const double p = rho[i];
    const double eps = p > 0.0 ? __ddiv_rn(__dmul_rn(ri, ri), p) : 0.0;
    const unsigned long long key = make_key(eps, (unsigned long long)(row0 + i), k, 1u, seed);
    keys[i] = key;
    atomicAdd(&h[key >> L1_SHIFT], 1u);
    if ((int)(key >> L1_SHIFT) == pred) atomicAdd(&spec[(key >> L2_SHIFT) & 0xFFFull], 1u);
  }
  __syncthreads();
  flush_hist<NT>(h, gh, NBINS);
  if (st->dist) return;                      // histogram is allreduced, then k_sel_fin
  if (!last_block(&st->counters[C_MSIDE])) return;
  finalize_level1<NT>(&st->selm, gh, m_loc, st->kr);
  spec_decide<NT>(&st->selm, &st->spec_pred[1], spec);
}

// ---------------------------------------------------------------------------
// mask m: xi = r on J; X, |J|, hash(J); x-update becomes pending.
// ---------------------------------------------------------------------------
__device__ void maskm_finish(Scal* st, TraceRec* tr, long long kpp, unsigned long long hj) {
  const SelState& ss = st->selm;
  if (kpp != (ss.mode == SEL_NONE ? 0 : ss.target)) st->error |= 2;
  st->kpp = kpp;
  st->hashJ = hj;
  st->kp_prev = st->kp;
  st->kpp_prev = kpp;
  st->pending = 1;
  if (TraceRec* t = trace_at(tr, st, st->k)) { t->kpp = kpp; t->hash_j = hj; }
}

__global__ void __launch_bounds__(NT) k_mask_m(const unsigned long long* __restrict__ keys,
                                              const double* __restrict__ r,
                                              double* __restrict__ xi,
                                              unsigned char* __restrict__ selmask, int m_loc,
                                              long long row0, Scal* st, TraceRec* tr,
                                              double* bpart, double* xslot) {
  if (st->halted) return;
  __shared__ double sh[NT / 32];
  const SelState ss = st->selm;
  double Xp = 0.0;
  long long cnt = 0;
  unsigned long long hs = 0ull;
  if (selmask) selmask += (st->k & 1) * (long long)m_loc;      // parity of k (get_blocks)
  // 4 rows in flight per thread (independent loads), visited in the same order
  const long long stride = (long long)gridDim.x * NT;
  for (long long i0 = (long long)blockIdx.x * NT + threadIdx.x; i0 < m_loc; i0 += 4 * stride) {
    unsigned long long kk[4];
    double rr[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + u * stride;
      kk[u] = i < m_loc ? keys[i] : 0ull;
      rr[u] = i < m_loc ? r[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + u * stride;
      if (i >= m_loc) break;
      const long long gi = row0 + i;
      const bool sel = is_selected(ss, kk[u], gi);
      const double ri = rr[u];
      xi[i] = sel ? ri : 0.0;
      if (sel) {
        Xp += ri * ri;
        cnt += 1;
        hs += splitmix64((unsigned long long)gi);
      }
      if (selmask) selmask[i] = sel ? 1 : 0;
    }
  }
  cnt = warp_sum_ll(cnt);
  hs = warp_sum_u64(hs);
  if ((threadIdx.x & 31) == 0 && (cnt || hs)) {
    atomicAdd((unsigned long long*)&st->cnt_acc, (unsigned long long)cnt);
    atomicAdd(&st->hash_acc, hs);
  }
  const double Xb = block_sum<NT>(Xp, sh);
  if (threadIdx.x == 0) bpart[blockIdx.x] = Xb;
  if (!last_block(&st->counters[C_MASKM])) return;
  const double X = reduce_partials<NT>(bpart, gridDim.x, sh);
  if (threadIdx.x == 0) {
    const long long kpp = __ldcg(&st->cnt_acc);
    const unsigned long long hj = __ldcg(&st->hash_acc);
    st->cnt_acc = 0;
    st->hash_acc = 0ull;
    *xslot = X;            // rides in the next pass-T allreduce [s | v | X] when sharded
    if (st->dist) {        // |J|, hash(J) of this rank: allreduced, then k_maskm_finish
      st->jacc[0] = (unsigned long long)kpp;
      st->jacc[1] = hj;
      return;
    }
    maskm_finish(st, tr, kpp, hj);
  }
}

__global__ void k_maskm_finish(Scal* st, TraceRec* tr) {
  if (st->halted) return;
  maskm_finish(st, tr, (long long)st->jacc[0], st->jacc[1]);
}

// ---------------------------------------------------------------------------
// tail: k++ unless halted; drive the graph's WHILE node.
// ---------------------------------------------------------------------------
__global__ void k_tail(Scal* st, cudaGraphConditionalHandle h, int use_cond) {
  const int halted = st->halted;
  if (!halted) st->k += 1;
  if (use_cond) cudaGraphSetConditional(h, halted ? 0u : 1u);
}

// Timing hook (rgdbek_launch_kernel): pass T runs its second product too.
__global__ void k_set_pending(Scal* st) { st->pending = 1; }

// Call prologue: arm the stop test for this call.
__global__ void k_call_begin(Scal* st, long long n_or_max, int is_step, double tol, int stop_mode) {
  st->k_begin = st->k;
  st->k_end = is_step ? st->k + n_or_max : n_or_max;
  st->tol = tol;
  st->stop_mode = stop_mode;
  st->halted = 0;
  st->outcome = RGDBEK_MAX_ITER;
  st->iters = st->k;
}

// reset(seed): x = 0, z = b, k = 0
__global__ void k_reset_vecs(double* x, int n, double* z, const double* b, int m_loc) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long str = (long long)gridDim.x * blockDim.x;
  for (long long j = t; j < n; j += str) x[j] = 0.0;
  for (long long i = t; i < m_loc; i += str) z[i] = b[i];
}
// multi-RHS reset: x = 0 ([n][nr]), z = b ([m][nr], interleaved)
__global__ void k_reset_multi(double* x, long long nx, double* z, const double* b, long long nz) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long str = (long long)gridDim.x * blockDim.x;
  for (long long j = t; j < nx; j += str) x[j] = 0.0;
  for (long long i = t; i < nz; i += str) z[i] = b[i];
}
// [nr][len] <-> [len][nr]
__global__ void k_interleave(const double* src, double* dst, long long len, int nr, int to_inter) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < len * nr;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / nr, q = e - i * nr;       // dst/src index e = i * nr + q
    if (to_inter) dst[e] = src[q * len + i];
    else dst[q * len + i] = src[e];
  }
}

__global__ void k_reset_scal(Scal* st, unsigned long long seed, long long k) {
  st->k = k;
  st->k_begin = k;
  st->k_end = k;
  st->seed = seed;
  st->halted = 0;
  st->pending = 0;
  st->do_x = 0;
  st->kp = st->kpp = -1;
  st->kp_prev = st->kpp_prev = -1;
  st->X = st->V = st->Z = st->W = st->Y = 0.0;
  st->alpha_x = 0.0;
  st->cnt_acc = 0;
  st->hash_acc = 0ull;
  st->error = 0;
  st->npass = 0;
  st->abytes = 0.0;
  st->seln.mode = SEL_NONE;
  st->selm.mode = SEL_NONE;
  st->seln.ncand = st->selm.ncand = 0u;
  for (int c = 0; c < C_NUM; ++c) st->counters[c] = 0u;
}

}  // namespace rg
