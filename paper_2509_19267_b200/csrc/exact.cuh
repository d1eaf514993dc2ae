// exact.cuh — exact-projection mode: Algorithm 1 with its pseudoinverse
// updates, SURVEY §8(f) NEXT #1.
//
//   z_{k+1} = z_k - A_U A_U^+ z_k
//   x_{k+1} = x_k + (A^J)^+ (b^J - z^J_{k+1} - A^J x_k)
//
// The paper solves both subproblems with LSQR (Remark 2).  Here the
// two Krylov solvers mathematically equivalent to LSQR on them are used
// (reading R1b): CGLS — LSQR's mathematical equivalent — on both least-squares
// subproblems from y = 0: min_y ||A_U y - z_k|| (its residual z_k - A_U y is
// z_{k+1}; its first iterate is the pseudoinverse-free z-step) and
// min_y ||A^J y - r^J|| (from y = 0 its iterates stay in range(A^J^T), so the
// limit is the minimum-norm solution (A^J)^+ r^J for fat or tall A^J alike).
// Each runs until its normal-equation residual ||A^T (.)|| has dropped by
// inner_tol relative to the start, or inner_max iterations.  Every inner
// iteration is one full pass over A of each kind; block selection, keys and
// the stop test are those of the pseudoinverse-free engine.
//
// Iteration k (all phases of one persistent cooperative kernel):
//   column step: s = A^T z; keys; U; CGLS { q = A p; z -= (gamma/|q|^2) q;
//                s' = A^T z; gamma' = |s'_U|^2; p = s'_U + (gamma'/gamma) p }
//   row step:    r = b - z - A x; keys; J; CGLS { u = A p; x += (gamma/|u_J|^2) p;
//                r_J -= alpha u_J; t = A^T r_J; p = t + (gamma'/gamma) p }
//   end:         A x_{k+1} -> RSE -> stop test (A x_{k+1} is reused by the next row step)
#pragma once
#include "persistent.cuh"

namespace rg {

#ifndef RG_EX_MASK
#define RG_EX_MASK 1        // dense x-solve passes read only the rows of A^J
#endif

struct EArgs {
  double inner_tol;
  int inner_max;
  double bytesT, bytesN;   // algorithmic bytes of one full pass T / pass N over A
  double* px;      // Craig search direction (n)
  double* u;       // A px (m_loc)
};

// Sum over the G CTA column partials written by p_dense_passT (CTA-parallel,
// coalesced, fixed order), for all columns: o1 (and o2 when use2).
__device__ void ex_dense_colreduce(const PArgs& a, int use2, double* o1, double* o2, double* red) {
  constexpr int CW = 64, NG = PT / CW;
  const int G = gridDim.x, n = a.n;
  const int cpb = (n + G - 1) / G;
  const int c0 = min(n, blockIdx.x * cpb), c1 = min(n, c0 + cpb);
  const int cl = threadIdx.x % CW, g = threadIdx.x / CW;
  for (int cb = c0; cb < c1; cb += CW) {
    const int j = cb + cl;
    double sj = 0.0, vj = 0.0;
    if (j < c1) {
      for (int p = g; p < G; p += NG) {
        const double* q = a.part + (long long)p * 2 * n + j;
        sj += __ldcg(q);
        if (use2) vj += __ldcg(q + n);
      }
    }
    red[g * CW + cl] = sj;
    red[(NG + g) * CW + cl] = vj;
    __syncthreads();
    if (g == 0 && j < c1) {
      double ts = 0.0, tv = 0.0;
#pragma unroll
      for (int q = 0; q < NG; ++q) { ts += red[q * CW + cl]; tv += red[(NG + q) * CW + cl]; }
      o1[j] = ts;
      if (use2) o2[j] = tv;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Row-masked dense passes (the x-solve of the exact mode works on A^J only): rows outside
// the row block J are not read at all, so an inner iteration of the x-solve streams
// |J| / m of A instead of all of it.  Rows keep their order (a CTA compacts the selected
// rows of each chunk by a block-wide prefix count), so the sums are deterministic.
// ---------------------------------------------------------------------------
// Selected rows of [r0, r0 + rows) in order -> rid[0..cnt); returns cnt (all threads).
__device__ int ex_compact_rows(const PArgs& a, const PSel* rs, int r0, int rows, int* rid, int* wsum) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int total = 0;
  for (int b0 = 0; b0 < rows; b0 += PT) {
    const int i = b0 + threadIdx.x;
    const bool sel = i < rows && p_selected(rs, a.keys_m[r0 + i], a.row0 + r0 + i);
    const unsigned bal = __ballot_sync(0xffffffffu, sel);
    __syncthreads();
    if (lane == 0) wsum[w] = __popc(bal);
    __syncthreads();
    int before = total;
    for (int q = 0; q < w; ++q) before += wsum[q];
    if (sel) rid[before + __popc(bal & ((1u << lane) - 1u))] = r0 + i;
    int t = 0;
    for (int q = 0; q < PW; ++q) t += wsum[q];
    total += t;
  }
  __syncthreads();
  return total;
}

// part[cta] = A^T in1 restricted to the selected rows of this CTA's row range.
__device__ void ex_dense_passT_rows(const PArgs& a, const PSel* rs, const double* in1, double* smem) {
  const int G = gridDim.x, bb = blockIdx.x;
  const int rb = (int)((long long)a.m_loc * bb / G), re = (int)((long long)a.m_loc * (bb + 1) / G);
  const int ntiles = (a.n + 2 * PT - 1) / (2 * PT);
  double* zs = smem;                                         // [ZCH] values
  int* rid = reinterpret_cast<int*>(smem + ZCH);             // [ZCH] row ids
  int* wsum = rid + ZCH;                                     // [PW]
  double* out = a.part + (long long)bb * 2 * a.n;
  for (int t = 0; t < ntiles; ++t) {
    const int c = t * 2 * PT + 2 * threadIdx.x;
    double s0 = 0.0, s1 = 0.0;
    for (int rc = rb; rc < re; rc += ZCH) {
      const int rows = min(ZCH, re - rc);
      __syncthreads();
      const int cnt = ex_compact_rows(a, rs, rc, rows, rid, wsum);
      for (int i = threadIdx.x; i < cnt; i += PT) zs[i] = in1[rid[i]];
      __syncthreads();
      if (c + 1 < a.n) {
#pragma unroll 8
        for (int i = 0; i < cnt; ++i) {
          const double2 av = ld_stream2(a.A + (long long)rid[i] * a.lda + c);
          s0 = fma(av.x, zs[i], s0);
          s1 = fma(av.y, zs[i], s1);
        }
      } else if (c < a.n) {
        for (int i = 0; i < cnt; ++i) s0 = fma(ld_stream(a.A + (long long)rid[i] * a.lda + c), zs[i], s0);
      }
    }
    if (c + 1 < a.n) { out[c] = s0; out[c + 1] = s1; }
    else if (c < a.n) out[c] = s0;
  }
}

// out1 = A in1 on the selected rows of this CTA's row range (other rows untouched); one
// warp per selected row, columns strided, fixed shuffle tree.  Returns nothing: the
// caller forms its sums over J from out1.
__device__ void ex_dense_passN_rows(const PArgs& a, const PSel* rs, const double* in1, double* out1,
                                    double* smem) {
  const int G = gridDim.x, bb = blockIdx.x;
  const int rb = (int)((long long)a.m_loc * bb / G), re = (int)((long long)a.m_loc * (bb + 1) / G);
  int* rid = reinterpret_cast<int*>(smem);
  int* wsum = rid + ZCH;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int rc = rb; rc < re; rc += ZCH) {
    const int rows = min(ZCH, re - rc);
    __syncthreads();
    const int cnt = ex_compact_rows(a, rs, rc, rows, rid, wsum);
    for (int u = wid; u < cnt; u += PW) {
      const double* ar = a.A + (long long)rid[u] * a.lda;
      double acc = 0.0;
      int c = lane * 2;
      for (; c + 192 < a.n - 1; c += 256) {
        double2 v[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) v[g] = ld_stream2(ar + c + 64 * g);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const double2 p = *reinterpret_cast<const double2*>(in1 + c + 64 * g);
          acc = fma(v[g].x, p.x, acc);
          acc = fma(v[g].y, p.y, acc);
        }
      }
      for (; c + 1 < a.n; c += 64) {
        const double2 v = ld_stream2(ar + c);
        const double2 p = *reinterpret_cast<const double2*>(in1 + c);
        acc = fma(v.x, p.x, acc);
        acc = fma(v.y, p.y, acc);
      }
      if (c < a.n) acc = fma(ld_stream(ar + c), in1[c], acc);
      acc = warp_sum(acc);
      if (lane == 0) out1[rid[u]] = acc;
    }
  }
  __syncthreads();
}

// o1 = A^T in1 (and o2 = A^T in2 when use2) over all columns; ends after a grid barrier.
template <bool DENSE>
__device__ void ex_passT(const PArgs& a, TileRing& ring, const double* in1, const double* in2, int use2,
                         double* o1, double* o2, double* dyn, unsigned int& bgen) {
  if constexpr (DENSE) {
    p_dense_passT(a, use2, dyn, in1, in2);
    grid_sync(a.bar, bgen);
    ex_dense_colreduce(a, use2, o1, o2, dyn);
  } else {
    double d1 = 0.0, d2 = 0.0;
    const int g = threadIdx.x / TG;
    csr_tiles(blockIdx.x * (PT / TG) + g, gridDim.x * (PT / TG), threadIdx.x % TG, 1 + g,
              reinterpret_cast<TileSmem*>(dyn) + g, ring, a.cp, a.ri, a.rv, a.tilesT, a.tilepT,
              a.ntilesT, in1,
              in2, use2, nullptr, o1, o2, d1, d2, nullptr, 0, a.vecT);
  }
  grid_sync(a.bar, bgen);
}

// o1 = A in1, o2 = A in2 over this rank's rows.  W += o1^2; Y += (b - o2)^2 if b else o2^2.
// No barrier at the end (the caller publishes W / Y partials first).
template <bool DENSE>
__device__ void ex_passN(const PArgs& a, TileRing& ring, const double* in1, const double* in2, double* o1,
                         double* o2, const double* bvec, double& Wp, double& Yp, double* dyn) {
  if constexpr (DENSE) {
    p_dense_passN(a, dyn, Wp, Yp, in1, in2, o1, o2, bvec, bvec != nullptr);
  } else {
    const int g = threadIdx.x / TG;
    csr_tiles(blockIdx.x * (PT / TG) + g, gridDim.x * (PT / TG), threadIdx.x % TG, 1 + g,
              reinterpret_cast<TileSmem*>(dyn) + g, ring, a.rp, a.ci, a.cv, a.tilesN, a.tilepN,
              a.ntilesN, in1,
              in2, 1, bvec, o1, o2, Wp, Yp, nullptr, bvec ? 0 : 1, a.vecN, RG_REV_N);
  }
}

// Publish two per-CTA partials, barrier, return both global sums (same in every CTA).
__device__ __forceinline__ void ex_allsum2(const PArgs& a, double p1, double p2, int slot1,
                                           int slot2, double* sh, unsigned int& bgen, double& s1,
                                           double& s2) {
  const int G = gridDim.x;
  const double b1 = pblock_sum(p1, sh);
  const double b2 = pblock_sum(p2, sh);
  if (threadIdx.x == 0) { a.bpart[slot1 * G + blockIdx.x] = b1; a.bpart[slot2 * G + blockIdx.x] = b2; }
  grid_sync(a.bar, bgen);
  s1 = slot_sum(a.bpart, slot1, sh);
  s2 = slot_sum(a.bpart, slot2, sh);
}

template <bool DENSE>
__global__ void __launch_bounds__(PT, 1) k_persistent_exact(PArgs a, EArgs e) {
  __shared__ __align__(16) unsigned int h[NBINS];
  __shared__ __align__(8) unsigned long long tbar[(PT / TG) * TRING];
  __shared__ double sh[PW];
  __shared__ unsigned int sh_u[4];
  __shared__ long long sh_l[40];
  __shared__ PSel ps;
  extern __shared__ __align__(16) double dyn[];
  TileRing ring{tbar + (threadIdx.x / TG) * TRING, 0u};
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
  const double bnorm2 = st->bnorm2, xsnorm2 = st->xsnorm2;
  const long long kc = st->kc, kr = st->kr;
  const int n = a.n, m_loc = a.m_loc;
  unsigned int* hn = a.hist;
  unsigned int* hm = a.hist + 3 * NBINS;
  Cand* cn = a.cand;
  Cand* cm = a.cand + CAND_CAP;
  const double tol2 = e.inner_tol * e.inner_tol;
  unsigned int bgen = 0;
  if (threadIdx.x == 0) bgen = ld_acquire_u32(&a.bar->gen);
  long long npass = 0;                       // passes over A in this launch
  // algorithmic bytes of A read in this launch: a full pass reads all of A, a row-masked
  // dense x-solve pass only the |J| selected rows
  double abytes = 0.0;

  // ---- prologue: A x_k (the first row step's residual and the RSE of x_k) ----
  double Yk;
  {
    double Wd = 0.0, Yp = 0.0;
    ++npass;
    abytes += e.bytesN;
    ex_passN<DENSE>(a, ring, a.x, a.x, e.u, a.ax, a.b, Wd, Yp, dyn);
    double Wsum;
    ex_allsum2(a, Wd, Yp, SL_W, SL_Y, sh, bgen, Wsum, Yk);
  }
  if (k_end == k_begin) {
    if (lead) {
      const double rse = Yk / bnorm2;
      st->halted = 1; st->outcome = RGDBEK_MAX_ITER; st->iters = k; st->rse_out = rse;
      st->relerr_out = __longlong_as_double(0x7FF8000000000000ll);
      st->npass += npass;
      st->abytes += abytes;
    }
    return;
  }

  for (;;) {
    // ======================= column step =======================
    for (int i = threadIdx.x; i < NBINS; i += PT) h[i] = 0u;
    __syncthreads();
    ++npass;
    abytes += e.bytesT;
    ex_passT<DENSE>(a, ring, a.z, a.z, 0, a.s, a.v, dyn, bgen);                 // s = A^T z_k
    p_zero_side(a, 1);
    double Emax = 0.0;
    for (int j = blockIdx.x * PT + threadIdx.x; j < n; j += G * PT) {
      const double sj = a.s[j];
      const double gm = a.gamma[j];
      const double eps = gm > 0.0 ? __ddiv_rn(__dmul_rn(sj, sj), gm) : 0.0;
      Emax = fmax(Emax, eps);
      const unsigned long long key = sel_key(eps, (unsigned long long)j, k, 0u, seed, a.greedy);
      a.keys_n[j] = key;
      atomicAdd(&h[key >> L1_SHIFT], 1u);
    }
    __syncthreads();
    flush_hist<PT>(h, hn, NBINS);
    {
      const double eb = pblock_max(Emax, sh);
      if (threadIdx.x == 0) bp[SL_MAXN * G + blockIdx.x] = eb;
    }
    grid_sync(a.bar, bgen);
    if (a.greedy) {
      p_sel_greedy(&ps, slot_max(bp, SL_MAXN, sh), a.eta);
    } else if (n <= LOCAL_SEL_MAX) {
      p_sel_level1(&ps, hn, n, kc, sh_u, sh_l);
      p_sel_local(&ps, a.keys_n, n, 0, h, sh_u, sh_l);
    } else {
      p_sel_level1(&ps, hn, n, kc, sh_u, sh_l);
      p_sel_scan<2>(&ps, a.keys_n, n, 0, hn + NBINS, cn, a.ncand, h);
      grid_sync(a.bar, bgen);
      p_sel_level2(&ps, hn + NBINS, sh_u, sh_l);
      p_sel_scan<3>(&ps, a.keys_n, n, 0, hn + 2 * NBINS, cn, a.ncand, h);
      grid_sync(a.bar, bgen);
      p_sel_level3(&ps, hn + 2 * NBINS, cn, a.ncand, a.keys_n, n, 0, h, sh_u, sh_l);
    }
    if (lead && ps.slow) st->selstat[1] += 1;
    // zeta = s on U (the CGLS direction p), Z = |zeta|^2, |U|, hash(U)
    double Z, dummy;
    {
      double Zp = 0.0;
      long long cnt = 0;
      unsigned long long hs = 0ull;
      for (int j = blockIdx.x * PT + threadIdx.x; j < n; j += G * PT) {
        const double sj = a.s[j];
        const bool sel = p_selected(&ps, a.keys_n[j], j);
        a.zeta[j] = sel ? sj : 0.0;
        if (sel) { Zp += sj * sj; cnt += 1; hs += splitmix64((unsigned long long)j); }
        if (a.capU) a.capU[(k & 1) * (long long)n + j] = sel ? 1 : 0;
      }
      cnt = warp_sum_ll(cnt);
      hs = warp_sum_u64(hs);
      if ((threadIdx.x & 31) == 0 && (cnt || hs)) {
        atomicAdd(&a.acc[0], (unsigned long long)cnt);
        atomicAdd(&a.acc[1], hs);
      }
      ex_allsum2(a, Zp, 0.0, SL_Z, SL_R, sh, bgen, Z, dummy);
    }
    const long long kp = (long long)__ldcg(&a.acc[0]);
    const unsigned long long hashU = __ldcg(&a.acc[1]);
    if (lead) {
      if (!a.greedy && kp != (ps.mode == SEL_NONE ? 0 : ps.target)) st->error |= 1;
      if (TraceRec* t = trace_at(tr, st, k)) { t->k = k; t->kp = kp; t->hash_u = hashU; t->Z = Z; }
    }
    // CGLS on min ||A_U y - z_k||: z is its residual
    double gam = Z, W0 = 0.0;
    for (int it = 0; it < e.inner_max && kp > 0 && gam > 0.0; ++it) {
      double Wp = 0.0, Yd = 0.0;
      ++npass;
      abytes += e.bytesN;
      ex_passN<DENSE>(a, ring, a.zeta, a.zeta, a.w, e.u, nullptr, Wp, Yd, dyn);           // q = A p
      double Wq, d2;
      ex_allsum2(a, Wp, 0.0, SL_W, SL_Y, sh, bgen, Wq, d2);
      if (it == 0) W0 = Wq;
      if (!(Wq > 0.0)) break;
      const double al = __ddiv_rn(gam, Wq);
      for (int i = blockIdx.x * PT + threadIdx.x; i < m_loc; i += G * PT)
        a.z[i] = __dsub_rn(a.z[i], __dmul_rn(al, a.w[i]));
      if (it + 1 == e.inner_max) break;
      grid_sync(a.bar, bgen);
      ++npass;
      abytes += e.bytesT;
      ex_passT<DENSE>(a, ring, a.z, a.z, 0, a.s, a.v, dyn, bgen);                         // s' = A^T z
      double gp = 0.0;
      for (int j = blockIdx.x * PT + threadIdx.x; j < n; j += G * PT)
        if (p_selected(&ps, a.keys_n[j], j)) gp += a.s[j] * a.s[j];
      double gnew, d3;
      ex_allsum2(a, gp, 0.0, SL_V, SL_X, sh, bgen, gnew, d3);
      if (gnew <= tol2 * Z) break;
      const double be = __ddiv_rn(gnew, gam);
      for (int j = blockIdx.x * PT + threadIdx.x; j < n; j += G * PT)
        a.zeta[j] = p_selected(&ps, a.keys_n[j], j) ? __dadd_rn(a.s[j], __dmul_rn(be, a.zeta[j])) : 0.0;
      gam = gnew;
      grid_sync(a.bar, bgen);
    }
    grid_sync(a.bar, bgen);
    if (lead) { if (TraceRec* t = trace_at(tr, st, k)) t->W = W0; }
    p_zero_side(a, 0);

    // ======================= row step =======================
    for (int i = threadIdx.x; i < NBINS; i += PT) h[i] = 0u;
    __syncthreads();
    double EmaxM = 0.0;
    for (int i = blockIdx.x * PT + threadIdx.x; i < m_loc; i += G * PT) {
      const double ri = __dsub_rn(__dsub_rn(a.b[i], a.z[i]), a.ax[i]);
      a.r[i] = ri;
      const double p = a.rho[i];
      const double eps = p > 0.0 ? __ddiv_rn(__dmul_rn(ri, ri), p) : 0.0;
      EmaxM = fmax(EmaxM, eps);
      const unsigned long long key = sel_key(eps, (unsigned long long)(a.row0 + i), k, 1u, seed, a.greedy);
      a.keys_m[i] = key;
      atomicAdd(&h[key >> L1_SHIFT], 1u);
    }
    __syncthreads();
    flush_hist<PT>(h, hm, NBINS);
    {
      const double eb = pblock_max(EmaxM, sh);
      if (threadIdx.x == 0) bp[SL_MAXM * G + blockIdx.x] = eb;
    }
    grid_sync(a.bar, bgen);
    if (a.greedy) {
      p_sel_greedy(&ps, slot_max(bp, SL_MAXM, sh), a.eta);
    } else if (m_loc <= LOCAL_SEL_MAX) {
      p_sel_level1(&ps, hm, m_loc, kr, sh_u, sh_l);
      p_sel_local(&ps, a.keys_m, m_loc, a.row0, h, sh_u, sh_l);
    } else {
      p_sel_level1(&ps, hm, m_loc, kr, sh_u, sh_l);
      p_sel_scan<2>(&ps, a.keys_m, m_loc, a.row0, hm + NBINS, cm, a.ncand + 1, h);
      grid_sync(a.bar, bgen);
      p_sel_level2(&ps, hm + NBINS, sh_u, sh_l);
      p_sel_scan<3>(&ps, a.keys_m, m_loc, a.row0, hm + 2 * NBINS, cm, a.ncand + 1, h);
      grid_sync(a.bar, bgen);
      p_sel_level3(&ps, hm + 2 * NBINS, cm, a.ncand + 1, a.keys_m, m_loc, a.row0, h, sh_u, sh_l);
    }
    if (lead && ps.slow) st->selstat[1] += 1;
    // xi = r on J (Craig's residual rho_J), X, |J|, hash(J); px = 0
    double X;
    {
      double Xp = 0.0;
      long long cnt = 0;
      unsigned long long hs = 0ull;
      for (int i = blockIdx.x * PT + threadIdx.x; i < m_loc; i += G * PT) {
        const long long gi = a.row0 + i;
        const bool sel = p_selected(&ps, a.keys_m[i], gi);
        const double ri = a.r[i];
        a.xi[i] = sel ? ri : 0.0;
        if (a.capJ) a.capJ[(k & 1) * (long long)m_loc + i] = sel ? 1 : 0;
        if (sel) { Xp += ri * ri; cnt += 1; hs += splitmix64((unsigned long long)gi); }
      }
      cnt = warp_sum_ll(cnt);
      hs = warp_sum_u64(hs);
      if ((threadIdx.x & 31) == 0 && (cnt || hs)) {
        atomicAdd(&a.acc[2], (unsigned long long)cnt);
        atomicAdd(&a.acc[3], hs);
      }
      double d4;
      ex_allsum2(a, Xp, 0.0, SL_X, SL_R, sh, bgen, X, d4);
    }
    const long long kpp = (long long)__ldcg(&a.acc[2]);
    const unsigned long long hashJ = __ldcg(&a.acc[3]);
    if (lead) {
      if (!a.greedy && kpp != (ps.mode == SEL_NONE ? 0 : ps.target)) st->error |= 2;
      if (TraceRec* t = trace_at(tr, st, k)) { t->kpp = kpp; t->hash_j = hashJ; t->X = X; }
    }
    // CGLS on min ||A^J y - r^J|| from y = 0 (limit: (A^J)^+ r^J): x += y.
    // a.xi holds its residual restricted to J; e.px its direction.
    double V0 = 0.0;
    if (kpp > 0 && X > 0.0) {
      ++npass;
      if constexpr (DENSE && RG_EX_MASK) {       // rows outside J hold r_J = 0: not read
        ex_dense_passT_rows(a, &ps, a.xi, dyn);
        grid_sync(a.bar, bgen);
        ex_dense_colreduce(a, 0, a.v, a.s, dyn);
        grid_sync(a.bar, bgen);
        abytes += 8.0 * (double)kpp * (double)n;
      } else {
        abytes += e.bytesT;
        ex_passT<DENSE>(a, ring, a.xi, a.xi, 0, a.v, a.s, dyn, bgen);                    // t = A^T r_J
      }
      double gp = 0.0;
      for (int j = blockIdx.x * PT + threadIdx.x; j < n; j += G * PT) {
        const double t = a.v[j];
        e.px[j] = t;
        gp += t * t;
      }
      double gam0, d5;
      ex_allsum2(a, gp, 0.0, SL_V, SL_Z, sh, bgen, gam0, d5);
      V0 = gam0;
      double gam = gam0;
      for (int it = 0; it < e.inner_max && gam > 0.0; ++it) {
        double Wd = 0.0, Yd = 0.0;
        ++npass;
        if constexpr (DENSE && RG_EX_MASK) {     // u is only used on J: A^J p
          ex_dense_passN_rows(a, &ps, e.px, e.u, dyn);
          abytes += 8.0 * (double)kpp * (double)n;
        } else {
          abytes += e.bytesN;
          ex_passN<DENSE>(a, ring, e.px, e.px, e.u, a.w, nullptr, Wd, Yd, dyn);          // u = A p
        }
        grid_sync(a.bar, bgen);   // sparse tiles spread rows over all CTAs
        double qp = 0.0;
        for (int i = blockIdx.x * PT + threadIdx.x; i < m_loc; i += G * PT)
          if (p_selected(&ps, a.keys_m[i], a.row0 + i)) qp += e.u[i] * e.u[i];
        double Wq, d6;
        ex_allsum2(a, qp, 0.0, SL_R, SL_W, sh, bgen, Wq, d6);
        if (!(Wq > 0.0)) break;
        const double al = __ddiv_rn(gam, Wq);
        for (int j = blockIdx.x * PT + threadIdx.x; j < n; j += G * PT)
          a.x[j] = __dadd_rn(a.x[j], __dmul_rn(al, e.px[j]));
        for (int i = blockIdx.x * PT + threadIdx.x; i < m_loc; i += G * PT)
          if (p_selected(&ps, a.keys_m[i], a.row0 + i))
            a.xi[i] = __dsub_rn(a.xi[i], __dmul_rn(al, e.u[i]));
        if (it + 1 == e.inner_max) break;
        grid_sync(a.bar, bgen);
        ++npass;
        if constexpr (DENSE && RG_EX_MASK) {
          ex_dense_passT_rows(a, &ps, a.xi, dyn);
          grid_sync(a.bar, bgen);
          ex_dense_colreduce(a, 0, a.v, a.s, dyn);
          grid_sync(a.bar, bgen);
          abytes += 8.0 * (double)kpp * (double)n;
        } else {
          abytes += e.bytesT;
          ex_passT<DENSE>(a, ring, a.xi, a.xi, 0, a.v, a.s, dyn, bgen);                  // t = A^T r_J
        }
        double gq = 0.0;
        for (int j = blockIdx.x * PT + threadIdx.x; j < n; j += G * PT) gq += a.v[j] * a.v[j];
        double gnew, d7;
        ex_allsum2(a, gq, 0.0, SL_V, SL_Z, sh, bgen, gnew, d7);
        if (gnew <= tol2 * gam0) break;
        const double be = __ddiv_rn(gnew, gam);
        for (int j = blockIdx.x * PT + threadIdx.x; j < n; j += G * PT)
          e.px[j] = __dadd_rn(a.v[j], __dmul_rn(be, e.px[j]));
        gam = gnew;
        grid_sync(a.bar, bgen);
      }
    }
    grid_sync(a.bar, bgen);
    if (lead) { if (TraceRec* t = trace_at(tr, st, k)) t->V = V0; }

    // ======================= end of iteration: A x_{k+1}, stop test =======================
    double Y, relerr2;
    {
      double Wd = 0.0, Yp = 0.0, Rp = 0.0;
      ++npass;
      abytes += e.bytesN;
      ex_passN<DENSE>(a, ring, a.x, a.x, e.u, a.ax, a.b, Wd, Yp, dyn);
      if (has_ref)
        for (int j = blockIdx.x * PT + threadIdx.x; j < n; j += G * PT) {
          const double d = a.x[j] - a.xstar[j];
          Rp += d * d;
        }
      ex_allsum2(a, Yp, Rp, SL_Y, SL_R, sh, bgen, Y, relerr2);
    }
    k += 1;
    const double rse = Y / bnorm2;
    const double rel = has_ref ? sqrt(relerr2 / xsnorm2) : __longlong_as_double(0x7FF8000000000000ll);
    if (lead) { if (TraceRec* t = trace_at(tr, st, k - 1)) t->rse = rse; }
    int halt = 0, outcome = RGDBEK_MAX_ITER;
    if (stop_mode == RGDBEK_STOP_RSE && rse <= tol) { halt = 1; outcome = RGDBEK_CONVERGED; }
    else if (stop_mode == RGDBEK_STOP_REL_ERR && rel <= tol) { halt = 1; outcome = RGDBEK_CONVERGED; }
    else if (kp == 0 && kpp == 0) { halt = 1; outcome = RGDBEK_STALLED; }
    else if (k >= k_end) { halt = 1; outcome = RGDBEK_MAX_ITER; }
    p_zero_side(a, 1);
    if (halt) {
      if (lead) {
        st->halted = 1; st->outcome = outcome; st->iters = k; st->rse_out = rse;
        st->relerr_out = rel; st->k = k; st->pending = 0; st->kp_prev = kp; st->kpp_prev = kpp;
        st->npass += npass;
        st->abytes += abytes;
      }
      return;
    }
    grid_sync(a.bar, bgen);
  }
}

}  // namespace rg
