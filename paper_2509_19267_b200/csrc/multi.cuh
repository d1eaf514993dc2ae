// multi.cuh — several right-hand sides sharing one sparse A (PAPER.md
// the three colour channels of the deblurring problem solve A x_i = b_i with
// the same blur operator A).
//
// NR <= 4 independent Algorithm-1 solves (reading R29): RHS rho has its own z, x, blocks
// U_rho / J_rho and its own Philox stream (seed + rho); every pass over A serves all NR
// solves, so A's bytes per RHS-iteration drop by NR.  Vectors that the passes gather are
// interleaved [index][rho] (one gather of a column fetches the NR values of one 32-byte
// sector); keys are per RHS [rho][index] (the selection scans stream them).  The block
// selections of the NR solves share the grid barriers.  Pseudoinverse-free update, random
// selection, CSR / CSC tiles (csr_tiles.cuh's TMA ring), one persistent kernel.
#pragma once
#include "persistent.cuh"

namespace rg {

constexpr int MAXRHS = 4;
// gather entries per lane per round for NR = 2, 3, 4 right-hand sides (registers: the
// gathered values are RU x 2 x NR doubles per lane)
#ifndef RG_MRU2
#define RG_MRU2 3
#endif
#ifndef RG_MRU3
#define RG_MRU3 2
#endif
#ifndef RG_MRU4
#define RG_MRU4 2
#endif

struct MArgs {
  int nr;                                 // right-hand sides
  double *x, *s, *v, *zeta;               // [n][nr]
  double *z, *w, *ax, *r, *xi, *b;        // [m][nr]
  unsigned long long* keys_n[MAXRHS];     // [n] each
  unsigned long long* keys_m[MAXRHS];     // [m] each
  unsigned int* hist[MAXRHS];             // [2 sides][3 levels][NBINS] each
  Cand* cand[MAXRHS];                     // [2][CAND_CAP] each
  unsigned long long* acc[MAXRHS];        // [4] each
  unsigned int* ncand[MAXRHS];            // [2] each
  Scal* st[MAXRHS];                       // per-RHS scalars (st[0] also holds the call control)
  TraceRec* tr[MAXRHS];                   // per-RHS trace rings
  double* xstar;                          // [n][nr]
};

// One staged tile's rows for NR interleaved input vectors (csr_tiles.cuh's tile_rows with
// NR products per nonzero and each gather fetching the NR values of a column).
template <int LV, int NR>
__device__ __forceinline__ void tile_rows_m(const TileRows& t, double (&Wp)[NR], double (&Yp)[NR]) {
  constexpr int v = 1 << LV, spw = 32 >> LV;
  constexpr int RU = NR == 1 ? RG_RU : (NR == 2 ? RG_MRU2 : (NR == 3 ? RG_MRU3 : RG_MRU4));
  const int sub = t.lane >> LV, sl = t.lane & (v - 1);
  for (int base = t.lw * spw; base < t.nr; base += (TG / 32) * spw) {
    const int r = base + sub;
    const bool valid = r < t.nr;
    double s1[NR], s2[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) { s1[q] = 0.0; s2[q] = 0.0; }
    if (valid) {
      int p = (int)(t.R[r] - t.p0) + sl;
      const int p1 = (int)(t.R[r + 1] - t.p0);
      for (; p < p1; p += RU * v) {
        int c[RU];
        double g1[RU][NR], g2[RU][NR];
#pragma unroll
        for (int e = 0; e < RU; ++e) c[e] = p + e * v < p1 ? t.I[p + e * v] : -1;
#pragma unroll
        for (int e = 0; e < RU; ++e) {
#pragma unroll
          for (int q = 0; q < NR; ++q) {
            g1[e][q] = c[e] >= 0 ? t.in1[(long long)c[e] * NR + q] : 0.0;
            g2[e][q] = (t.use2 && c[e] >= 0) ? t.in2[(long long)c[e] * NR + q] : 0.0;
          }
        }
#pragma unroll
        for (int e = 0; e < RU; ++e) {
          if (c[e] >= 0) {
            const double a = t.V[p + e * v];
#pragma unroll
            for (int q = 0; q < NR; ++q) { s1[q] = fma(a, g1[e][q], s1[q]); s2[q] = fma(a, g2[e][q], s2[q]); }
          }
        }
      }
    }
#pragma unroll
    for (int o = v >> 1; o > 0; o >>= 1) {           // fixed shuffle tree (deterministic)
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        s1[q] += __shfl_xor_sync(0xffffffffu, s1[q], o);
        s2[q] += __shfl_xor_sync(0xffffffffu, s2[q], o);
      }
    }
    if (valid && sl == 0) {
      const long long row = t.r0 + r;
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        t.o1[row * NR + q] = s1[q];
        t.o2[row * NR + q] = s2[q];
        if (t.has_b) {
          const double y = t.b[row * NR + q] - s2[q];
          Wp[q] += s1[q] * s1[q];
          Yp[q] += y * y;
        }
      }
    }
  }
}

// csr_tiles with NR interleaved vectors per product (no fused key epilogue: the keys of
// the NR solves are made in a separate sweep).
template <int NR>
__device__ void csr_tiles_m(int gid, int ngroups, int lt, int bar_id, TileSmem* sm, TileRing& ring,
                            const long long* __restrict__ ptr, const int* __restrict__ idx,
                            const double* __restrict__ val, const int* __restrict__ tiles,
                            const long long* __restrict__ tilep, int ntiles, const double* in1,
                            const double* in2, int use2, const double* __restrict__ b, double* o1,
                            double* o2, double (&Wp)[NR], double (&Yp)[NR], int vec, int rev) {
  const int tb = gid, tstep = ngroups;
  const int cnt = gid < ntiles ? (ntiles - gid + ngroups - 1) / ngroups : 0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  group_bar(bar_id);
  unsigned long long* full = ring.full;
  unsigned long long* rel = ring.full + TBUF;
  if (lt == 0) {
    for (int i = 0; i < cnt && i < TBUF; ++i) {
      const unsigned u = ring.used + i;
      const int ti = tb + i * tstep;
      tile_issue(sm, u % TBUF, &full[u % TBUF], tile_desc(rev ? ntiles - 1 - ti : ti, tiles, tilep),
                 ptr, idx, val);
    }
  }
  const int lane = lt & 31, lw = lt >> 5;
  const int lvec = __ffs(vec) - 1;
  const bool has_b = b != nullptr;
  for (int i = 0; i < cnt; ++i) {
    const int t = tb + i * tstep;
    const unsigned u = ring.used + i, bi = u % TBUF;
    TileDesc nd{0, 0, 0, 0};
    const bool refill = lane == 0 && i + TBUF < cnt;
    if (refill) {
      const int tn = t + TBUF * tstep;
      nd = tile_desc(rev ? ntiles - 1 - tn : tn, tiles, tilep);
    }
    mbar_wait(&full[bi], (u / TBUF) & 1u);
    const int r0 = (int)sm->desc[bi][0], nr = (int)(sm->desc[bi][1] - sm->desc[bi][0]);
    const long long p0 = sm->desc[bi][2], p1 = sm->desc[bi][3];
    if (p1 - p0 > TILE_NNZ) {                        // one long row: group-wide reduction
      double a1[NR], a2[NR];
#pragma unroll
      for (int q = 0; q < NR; ++q) { a1[q] = 0.0; a2[q] = 0.0; }
      for (long long p = p0 + lt; p < p1; p += TG) {
        const double a = ld_stream(val + p);
        const long long c = __ldg(idx + p);
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          a1[q] = fma(a, ld_weak(in1 + c * NR + q), a1[q]);
          if (use2) a2[q] = fma(a, ld_weak(in2 + c * NR + q), a2[q]);
        }
      }
      for (int q = 0; q < NR; ++q) {
        const double w1 = warp_sum(a1[q]), w2 = warp_sum(a2[q]);
        group_bar(bar_id);
        if (lane == 0) { sm->red[2 * lw] = w1; sm->red[2 * lw + 1] = w2; }
        group_bar(bar_id);
        if (lt == 0) {
          double s1 = 0.0, s2 = 0.0;
          for (int w = 0; w < TG / 32; ++w) { s1 += sm->red[2 * w]; s2 += sm->red[2 * w + 1]; }
          o1[(long long)r0 * NR + q] = s1;
          o2[(long long)r0 * NR + q] = s2;
          if (has_b) {
            const double y = b[(long long)r0 * NR + q] - s2;
            Wp[q] += s1 * s1;
            Yp[q] += y * y;
          }
        }
      }
      group_bar(bar_id);
    } else {
      int lv = lvec;
      while (lv < 5 && (nr << (lv + 1)) <= TG) ++lv;
      const TileBuf& B = sm->buf[bi];
      const TileRows tr{B.rp + (r0 & 1), B.val + (p0 & 1), B.idx + (p0 & 3), p0, r0, nr, lane, lw,
                        has_b, b, in1, in2, use2, o1, o2, nullptr, 0, nullptr, 0};
      switch (lv) {
        case 0: tile_rows_m<0, NR>(tr, Wp, Yp); break;
        case 1: tile_rows_m<1, NR>(tr, Wp, Yp); break;
        case 2: tile_rows_m<2, NR>(tr, Wp, Yp); break;
        case 3: tile_rows_m<3, NR>(tr, Wp, Yp); break;
        case 4: tile_rows_m<4, NR>(tr, Wp, Yp); break;
        default: tile_rows_m<5, NR>(tr, Wp, Yp); break;
      }
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      const unsigned long long done = atomicAdd(&rel[bi], 1ull);
      if (done == TG / 32 - 1) {
        __threadfence_block();
        rel[bi] = 0ull;
        if (refill) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          tile_issue(sm, bi, &full[bi], nd, ptr, idx, val);
        }
      }
    }
  }
  group_bar(bar_id);
  ring.used += cnt;
}

// Exact selection of one side of one RHS (all CTAs, identical results): CTA-local when
// the keys fit, else the grid-wide levels (two grid barriers, shared by the NR solves:
// the caller runs phase `step` of every RHS between its barriers).
__device__ __forceinline__ void m_zero_side(unsigned int* hist_side, unsigned long long* acc2,
                                            unsigned int* ncand1) {
  for (int i = blockIdx.x * PT + threadIdx.x; i < 3 * NBINS; i += gridDim.x * PT) hist_side[i] = 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) { acc2[0] = 0ull; acc2[1] = 0ull; *ncand1 = 0u; }
}

template <int NR>
__global__ void __launch_bounds__(PT, 1) k_multi(PArgs a, MArgs ma) {
  __shared__ __align__(16) unsigned int h[NBINS];
  __shared__ __align__(8) unsigned long long tbar[(PT / TG) * TRING];
  __shared__ double sh[PW];
  __shared__ unsigned int sh_u[4];
  __shared__ long long sh_l[40];
  __shared__ PSel ps[NR];
  extern __shared__ __align__(16) double dyn[];
  TileRing tring{tbar + (threadIdx.x / TG) * TRING, 0u};
  tile_rings_init(tbar);
  Scal* st = ma.st[0];
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  const int G = gridDim.x;
  long long k = st->k;
  const long long k_begin = st->k_begin, k_end = st->k_end;
  const double tol = st->tol;
  const int stop_mode = st->stop_mode, has_ref = st->has_ref;
  const unsigned long long seed = st->seed;
  const long long kc = st->kc, kr = st->kr;
  int pending = st->pending;
  double X[NR], bnorm2[NR], xsnorm2[NR];
  long long kp_prev[NR], kpp_prev[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    X[q] = ma.st[q]->X; kp_prev[q] = ma.st[q]->kp_prev; kpp_prev[q] = ma.st[q]->kpp_prev;
    bnorm2[q] = ma.st[q]->bnorm2; xsnorm2[q] = ma.st[q]->xsnorm2;
  }
  const int n = a.n, m_loc = a.m_loc;
  unsigned int bgen = 0;
  if (threadIdx.x == 0) bgen = ld_acquire_u32(&a.bar->gen);
  double* bp = a.bpart;                                 // [NR][SL_NUM][G]
#define MSLOT(q, s) (bp + ((q) * SL_NUM + (s)) * G)

  for (;;) {
    // ===== P1: pass T  (s = A^T z, v = A^T xi for every RHS) =====
    {
      double d1[NR], d2[NR];
      const int g = threadIdx.x / TG;
      csr_tiles_m<NR>(blockIdx.x * (PT / TG) + g, G * (PT / TG), threadIdx.x % TG, 1 + g,
                      reinterpret_cast<TileSmem*>(dyn) + g, tring, a.cp, a.ri, a.rv, a.tilesT,
                      a.tilepT, a.ntilesT, ma.z, ma.xi, pending, nullptr, ma.s, ma.v, d1, d2,
                      a.vecT, 0);
    }
    grid_sync(a.bar, bgen);
    // ===== P2: column scores and keys of every RHS, level-1 histograms, V partials =====
    {
      unsigned int* hq = reinterpret_cast<unsigned int*>(dyn);       // [NR][NBINS] (free now)
      for (int i = threadIdx.x; i < NR * NBINS; i += PT) hq[i] = 0u;
      __syncthreads();
      double Vp[NR];
#pragma unroll
      for (int q = 0; q < NR; ++q) Vp[q] = 0.0;
      for (int j = blockIdx.x * PT + threadIdx.x; j < n; j += G * PT) {
        const double gm = a.gamma[j];
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const double sj = ma.s[(long long)j * NR + q];
          if (pending) { const double vj = ma.v[(long long)j * NR + q]; Vp[q] += vj * vj; }
          const double eps = gm > 0.0 ? __ddiv_rn(__dmul_rn(sj, sj), gm) : 0.0;
          const unsigned long long key = make_key(eps, (unsigned long long)j, k, 0u, seed + q);
          ma.keys_n[q][j] = key;
          atomicAdd(&hq[q * NBINS + (key >> L1_SHIFT)], 1u);
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        flush_hist<PT>(hq + q * NBINS, ma.hist[q], NBINS);
        const double vb = pblock_sum(Vp[q], sh);
        if (threadIdx.x == 0) MSLOT(q, SL_V)[blockIdx.x] = vb;
        m_zero_side(ma.hist[q] + 3 * NBINS, ma.acc[q] + 2, ma.ncand[q] + 1);   // m-side: consumed
      }
    }
    grid_sync(a.bar, bgen);
    // ===== P3-P5: the NR column selections; zeta, Z, |U|, hash; x_k =====
    double V[NR], alpha_x[NR];
    int do_x[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      V[q] = slot_sum(MSLOT(q, SL_V), 0, sh);
      do_x[q] = pending && kpp_prev[q] > 0 && V[q] > 0.0;
      alpha_x[q] = do_x[q] ? __ddiv_rn(X[q], V[q]) : 0.0;
      if (lead && pending) { if (TraceRec* t = trace_at(ma.tr[q], st, k - 1)) t->V = V[q]; }
      p_sel_level1(&ps[q], ma.hist[q], n, kc, sh_u, sh_l);
    }
    if (n <= LOCAL_SEL_MAX) {
      for (int q = 0; q < NR; ++q)
        if (!p_sel_local_smem(&ps[q], ma.keys_n[q], n, 0, ma.hist[q], h, sh_u, sh_l,
                              reinterpret_cast<Cand*>(dyn), reinterpret_cast<Cand*>(dyn) + LCAND_CAP))
          p_sel_local(&ps[q], ma.keys_n[q], n, 0, h, sh_u, sh_l);
    } else {
      for (int q = 0; q < NR; ++q)
        p_sel_scan<2>(&ps[q], ma.keys_n[q], n, 0, ma.hist[q] + NBINS, ma.cand[q], ma.ncand[q], h);
      grid_sync(a.bar, bgen);
      for (int q = 0; q < NR; ++q) {
        p_sel_level2(&ps[q], ma.hist[q] + NBINS, sh_u, sh_l);
        p_sel_scan<3>(&ps[q], ma.keys_n[q], n, 0, ma.hist[q] + 2 * NBINS, ma.cand[q], ma.ncand[q], h);
      }
      grid_sync(a.bar, bgen);
      for (int q = 0; q < NR; ++q)
        p_sel_level3(&ps[q], ma.hist[q] + 2 * NBINS, ma.cand[q], ma.ncand[q], ma.keys_n[q], n, 0, h,
                     sh_u, sh_l);
    }
    {
      double Zp[NR], Rp[NR];
      long long cnt[NR];
      unsigned long long hs[NR];
#pragma unroll
      for (int q = 0; q < NR; ++q) { Zp[q] = 0.0; Rp[q] = 0.0; cnt[q] = 0; hs[q] = 0ull; }
      for (int j = blockIdx.x * PT + threadIdx.x; j < n; j += G * PT) {
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const long long e = (long long)j * NR + q;
          const double sj = ma.s[e];
          const bool sel = p_selected(&ps[q], ma.keys_n[q][j], j);
          ma.zeta[e] = sel ? sj : 0.0;
          if (sel) { Zp[q] += sj * sj; cnt[q] += 1; hs[q] += splitmix64((unsigned long long)j); }
          double xj = ma.x[e];
          if (do_x[q]) { xj = __dadd_rn(xj, __dmul_rn(alpha_x[q], ma.v[e])); ma.x[e] = xj; }
          if (has_ref) { const double d = xj - ma.xstar[e]; Rp[q] += d * d; }
        }
      }
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const long long c = warp_sum_ll(cnt[q]);
        const unsigned long long hh = warp_sum_u64(hs[q]);
        if ((threadIdx.x & 31) == 0 && (c || hh)) {
          atomicAdd(&ma.acc[q][0], (unsigned long long)c);
          atomicAdd(&ma.acc[q][1], hh);
        }
        const double zb = pblock_sum(Zp[q], sh);
        const double rb = pblock_sum(Rp[q], sh);
        if (threadIdx.x == 0) { MSLOT(q, SL_Z)[blockIdx.x] = zb; MSLOT(q, SL_R)[blockIdx.x] = rb; }
      }
    }
    pending = 0;
    grid_sync(a.bar, bgen);
    // ===== P6: pass N (w = A zeta, A x_k for every RHS), W / ||b - A x||^2 =====
    double Z[NR], relerr2[NR];
    long long kp[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      Z[q] = slot_sum(MSLOT(q, SL_Z), 0, sh);
      relerr2[q] = slot_sum(MSLOT(q, SL_R), 0, sh);
      kp[q] = (long long)__ldcg(&ma.acc[q][0]);
      if (lead) {
        if (kp[q] != (ps[q].mode == SEL_NONE ? 0 : ps[q].target)) st->error |= 1;
        if (TraceRec* t = trace_at(ma.tr[q], st, k)) {
          t->k = k; t->kp = kp[q]; t->hash_u = __ldcg(&ma.acc[q][1]); t->Z = Z[q];
        }
      }
    }
    {
      double Wp[NR], Yp[NR];
#pragma unroll
      for (int q = 0; q < NR; ++q) { Wp[q] = 0.0; Yp[q] = 0.0; }
      const int g = threadIdx.x / TG;
      csr_tiles_m<NR>(blockIdx.x * (PT / TG) + g, G * (PT / TG), threadIdx.x % TG, 1 + g,
                      reinterpret_cast<TileSmem*>(dyn) + g, tring, a.rp, a.ci, a.cv, a.tilesN,
                      a.tilepN, a.ntilesN, ma.zeta, ma.x, 1, ma.b, ma.w, ma.ax, Wp, Yp, a.vecN,
                      RG_REV_N);
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const double wb = pblock_sum(Wp[q], sh);
        const double yb = pblock_sum(Yp[q], sh);
        if (threadIdx.x == 0) { MSLOT(q, SL_W)[blockIdx.x] = wb; MSLOT(q, SL_Y)[blockIdx.x] = yb; }
      }
    }
    grid_sync(a.bar, bgen);
    // ===== P8: stop test (every RHS); z_{k+1}, r, row keys, level-1 histograms =====
    double W[NR];
    {
      int all_done = 1, all_conv = 1;
      double Y[NR];
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        W[q] = slot_sum(MSLOT(q, SL_W), 0, sh);
        Y[q] = slot_sum(MSLOT(q, SL_Y), 0, sh);
        const double rse = Y[q] / bnorm2[q];
        const double rel = has_ref ? sqrt(relerr2[q] / xsnorm2[q]) : __longlong_as_double(0x7FF8000000000000ll);
        const int conv = (stop_mode == RGDBEK_STOP_RSE && rse <= tol) ||
                         (stop_mode == RGDBEK_STOP_REL_ERR && rel <= tol);
        const int stall = kp_prev[q] == 0 && kpp_prev[q] == 0;
        all_done &= conv | stall;
        all_conv &= conv;
        if (lead) {
          if (TraceRec* t = trace_at(ma.tr[q], st, k)) t->W = W[q];
          if (k >= 1) { if (TraceRec* t = trace_at(ma.tr[q], st, k - 1)) t->rse = rse; }
          ma.st[q]->rse_out = rse;
          ma.st[q]->relerr_out = rel;
        }
      }
      int halt = 0, outcome = RGDBEK_MAX_ITER;
      if (k > k_begin && all_done) { halt = 1; outcome = all_conv ? RGDBEK_CONVERGED : RGDBEK_STALLED; }
      if (!halt && (k > k_begin || k_end == k_begin) && k >= k_end) { halt = 1; outcome = RGDBEK_MAX_ITER; }
      if (halt) {
        for (int q = 0; q < NR; ++q)
          m_zero_side(ma.hist[q], ma.acc[q], ma.ncand[q]);
        if (lead) {
          st->halted = 1; st->outcome = outcome; st->iters = k; st->k = k; st->pending = 0;
          st->npass += 2 * (k - k_begin + 1);
          for (int q = 0; q < NR; ++q) {
            ma.st[q]->X = X[q]; ma.st[q]->kp_prev = kp_prev[q]; ma.st[q]->kpp_prev = kpp_prev[q];
          }
        }
        return;
      }
    }
    {
      unsigned int* hq = reinterpret_cast<unsigned int*>(dyn);
      for (int i = threadIdx.x; i < NR * NBINS; i += PT) hq[i] = 0u;
      __syncthreads();
      double az[NR];
      int doz[NR];
#pragma unroll
      for (int q = 0; q < NR; ++q) { doz[q] = kp[q] > 0 && W[q] > 0.0; az[q] = doz[q] ? __ddiv_rn(Z[q], W[q]) : 0.0; }
      for (int i = blockIdx.x * PT + threadIdx.x; i < m_loc; i += G * PT) {
        const double p = a.rho[i];
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const long long e = (long long)i * NR + q;
          double zi = ma.z[e];
          if (doz[q]) { zi = __dsub_rn(zi, __dmul_rn(az[q], ma.w[e])); ma.z[e] = zi; }
          const double ri = __dsub_rn(__dsub_rn(ma.b[e], zi), ma.ax[e]);
          ma.r[e] = ri;
          const double eps = p > 0.0 ? __ddiv_rn(__dmul_rn(ri, ri), p) : 0.0;
          const unsigned long long key = make_key(eps, (unsigned long long)(a.row0 + i), k, 1u, seed + q);
          ma.keys_m[q][i] = key;
          atomicAdd(&hq[q * NBINS + (key >> L1_SHIFT)], 1u);
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        flush_hist<PT>(hq + q * NBINS, ma.hist[q] + 3 * NBINS, NBINS);
        m_zero_side(ma.hist[q], ma.acc[q], ma.ncand[q]);              // n-side: consumed
      }
    }
    grid_sync(a.bar, bgen);
    // ===== P9-P11: the NR row selections; xi, X, |J|, hash =====
#pragma unroll
    for (int q = 0; q < NR; ++q) p_sel_level1(&ps[q], ma.hist[q] + 3 * NBINS, m_loc, kr, sh_u, sh_l);
    if (m_loc <= LOCAL_SEL_MAX) {
      for (int q = 0; q < NR; ++q)
        if (!p_sel_local_smem(&ps[q], ma.keys_m[q], m_loc, a.row0, ma.hist[q] + 3 * NBINS, h, sh_u,
                              sh_l, reinterpret_cast<Cand*>(dyn), reinterpret_cast<Cand*>(dyn) + LCAND_CAP))
          p_sel_local(&ps[q], ma.keys_m[q], m_loc, a.row0, h, sh_u, sh_l);
    } else {
      for (int q = 0; q < NR; ++q)
        p_sel_scan<2>(&ps[q], ma.keys_m[q], m_loc, a.row0, ma.hist[q] + 4 * NBINS, ma.cand[q] + CAND_CAP,
                      ma.ncand[q] + 1, h);
      grid_sync(a.bar, bgen);
      for (int q = 0; q < NR; ++q) {
        p_sel_level2(&ps[q], ma.hist[q] + 4 * NBINS, sh_u, sh_l);
        p_sel_scan<3>(&ps[q], ma.keys_m[q], m_loc, a.row0, ma.hist[q] + 5 * NBINS, ma.cand[q] + CAND_CAP,
                      ma.ncand[q] + 1, h);
      }
      grid_sync(a.bar, bgen);
      for (int q = 0; q < NR; ++q)
        p_sel_level3(&ps[q], ma.hist[q] + 5 * NBINS, ma.cand[q] + CAND_CAP, ma.ncand[q] + 1,
                     ma.keys_m[q], m_loc, a.row0, h, sh_u, sh_l);
    }
    {
      double Xp[NR];
      long long cnt[NR];
      unsigned long long hs[NR];
#pragma unroll
      for (int q = 0; q < NR; ++q) { Xp[q] = 0.0; cnt[q] = 0; hs[q] = 0ull; }
      for (int i = blockIdx.x * PT + threadIdx.x; i < m_loc; i += G * PT) {
        const long long gi = a.row0 + i;
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          const long long e = (long long)i * NR + q;
          const double ri = ma.r[e];
          const bool sel = p_selected(&ps[q], ma.keys_m[q][i], gi);
          ma.xi[e] = sel ? ri : 0.0;
          if (sel) { Xp[q] += ri * ri; cnt[q] += 1; hs[q] += splitmix64((unsigned long long)gi); }
        }
      }
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const long long c = warp_sum_ll(cnt[q]);
        const unsigned long long hh = warp_sum_u64(hs[q]);
        if ((threadIdx.x & 31) == 0 && (c || hh)) {
          atomicAdd(&ma.acc[q][2], (unsigned long long)c);
          atomicAdd(&ma.acc[q][3], hh);
        }
        const double xb = pblock_sum(Xp[q], sh);
        if (threadIdx.x == 0) MSLOT(q, SL_X)[blockIdx.x] = xb;
      }
    }
    grid_sync(a.bar, bgen);
    // ===== P12: X, |J| per RHS; k++ =====
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      X[q] = slot_sum(MSLOT(q, SL_X), 0, sh);
      const long long kpp = (long long)__ldcg(&ma.acc[q][2]);
      if (lead) {
        if (kpp != (ps[q].mode == SEL_NONE ? 0 : ps[q].target)) st->error |= 2;
        if (TraceRec* t = trace_at(ma.tr[q], st, k)) { t->kpp = kpp; t->hash_j = __ldcg(&ma.acc[q][3]); t->X = X[q]; }
      }
      kpp_prev[q] = kpp;
      kp_prev[q] = kp[q];
    }
    pending = 1;
    k += 1;
    __syncthreads();
  }
#undef MSLOT
}

}  // namespace rg
