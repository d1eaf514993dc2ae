// csr_tiles.cuh — CSR (or CSC) dual SpMV by nnz tiles, fed by TMA bulk copies.
//
// A sparse pass computes o1 = A in1 and o2 = A in2 over rows (pass N: A zeta,
// A x; pass T over the CSC: A^T z, A^T xi).  Rows are short (5-41 nnz in the
// paper's workloads), so a row-per-thread loop is a chain of three dependent
// memory round trips per row (row pointer -> value/index -> gathered vector)
// and keeps almost nothing in flight.  Instead a worker group of TG threads
// takes tiles of consecutive rows holding <= TILE_NNZ nonzeros (precomputed at
// create, with each tile's first nonzero offset), and:
//   * one thread of the group streams the tile's row pointers, values and
//     column indices into shared memory with cp.async.bulk (TMA bulk copies,
//     completion on an mbarrier), TBUF tiles ahead of the group, so the
//     matrix stream is always in flight while the group works; the last
//     warp to finish with a buffer refills it (no warp waits for another);
//   * the group sums each row from shared memory, `vec` lanes per row, with
//     the gathers in1[c], in2[c] issued four entries at a time; partial sums
//     are combined by a fixed shuffle tree (deterministic).
// A row longer than TILE_NNZ is a tile by itself, read straight from global
// memory and reduced across the group.
#pragma once
#include "common.cuh"

namespace rg {

// Geometry (compile-time; -D overrides exist for A/B builds, tools/ab_variants.py).
#ifndef RG_TILE_NNZ
#define RG_TILE_NNZ 1120
#endif
#ifndef RG_TILE_ROWS
#define RG_TILE_ROWS 256
#endif
#ifndef RG_TBUF
#define RG_TBUF 3
#endif
#ifndef RG_PEND
#define RG_PEND 320
#endif
#ifndef RG_RU
#define RG_RU 6
#endif
#ifndef RG_REV_N
#define RG_REV_N 1        // pass N walks the tiles / rows in reverse (L2 reuse after pass T)
#endif
#ifndef RG_TG
#define RG_TG 256
#endif
#ifndef RG_RU5
// gather entries per lane per round at 32 lanes per row (tiles of a few long rows, e.g. the
// ~200-entry CSC columns of C5): 7 covers a 224-entry row in ONE round trip instead of
// two (tools/ab_pass.py, profiles/r2/ab_pass_2.log: C5m pass T +13 %, iteration +8.6 %;
// 8 the same, 6 = RG_RU the old default)
#define RG_RU5 7
#endif
constexpr int TG = RG_TG;            // threads per worker group
constexpr int TILE_NNZ = RG_TILE_NNZ;    // nonzeros per tile
constexpr int TILE_ROWS = RG_TILE_ROWS;  // rows per tile
#ifndef RG_GRAPH_TBUF
// ring depth of the graph engine's standalone tile kernel: with 2 buffers shared memory
// admits 6 blocks per SM where 3 admit 4 (registers then cap pass N at 5: 40-48 tile warps)
// — more consumer warps is what the sparse passes need
// (C5c: graph engine 129 -> 135 it/s, C5m +6 %; profiles/r2/ab_engine_c5.jsonl)
#define RG_GRAPH_TBUF 2
#endif
constexpr int TBUF = RG_TBUF;        // staged tiles per group (one in use, the rest in flight)
constexpr int TRING = 2 * TBUF;      // ring words per group: full[TBUF] mbarriers, rel[TBUF] counters
constexpr int GRAPH_TBUF = RG_GRAPH_TBUF;
constexpr int PEND = RG_PEND;        // pass-T columns batched for the key epilogue
static_assert(PEND >= TILE_ROWS, "a whole tile's columns must fit the pending list");

// One staged tile.  Windows are widened to 16-byte boundaries (bulk-copy
// alignment): val from p0 & ~1, idx from p0 & ~3, rp from r0 & ~1.
struct __align__(16) TileBuf {
  double val[TILE_NNZ + 2];
  int idx[TILE_NNZ + 8];
  long long rp[TILE_ROWS + 4];
};
static_assert(sizeof(TileBuf) % 16 == 0, "TileBuf must keep 16-byte alignment");

// Pass-T column results waiting for the key epilogue (batched so a tile of a
// few long columns does not run the ALU-heavy key chain on a few threads).
struct TilePend {
  double s1[PEND], s2[PEND];
  int row[PEND];
};

template <int NB>
struct __align__(16) TileSmemT {
  TileBuf buf[NB];
  long long desc[NB][4];         // r0, r1, p0, p1 of the staged tile (written by the producer)
  double red[2 * (TG / 32)];
  TilePend pend;
};
using TileSmem = TileSmemT<TBUF>;      // the persistent kernels' ring

// Barrier over this worker group's TG threads (named barrier id >= 1).
__device__ __forceinline__ void group_bar(int id) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(TG) : "memory");
}

// Per-group ring state in static shared memory (so other phases may reuse the
// TileSmem area as scratch): full[b], an mbarrier completing when buffer b's
// bulk copies have landed, and rel[b], the number of the group's warps done
// with buffer b (the last one refills it); plus the number of tiles this group
// has consumed so far (identical in all its threads).
struct TileRing {
  unsigned long long* full;   // [TRING]: full[0..TBUF), then rel[0..TBUF)
  unsigned int used;
};

// Initialise a group's barriers (one thread), before the first csr_tiles call;
// the caller follows with fence.mbarrier_init + a CTA barrier.
template <int NB = TBUF>
__device__ __forceinline__ void tile_ring_init(unsigned long long* bars) {
  for (int i = 0; i < NB; ++i) {
    mbar_init(&bars[i], 1);
    bars[NB + i] = 0ull;                           // release counter of buffer i
  }
}

// CTA prologue of a kernel running csr_tiles: every group's barriers, made
// visible to the async proxy and to the whole CTA.
template <int NB = TBUF>
__device__ __forceinline__ void tile_rings_init(unsigned long long* bars) {
  if (threadIdx.x % TG == 0) tile_ring_init<NB>(bars + (threadIdx.x / TG) * (2 * NB));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
}

// Tile descriptor: rows [r0, r1), nonzeros [p0, p1).
struct TileDesc {
  long long r0, r1, p0, p1;
};

__device__ __forceinline__ TileDesc tile_desc(int t, const int* __restrict__ tiles,
                                              const long long* __restrict__ tilep) {
  return TileDesc{__ldg(tiles + t), __ldg(tiles + t + 1), __ldg(tilep + t), __ldg(tilep + t + 1)};
}

// Issue the bulk copies of tile d into buffer b (one thread).  The descriptor
// goes to shared memory before the barrier's arrive (release), so consumers
// read it after their wait (acquire).  Bytes are counted on the barrier
// before the copies start (arrive.expect_tx).
template <int NB>
__device__ __forceinline__ void tile_issue(TileSmemT<NB>* sm, int b, unsigned long long* bar,
                                           const TileDesc& d, const long long* ptr,
                                           const int* idx, const double* val) {
  TileBuf* B = &sm->buf[b];
  sm->desc[b][0] = d.r0; sm->desc[b][1] = d.r1; sm->desc[b][2] = d.p0; sm->desc[b][3] = d.p1;
  const long long rs = d.r0 & ~1LL, re = (d.r1 + 2) & ~1LL;     // covers rp[r0..r1]
  const unsigned rb = (unsigned)((re - rs) * sizeof(long long));
  const bool stage = d.p1 > d.p0 && d.p1 - d.p0 <= TILE_NNZ;
  const long long vs = d.p0 & ~1LL, ve = (d.p1 + 1) & ~1LL;
  const long long is = d.p0 & ~3LL, ie = (d.p1 + 3) & ~3LL;
  const unsigned vb = stage ? (unsigned)((ve - vs) * sizeof(double)) : 0u;
  const unsigned ib = stage ? (unsigned)((ie - is) * sizeof(int)) : 0u;
  mbar_expect_tx(bar, rb + vb + ib);
  bulk_g2s(B->rp, ptr + rs, rb, bar);
  if (stage) {
    bulk_g2s(B->val, val + vs, vb, bar);
    bulk_g2s(B->idx, idx + is, ib, bar);
  }
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
  unsigned int* spec;      // speculative level-2 histogram (global) of the keys whose level-1
  int pred;                // digit is `pred` (the last iteration's bucket), or nullptr
};

__device__ __forceinline__ void colkey_epilogue(const ColKeyEpi* ep, int j, double sj, double vj,
                                                double& Vp, double& Emax, double g) {
  if (ep->pending) Vp += vj * vj;
  const double eps = g > 0.0 ? __ddiv_rn(__dmul_rn(sj, sj), g) : 0.0;
  Emax = fmax(Emax, eps);
  const unsigned long long key = sel_key(eps, (unsigned long long)j, ep->k, 0u, ep->seed, ep->greedy);
  ep->keys[j] = key;
  atomicAdd(&ep->hist[key >> L1_SHIFT], 1u);
  if (ep->spec && (int)(key >> L1_SHIFT) == ep->pred) atomicAdd(&ep->spec[(key >> L2_SHIFT) & 0xFFFull], 1u);
}

// Row results of pass N / the exact mode: outputs and the W / ||b - A x||^2
// (or ||o1||^2) partials; bv = b[row] loaded ahead by the caller.
__device__ __forceinline__ void tile_row_out(int row, double s1, double s2, bool has_b, double bv,
                                             double* o1, double* o2, double& Wp, double& Yp,
                                             int acc1) {
  o1[row] = s1;
  o2[row] = s2;
  if (has_b) {
    const double y = bv - s2;
    Wp += s1 * s1;
    Yp += y * y;
  }
  if (acc1) Wp += s1 * s1;
}

// Key epilogue of the pending pass-T columns (thread lt takes entries lt, lt + TG).
__device__ __forceinline__ void tile_flush(const ColKeyEpi* ep, TilePend* pd, int npend, int lt,
                                           double& Vp, double& Emax) {
  for (int e = lt; e < npend; e += TG) {
    const int j = pd->row[e];
    colkey_epilogue(ep, j, pd->s1[e], pd->s2[e], Vp, Emax, ep->gamma[j]);
  }
}

// One staged tile's rows, (1 << LV) lanes per row: R[r] = ptr[r0 + r],
// V[q] = val[p0 + q], I[q] = idx[p0 + q] in shared memory.
struct TileRows {
  const long long* R;
  const double* V;
  const int* I;
  long long p0;
  int r0, nr, lane, lw;
  bool has_b;
  const double* b;
  const double* in1;
  const double* in2;
  int use2;
  double* o1;
  double* o2;
  const ColKeyEpi* ep;
  int acc1;
  TilePend* pend;
  int npend;
};

template <int LV>
__device__ __forceinline__ void tile_rows(const TileRows& t, double& Wp, double& Yp) {
  constexpr int v = 1 << LV, spw = 32 >> LV;
  const int sub = t.lane >> LV, sl = t.lane & (v - 1);
  for (int base = t.lw * spw; base < t.nr; base += (TG / 32) * spw) {   // warp-uniform bounds
    const int r = base + sub;
    const bool valid = r < t.nr;
    double s1 = 0.0, s2 = 0.0;
    const double bv = t.has_b && valid && sl == 0 ? t.b[t.r0 + r] : 0.0;   // ahead of the gathers
    if (valid) {
      int q = (int)(t.R[r] - t.p0) + sl;
      const int q1 = (int)(t.R[r + 1] - t.p0);
      // RU entries per lane per round, predicated: one gather round trip
      // covers a whole row of up to RU * v entries
      constexpr int RU = LV == 5 ? RG_RU5 : RG_RU;
      for (; q < q1; q += RU * v) {
        int c[RU];
        double g1[RU], g2[RU];
#pragma unroll
        for (int e = 0; e < RU; ++e) c[e] = q + e * v < q1 ? t.I[q + e * v] : -1;
#pragma unroll
        for (int e = 0; e < RU; ++e) {
          g1[e] = c[e] >= 0 ? t.in1[c[e]] : 0.0;
          g2[e] = (t.use2 && c[e] >= 0) ? t.in2[c[e]] : 0.0;
        }
#pragma unroll
        for (int e = 0; e < RU; ++e) {
          if (c[e] >= 0) {
            const double a = t.V[q + e * v];
            s1 = fma(a, g1[e], s1);
            s2 = fma(a, g2[e], s2);
          }
        }
      }
    }
#pragma unroll
    for (int o = v >> 1; o > 0; o >>= 1) {         // fixed shuffle tree (deterministic)
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (valid && sl == 0) {
      const int row = t.r0 + r;
      if (t.ep) {
        t.o1[row] = s1;
        t.o2[row] = s2;
        const int e = t.npend + r;
        t.pend->s1[e] = s1; t.pend->s2[e] = s2; t.pend->row[e] = row;
      } else {
        tile_row_out(row, s1, s2, t.has_b, bv, t.o1, t.o2, Wp, Yp, t.acc1);
      }
    }
  }
}

// NB: ring depth (TBUF in the persistent kernels, GRAPH_TBUF in the graph engine's k_csr_tiles).
template <int NB = TBUF>
__device__ void csr_tiles(int gid, int ngroups, int lt, int bar_id, TileSmemT<NB>* sm, TileRing& ring,
                          const long long* __restrict__ ptr, const int* __restrict__ idx,
                          const double* __restrict__ val, const int* __restrict__ tiles,
                          const long long* __restrict__ tilep, int ntiles,
                          const double* in1, const double* in2, int use2,
                          const double* __restrict__ b, double* o1, double* o2,
                          double& Wp, double& Yp,
                          const ColKeyEpi* ep = nullptr, int acc1 = 0, int vec = 1,
                          int rev = 0) {
  // tiles gid, gid + ngroups, ...: at any moment the groups of the whole GPU stream one
  // contiguous window of the matrix (measured faster on C3 than a contiguous run of
  // tiles per group: -12 %)
  const int tb = gid, tstep = ngroups;
  const int cnt = gid < ntiles ? (ntiles - gid + ngroups - 1) / ngroups : 0;
  // the staging buffers may have been scratch of another phase (generic-proxy
  // writes): order those before the async-proxy (TMA) writes below
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  group_bar(bar_id);
  unsigned long long* full = ring.full;
  unsigned long long* rel = ring.full + NB;      // per-buffer count of warps done with it
  if (lt == 0) {
    for (int i = 0; i < cnt && i < NB; ++i) {
      const unsigned u = ring.used + i;
      const int ti = tb + i * tstep;
      tile_issue(sm, u % NB, &full[u % NB], tile_desc(rev ? ntiles - 1 - ti : ti, tiles, tilep),
                 ptr, idx, val);
    }
  }
  const int lane = lt & 31, lw = lt >> 5;
  const int lvec = __ffs(vec) - 1;                 // vec is a power of two
  const bool has_b = b != nullptr;
  int npend = 0;                                   // pass T: columns awaiting their keys
  for (int i = 0; i < cnt; ++i) {
    const int t = tb + i * tstep;                  // (reversed below when rev)
    const unsigned u = ring.used + i, bi = u % NB;
    // every warp's lane 0 fetches the descriptor of the tile this buffer is
    // refilled with (the last warp to release the buffer issues the refill)
    TileDesc nd{0, 0, 0, 0};
    const bool refill = lane == 0 && i + NB < cnt;
    if (refill) {
      const int tn = t + NB * tstep;
      nd = tile_desc(rev ? ntiles - 1 - tn : tn, tiles, tilep);
    }
    mbar_wait(&full[bi], (u / NB) & 1u);
    const int r0 = (int)sm->desc[bi][0], nr = (int)(sm->desc[bi][1] - sm->desc[bi][0]);
    const long long p0 = sm->desc[bi][2], p1 = sm->desc[bi][3];
    if (ep && npend + nr > PEND) {                 // make room in the pending list
      group_bar(bar_id);                           // every warp's entries are written
      tile_flush(ep, &sm->pend, npend, lt, Wp, Yp);
      npend = 0;
      group_bar(bar_id);
    }
    if (p1 - p0 > TILE_NNZ) {                      // one long row: group-wide reduction
      double a1 = 0.0, a2 = 0.0;
      const double bv = has_b && lt == 0 ? b[r0] : 0.0;
      for (long long p = p0 + lt; p < p1; p += TG) {
        const double a = ld_stream(val + p);
        const int c = __ldg(idx + p);
        a1 = fma(a, ld_weak(in1 + c), a1);
        if (use2) a2 = fma(a, ld_weak(in2 + c), a2);
      }
      a1 = warp_sum(a1);
      a2 = warp_sum(a2);
      if (lane == 0) { sm->red[2 * lw] = a1; sm->red[2 * lw + 1] = a2; }
      group_bar(bar_id);
      if (lt == 0) {
        double s1 = 0.0, s2 = 0.0;
        for (int q = 0; q < TG / 32; ++q) { s1 += sm->red[2 * q]; s2 += sm->red[2 * q + 1]; }
        if (ep) {
          o1[r0] = s1;
          o2[r0] = s2;
          sm->pend.s1[npend] = s1; sm->pend.s2[npend] = s2; sm->pend.row[npend] = r0;
        } else {
          tile_row_out(r0, s1, s2, has_b, bv, o1, o2, Wp, Yp, acc1);
        }
      }
      group_bar(bar_id);                           // red[] is free for the next long row
    } else {
      // lanes per row for this tile: the mean-length choice `vec`, raised so the
      // tile's rows cover the whole group (a tile of few long rows still keeps
      // every thread busy); a power of two <= 32, uniform across the tile
      int lv = lvec;                               // shifts only: no integer division
      while (lv < 5 && (nr << (lv + 1)) <= TG) ++lv;
      const TileBuf& B = sm->buf[bi];
      const TileRows tr{B.rp + (r0 & 1), B.val + (p0 & 1), B.idx + (p0 & 3), p0, r0, nr, lane, lw,
                        has_b, b, in1, in2, use2, o1, o2, ep, acc1, &sm->pend, npend};
      switch (lv) {                                // lanes per row as a compile-time constant
        case 0: tile_rows<0>(tr, Wp, Yp); break;
        case 1: tile_rows<1>(tr, Wp, Yp); break;
        case 2: tile_rows<2>(tr, Wp, Yp); break;
        case 3: tile_rows<3>(tr, Wp, Yp); break;
        case 4: tile_rows<4>(tr, Wp, Yp); break;
        default: tile_rows<5>(tr, Wp, Yp); break;
      }
    }
    npend += nr;
    // release buffer bi: each warp once its lanes are done with it; the last
    // of the group's warps refills it, so no warp ever waits for another here
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
  group_bar(bar_id);                               // buffers and pend list free for the next call
  if (ep) tile_flush(ep, &sm->pend, npend, lt, Wp, Yp);
  ring.used += cnt;
}

}  // namespace rg
