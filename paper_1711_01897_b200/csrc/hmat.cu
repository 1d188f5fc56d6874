// Device H-matrix assembly: near-field dense leaves + lock-step batched ACA
// over every admissible leaf (assemble_hmatrix, hmatrix.py:759-811).
//
// The reference runs aca() (hmatrix.py:271-382) block by block on the host,
// each step issuing one row job and one column job (hmatrix.py:625-672).
// Here all admissible blocks advance together in "waves": one launch
// evaluates the next ACA row of every active block (one CTA per block:
// integrals + residual update + column pivot search), a second launch the
// pivot column (integrals + residual + stopping test + Frobenius update +
// next row pivot).  Per-block decisions follow aca() exactly:
//   * first row = lowest unused index; next row = argmax |u_k| over rows not
//     yet used or retired (first index on ties, hmatrix.py:301-314);
//   * column pivot = argmax |residual row| over unused columns (329-332);
//   * vanishing residual row -> row retired to Z, next = lowest unused (334-338);
//   * update u v^T with |u||v| <= eps ||S_k||_F is dropped and the row retired;
//     two such updates in a row stop the block (347-357, 369-370);
//   * ||S_k||_F^2 updated incrementally with the cross terms (359-362).
// Factors live in a device pool: each accepted rank-1 term (u, v) is one
// contiguous record [u (h values) | v (w values)], its pool offset kept in a
// per-block term table.  Payload rules follow lowrank_leaf
// (hmatrix.py:721-735): converged and rank (h + w) < h w -> low rank,
// converged otherwise -> dense u v^T, rank cap without convergence -> dense
// exact rows.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include <cub/cub.cuh>

#include "hbem_internal.h"

namespace hb {

// ---------------------------------------------------------------------------
// value arithmetic (real T or complex as (re, im) pairs, numpy layout)
// ---------------------------------------------------------------------------
template <typename T> struct Cx { T re, im; };

template <typename T, bool C> struct Num;
template <typename T> struct Num<T, false> {
  using V = T;
  __device__ static V mk(T r, T) { return r; }
  __device__ static V fms(V a, V b, V c) { return a - b * c; }
  __device__ static double abs(V a) { return fabs((double)a); }
  __device__ static double nrm(V a) { return (double)a * (double)a; }
  __device__ static void cdot(double &re, double &, V a, V b) { re += (double)a * (double)b; }
  __device__ static V div(V a, V b) { return a / b; }
  __device__ static V zero() { return T(0); }
  __device__ static V fma_acc(V acc, V a, V b) { return acc + a * b; }
};
template <typename T> struct Num<T, true> {
  using V = Cx<T>;
  __device__ static V mk(T r, T i) { return V{r, i}; }
  __device__ static V fms(V a, V b, V c) {
    return V{a.re - (b.re * c.re - b.im * c.im), a.im - (b.re * c.im + b.im * c.re)};
  }
  __device__ static double abs(V a) { return hypot((double)a.re, (double)a.im); }
  __device__ static double nrm(V a) {
    return (double)a.re * (double)a.re + (double)a.im * (double)a.im;
  }
  __device__ static void cdot(double &re, double &im, V a, V b) {  // conj(a) b
    re += (double)a.re * (double)b.re + (double)a.im * (double)b.im;
    im += (double)a.re * (double)b.im - (double)a.im * (double)b.re;
  }
  __device__ static V div(V a, V b) {
    const T d = b.re * b.re + b.im * b.im;
    return V{(a.re * b.re + a.im * b.im) / d, (a.im * b.re - a.re * b.im) / d};
  }
  __device__ static V zero() { return V{T(0), T(0)}; }
  __device__ static V fma_acc(V acc, V a, V b) {
    return V{acc.re + (a.re * b.re - a.im * b.im), acc.im + (a.re * b.im + a.im * b.re)};
  }
};

// ---------------------------------------------------------------------------
// problem view: geometry + DOF maps
// ---------------------------------------------------------------------------
template <typename T> struct Prob {
  Geo<T> g;
  RuleTab<T> R;
  Geo64 G64;
  const int4 *elem;
  const int *rperm, *cperm;  // tree position -> DOF
  // DOF -> (element, local) incidence CSR (linear spaces)
  const int *tptr, *tel;
  const signed char *tloc;
  const int *sptr, *sel;
  const signed char *sloc;
};

// block of one element pair (any adjacency), thread-level
template <typename T, int OP, bool HELM, int NT, int NS>
__device__ __forceinline__ void pair_block(const Prob<T> &P, int e, int f, T (&re)[NT][NS],
                                           T (&im)[NT][NS], unsigned long long *nsing) {
  if (touching(P.elem[e], P.elem[f])) {
    double dr[NT][NS], di[NT][NS];
    singular_local<OP, HELM, NT, NS, 1>(P.G64, e, f, dr, di);
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
      for (int j = 0; j < NS; ++j) { re[i][j] = (T)dr[i][j]; im[i][j] = (T)di[i][j]; }
    if (nsing) atomicAdd(nsing, 1ull);
    return;
  }
  T x[18], y[18], na[4], nb[4];
  load_q<T>(P.g.q, e, x);
  load_q<T>(P.g.q, f, y);
  load_nj<T>(P.g.nj, e, na);
  load_nj<T>(P.g.nj, f, nb);
  const T *ca = nullptr, *cb = nullptr;
  if (OP == HBEM_HYPS) { ca = P.g.curl + 9 * (int64_t)e; cb = P.g.curl + 9 * (int64_t)f; }
  regular_pair<T, OP, HELM, NT, NS>(P.R, x, y, na, nb, ca, cb, re, im);
}

// Matrix entry (test DOF di, trial DOF dj): sum over the element pairs that
// carry both DOFs, in (test element asc, trial element asc) order — the
// accumulation order of _row_job/_col_job/dense_leaf (hmatrix.py:625-699).
template <typename T, bool C, int OP, bool HELM, int NT, int NS>
__device__ __forceinline__ typename Num<T, C>::V entry(const Prob<T> &P, int di, int dj,
                                                        unsigned long long *nsing) {
  using N = Num<T, C>;
  if (NT == 1 && NS == 1) {
    T re[1][1], im[1][1];
    pair_block<T, OP, HELM, 1, 1>(P, di, dj, re, im, nsing);
    return N::mk(re[0][0], im[0][0]);
  }
  typename N::V acc = N::zero();
  const int t0 = NT == 1 ? di : P.tptr[di], t1 = NT == 1 ? di + 1 : P.tptr[di + 1];
  const int s0 = NS == 1 ? dj : P.sptr[dj], s1 = NS == 1 ? dj + 1 : P.sptr[dj + 1];
  for (int t = t0; t < t1; ++t) {
    const int e = NT == 1 ? di : P.tel[t];
    const int a = NT == 1 ? 0 : P.tloc[t];
    for (int s = s0; s < s1; ++s) {
      const int f = NS == 1 ? dj : P.sel[s];
      const int b = NS == 1 ? 0 : P.sloc[s];
      T re[NT][NS], im[NT][NS];
      pair_block<T, OP, HELM, NT, NS>(P, e, f, re, im, nsing);
      T vr = T(0), vi = T(0);
#pragma unroll
      for (int u = 0; u < NT; ++u)
#pragma unroll
        for (int v = 0; v < NS; ++v)
          if (u == a && v == b) { vr = re[u][v]; vi = im[u][v]; }
      typename N::V val = N::mk(vr, vi);
      if constexpr (C) { acc.re += val.re; acc.im += val.im; }
      else acc += val;
    }
  }
  return acc;
}

// ---------------------------------------------------------------------------
// ACA state
// ---------------------------------------------------------------------------
enum : int { ST_ACTIVE = 0, ST_CONVERGED = 1, ST_FALLBACK = 2, ST_OVERFLOW = 3, ST_POOL = 4 };

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kE = 2;                  // entries per integration thread
constexpr int kChunk = kThreads * kE;  // entries per integration CTA

// Each accepted rank-1 term is one pool record [u (h) | v (w)]; v is stored
// scaled (v = row / pivot, hmatrix.py:339) once the update is accepted.
struct AcaDev {
  const int *h, *w, *r0, *c0;
  int *rank, *cur, *pcol, *small, *status, *exhausted;
  double *norm2, *resid, *rn2, *piv;  // piv: pivot of the pending row (re, im)
  long long *pend, *terms;
  int tmax;
  unsigned *rmask, *cmask;
  const long long *rmask_off, *cmask_off;
  void *pool;
  long long pool_cap, pool_base;
  int kmax_cfg;
  double eps;
  // wave lists: A (row phase), C (column phase), A2 (next wave)
  const int *listA;
  const longlong2 *needA, *scanA;  // (chunks, pool values) per position, inclusive scan
  int *listC;
  long long *needC;                // column chunks per position
  const long long *scanC;
  int *listA2;
  longlong2 *needA2;
  int *counts;                     // [0] |C|, [1] |A2|, [2] singular queue length
  int2 *squeue;                    // (position, entry index) of touching P0 pairs
  int squeue_cap;
  unsigned long long *stat;        // [0] entries evaluated, [1] singular pairs
  struct Job *jobs;                // per position of the current phase
  int *cmap;                       // chunk -> position
  void *coef;                      // per position: tmax residual coefficients
};

__device__ __forceinline__ bool better(double a, int ia, double b, int ib) {
  return a > b || (a == b && ia < ib);
}
__device__ __forceinline__ void warp_argmax_sum(double &best, int &bidx, double &sum) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (better(ob, oi, best, bidx)) { best = ob; bidx = oi; }
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
  }
}
__device__ __forceinline__ bool bit(const unsigned *m, int i) { return (m[i >> 5] >> (i & 31)) & 1u; }
__device__ __forceinline__ void set_bit(unsigned *m, int i) { atomicOr(m + (i >> 5), 1u << (i & 31)); }

// lowest index without its bit set (padding bits preset), or -1
__device__ int first_clear(const unsigned *m, int n) {
  const int nw = (n + 31) >> 5;
  for (int k = 0; k < nw; ++k) {
    const unsigned v = ~m[k];
    if (v) {
      const int i = (k << 5) + __ffs(v) - 1;
      return i < n ? i : -1;
    }
  }
  return -1;
}

__device__ __forceinline__ int upper_pos(const long long *scan, int n, long long x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (scan[mid] > x) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}
__device__ __forceinline__ int upper_pos2(const longlong2 *scan, int n, long long x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (scan[mid].x > x) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

__device__ __forceinline__ long long row_slot(const AcaDev &S, int pos, int b) {
  const long long pe = S.pend[b];
  return pe >= 0 ? pe : S.pool_base + S.scanA[pos].y - S.needA[pos].y;
}

__host__ __device__ __forceinline__ long long chunks_of(int n) { return (n + kChunk - 1) / kChunk; }

// regular P0 pair value with the element data of one side already loaded
template <typename T, bool C, int OP, bool HELM>
__device__ __forceinline__ typename Num<T, C>::V p0_value(const Prob<T> &P, const T (&x)[18],
                                                          const T (&na)[4], int f) {
  T y[18], nb[4], re[1][1], im[1][1];
  load_q<T>(P.g.q, f, y);
  load_nj<T>(P.g.nj, f, nb);
  regular_pair<T, OP, HELM, 1, 1>(P.R, x, y, na, nb, nullptr, nullptr, re, im);
  return Num<T, C>::mk(re[0][0], im[0][0]);
}
template <typename T, bool C, int OP, bool HELM>
__device__ __forceinline__ typename Num<T, C>::V p0_value_col(const Prob<T> &P, int e,
                                                              const T (&y)[18],
                                                              const T (&nb)[4]) {
  T x[18], na[4], re[1][1], im[1][1];
  load_q<T>(P.g.q, e, x);
  load_nj<T>(P.g.nj, e, na);
  regular_pair<T, OP, HELM, 1, 1>(P.R, x, y, na, nb, nullptr, nullptr, re, im);
  return Num<T, C>::mk(re[0][0], im[0][0]);
}

// ---------------------------------------------------------------------------
// Per-wave job tables.  After the chunk scan, one thread per job packs what
// the integration threads need (block shape, fixed element, pending pool
// slot, first chunk) into one record, fills the chunk -> job map and gathers
// the residual coefficients (row phase: u_l[i]; column phase: v_l[j]), so an
// integration thread reaches its geometry through two loads.
// ---------------------------------------------------------------------------
struct Job {
  int b, h, w, k;
  int fix;        // row phase: row i; column phase: column j
  int r0, c0;
  int elem;       // DOF of the fixed side (test DOF of row i / trial DOF of column j)
  long long pe;   // pending pool slot of this block
  long long cbase;
};

template <typename V>
__global__ void k_jobs(AcaDev S, const int *list, int n, int col_phase, const int *rperm,
                       const int *cperm) {
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= n) return;
  const int b = list[pos];
  Job J;
  J.b = b;
  J.h = S.h[b];
  J.w = S.w[b];
  J.k = S.rank[b];
  J.r0 = S.r0[b];
  J.c0 = S.c0[b];
  long long c1;
  if (!col_phase) {
    J.fix = S.cur[b];
    J.pe = row_slot(S, pos, b);
    J.elem = rperm[J.r0 + J.fix];
    J.cbase = pos ? S.scanA[pos - 1].x : 0;
    c1 = S.scanA[pos].x;
  } else {
    J.fix = S.pcol[b];
    J.pe = S.pend[b];
    J.elem = cperm[J.c0 + J.fix];
    J.cbase = pos ? S.scanC[pos - 1] : 0;
    c1 = S.scanC[pos];
  }
  for (long long ch = J.cbase; ch < c1; ++ch) S.cmap[ch] = pos;
  const V *pool = static_cast<const V *>(S.pool);
  V *coef = static_cast<V *>(S.coef) + (long long)pos * S.tmax;
  const long long *tl = S.terms + (long long)b * S.tmax;
  for (int l = 0; l < J.k; ++l)
    coef[l] = col_phase ? pool[tl[l] + J.h + J.fix] : pool[tl[l] + J.fix];
  S.jobs[pos] = J;
}

// ---------------------------------------------------------------------------
// K3a/K3b: ACA row / column integration.  One CTA = one chunk of kChunk
// entries of one job; each thread evaluates kE entries (integral, residual
// update with the gathered coefficients, store).  No barriers.
//   row:    val(c) = A(i, c) - sum_l u_l[i] v_l[c]   (hmatrix.py:323-327)
//   column: val(r) = A(r, j) - sum_l v_l[j] u_l[r]   (hmatrix.py:340-342)
// ---------------------------------------------------------------------------
template <typename T, bool C, int OP, bool HELM, int NT, int NS, bool COL>
__global__ void __launch_bounds__(kThreads) k_int(Prob<T> P, AcaDev S) {
  using N = Num<T, C>;
  using V = typename N::V;
  const int pos = S.cmap[blockIdx.x];
  const Job J = S.jobs[pos];
  const int base = (int)(blockIdx.x - J.cbase) * kChunk;
  const int n = COL ? J.h : J.w;
  if (base + (int)threadIdx.x >= n) return;
  V *pool = static_cast<V *>(S.pool);
  const V *coef = static_cast<const V *>(S.coef) + (long long)pos * S.tmax;
  const long long *tl = S.terms + (long long)J.b * S.tmax;
  const int vofs = COL ? 0 : J.h;  // residual factor read at [t + vofs + idx]
  V *dst = pool + J.pe + vofs;
  T x[18], nx[4];
  if constexpr (NT == 1 && NS == 1) {
    load_q<T>(P.g.q, J.elem, x);
    load_nj<T>(P.g.nj, J.elem, nx);
  }
  const int4 efix = P.elem[J.elem];
#pragma unroll 1
  for (int e = 0; e < kE; ++e) {
    const int idx = base + e * kThreads + threadIdx.x;
    if (idx >= n) break;
    const int dof = COL ? P.rperm[J.r0 + idx] : P.cperm[J.c0 + idx];
    V val;
    if constexpr (NT == 1 && NS == 1) {
      if (touching(efix, P.elem[dof])) {
        const int q = atomicAdd(S.counts + 2, 1);
        if (q < S.squeue_cap) S.squeue[q] = make_int2(pos, idx);
        continue;
      }
      if (COL) val = p0_value_col<T, C, OP, HELM>(P, dof, x, nx);
      else val = p0_value<T, C, OP, HELM>(P, x, nx, dof);
    } else {
      val = COL ? entry<T, C, OP, HELM, NT, NS>(P, dof, J.elem, S.stat + 1)
                : entry<T, C, OP, HELM, NT, NS>(P, J.elem, dof, S.stat + 1);
    }
    const int ro = COL ? 0 : J.h;  // where the other factor of term l lives
    for (int l = 0; l < J.k; ++l) val = N::fms(val, coef[l], pool[tl[l] + ro + idx]);
    dst[idx] = val;
  }
}

// touching P0 pairs queued by the integration kernels: warp per pair
// (Sauter-Schwab in float64, kernels.py:249-290), then the same residual.
template <typename T, bool C, int OP, bool HELM>
__global__ void __launch_bounds__(kThreads) k_int_singular(Prob<T> P, AcaDev S, int col_phase) {
  using N = Num<T, C>;
  using V = typename N::V;
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int n = min(S.counts[2], S.squeue_cap);
  V *pool = static_cast<V *>(S.pool);
  for (int q = warp; q < n; q += nw) {
    const int2 it = S.squeue[q];
    const Job J = S.jobs[it.x];
    const int idx = it.y;
    const int row = col_phase ? idx : J.fix, col = col_phase ? J.fix : idx;
    const int e = P.rperm[J.r0 + row], f = P.cperm[J.c0 + col];
    double re[1][1], im[1][1];
    singular_local<OP, HELM, 1, 1, 32>(P.G64, e, f, re, im);
    if (lane == 0) {
      V val = N::mk((T)re[0][0], (T)im[0][0]);
      const V *coef = static_cast<const V *>(S.coef) + (long long)it.x * S.tmax;
      const long long *tl = S.terms + (long long)J.b * S.tmax;
      const int ro = col_phase ? 0 : J.h;
      for (int l = 0; l < J.k; ++l) val = N::fms(val, coef[l], pool[tl[l] + ro + idx]);
      pool[J.pe + (col_phase ? 0 : J.h) + idx] = val;
      atomicAdd(S.stat + 1, 1ull);
    }
  }
}

// ---------------------------------------------------------------------------
// K3c: row finalize, warp per block: column pivot (argmax |row| over unused
// columns, first index on ties), vanishing-row test, schedule the column job.
// ---------------------------------------------------------------------------
template <typename T, bool C>
__global__ void __launch_bounds__(kThreads) k_fin_row(AcaDev S, int nA) {
  using N = Num<T, C>;
  using V = typename N::V;
  __shared__ unsigned long long s_ent[kWarps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int pos = blockIdx.x * kWarps + wid;
  unsigned long long ent = 0;
  if (pos < nA) {
    const int b = S.listA[pos];
    const int h = S.h[b], w = S.w[b], i = S.cur[b];
    const long long pe = row_slot(S, pos, b);
    const V *row = static_cast<const V *>(S.pool) + pe + h;
    const unsigned *cm = S.cmask + S.cmask_off[b];
    double best = -1.0, ss = 0.0;
    int bidx = 0x7fffffff;
    for (int c = lane; c < w; c += 32) {
      const V val = row[c];
      const double a = N::abs(val);
      ss += N::nrm(val);
      if (!bit(cm, c) && a > best) { best = a; bidx = c; }
    }
    warp_argmax_sum(best, bidx, ss);
    if (lane == 0) {
      ent = (unsigned long long)w;
      S.pend[b] = pe;
      if (best <= 0.0) {
        // residual row vanished: retire it to Z (hmatrix.py:334-338)
        unsigned *rm = S.rmask + S.rmask_off[b];
        set_bit(rm, i);
        const int next = first_clear(rm, h);
        if (next < 0) {
          S.status[b] = ST_CONVERGED;
          S.exhausted[b] = 1;
        } else {
          S.cur[b] = next;
          const int q = atomicAdd(S.counts + 1, 1);
          S.listA2[q] = b;
          S.needA2[q] = make_longlong2(chunks_of(w), 0);
        }
      } else {
        const V pv = row[bidx];
        S.pcol[b] = bidx;
        if constexpr (C) { S.piv[2 * b] = pv.re; S.piv[2 * b + 1] = pv.im; }
        else { S.piv[2 * b] = pv; S.piv[2 * b + 1] = 0.0; }
        S.rn2[b] = ss;
        const int q = atomicAdd(S.counts, 1);
        S.listC[q] = b;
        S.needC[q] = chunks_of(h);
      }
    }
  }
  if (lane == 0) s_ent[wid] = ent;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int k = 0; k < kWarps; ++k) t += s_ent[k];
    if (t) atomicAdd(S.stat, t);
  }
}

// ---------------------------------------------------------------------------
// K3d: column finalize, warp per block: |u||v| stopping test (two small
// updates in a row stop, hmatrix.py:343-357), Frobenius update with the
// cross terms (359-362), v = row / pivot, next row pivot argmax |u|.
// ---------------------------------------------------------------------------
template <typename T, bool C>
__global__ void __launch_bounds__(kThreads) k_fin_col(AcaDev S, int nC) {
  using N = Num<T, C>;
  using V = typename N::V;
  __shared__ unsigned long long s_ent[kWarps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int pos = blockIdx.x * kWarps + wid;
  unsigned long long ent = 0;
  if (pos < nC) {
    const int b = S.listC[pos];
    const int h = S.h[b], w = S.w[b], i = S.cur[b], j = S.pcol[b], k = S.rank[b];
    const long long pe = S.pend[b];
    V *pool = static_cast<V *>(S.pool);
    V *col = pool + pe;
    V *row = pool + pe + h;
    unsigned *rm = S.rmask + S.rmask_off[b];
    double best = -1.0, ss = 0.0;
    int bidx = 0x7fffffff;
    for (int r = lane; r < h; r += 32) {
      const V val = col[r];
      const double a = N::abs(val);
      ss += N::nrm(val);
      if (r != i && !bit(rm, r) && a > best) { best = a; bidx = r; }
    }
    warp_argmax_sum(best, bidx, ss);
    const int next = best >= 0.0 ? bidx : -1;
    const double pr = S.piv[2 * b], pim = S.piv[2 * b + 1];
    const double nu = sqrt(ss);
    const double nv = sqrt(S.rn2[b]) / hypot(pr, pim);
    const double upd = nu * nv;
    const double n2 = S.norm2[b];
    const int kmax_b = min(S.kmax_cfg, min(h, w));
    ent = (unsigned long long)h;
    if (n2 > 0.0 && upd <= S.eps * sqrt(n2)) {
      if (lane == 0) {
        S.resid[b] = upd / sqrt(n2);
        const int sm = S.small[b] + 1;
        S.small[b] = sm;
        if (sm >= 2) {
          S.status[b] = ST_CONVERGED;
        } else {
          set_bit(rm, i);
          if (next < 0) {
            S.status[b] = ST_CONVERGED;
            S.exhausted[b] = 1;
          } else {
            S.cur[b] = next;
            const int q = atomicAdd(S.counts + 1, 1);
            S.listA2[q] = b;
            S.needA2[q] = make_longlong2(chunks_of(w), 0);  // reuse the pending slot
          }
        }
      }
    } else {
      // accept: v = row / pivot in place, then the cross terms
      V pv;
      if constexpr (C) pv = V{(T)pr, (T)pim};
      else pv = (T)pr;
      for (int c = lane; c < w; c += 32) row[c] = N::div(row[c], pv);
      __syncwarp();
      double cross = 0.0;
      const long long *tl = S.terms + (long long)b * S.tmax;
      for (int l = 0; l < k; ++l) {
        const V *ul = pool + tl[l];
        const V *vl = ul + h;
        double ur = 0, ui = 0, vr = 0, vi = 0;
        for (int r = lane; r < h; r += 32) N::cdot(ur, ui, ul[r], col[r]);
        for (int c = lane; c < w; c += 32) N::cdot(vr, vi, vl[c], row[c]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          ur += __shfl_xor_sync(0xffffffffu, ur, o);
          ui += __shfl_xor_sync(0xffffffffu, ui, o);
          vr += __shfl_xor_sync(0xffffffffu, vr, o);
          vi += __shfl_xor_sync(0xffffffffu, vi, o);
        }
        cross += ur * vr - ui * vi;  // Re(vdot(u_l, u) * vdot(v_l, v))
      }
      if (lane == 0) {
        const double n2n = n2 + 2.0 * cross + upd * upd;
        S.norm2[b] = n2n;
        S.small[b] = 0;
        S.terms[(long long)b * S.tmax + k] = pe;
        S.pend[b] = -1;
        S.rank[b] = k + 1;
        set_bit(rm, i);
        set_bit(S.cmask + S.cmask_off[b], j);
        if (n2n > 0.0) {
          S.resid[b] = upd / sqrt(n2n);
          if (upd <= S.eps * sqrt(n2n)) S.small[b] = 1;
        }
        S.cur[b] = next;
        // loop head of the next iteration (hmatrix.py:318-322)
        if (k + 1 >= kmax_b) {
          S.status[b] = ST_FALLBACK;
        } else if (k + 1 >= S.tmax) {
          S.status[b] = ST_OVERFLOW;
        } else if (next < 0) {
          S.status[b] = ST_CONVERGED;
          S.exhausted[b] = 1;
        } else {
          const int q = atomicAdd(S.counts + 1, 1);
          S.listA2[q] = b;
          S.needA2[q] = make_longlong2(chunks_of(w), (long long)h + w);
        }
      }
    }
  }
  if (lane == 0) s_ent[wid] = ent;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int k = 0; k < kWarps; ++k) t += s_ent[k];
    if (t) atomicAdd(S.stat, t);
  }
}

// initial state; the wave-0 list is the size-sorted block order
__global__ void k_aca_init(AcaDev S, int n, const int *order, int *listA, longlong2 *needA) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int b = order[q];
  const int h = S.h[b], w = S.w[b];
  listA[q] = b;
  needA[q] = make_longlong2(chunks_of(w), (long long)h + w);
  S.rank[b] = 0;
  S.cur[b] = 0;
  S.small[b] = 0;
  S.status[b] = ST_ACTIVE;
  S.exhausted[b] = 0;
  S.norm2[b] = 0.0;
  S.resid[b] = INFINITY;
  S.pend[b] = -1;
  unsigned *rm = S.rmask + S.rmask_off[b];
  for (int k = 0; k < (h + 31) / 32; ++k) {
    const int valid = min(32, h - k * 32);
    rm[k] = valid == 32 ? 0u : ~((1u << valid) - 1u);
  }
  unsigned *cm = S.cmask + S.cmask_off[b];
  for (int k = 0; k < (w + 31) / 32; ++k) cm[k] = 0u;
}

__global__ void k_zero_ll2(longlong2 *p, int n) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) p[q] = make_longlong2(0, 0);
}
__global__ void k_zero_ll(long long *p, int n) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) p[q] = 0;
}

struct SumLL2 {
  __device__ __forceinline__ longlong2 operator()(const longlong2 &a, const longlong2 &b) const {
    return make_longlong2(a.x + b.x, a.y + b.y);
  }
};

// ---------------------------------------------------------------------------
// K4: dense entries (near-field leaves and ACA fallback blocks).
// tiles: (slot, first entry); slot -> (r0, c0, h, w, offset)
// P0 touching entries are queued for the warp-per-pair singular kernel.
// ---------------------------------------------------------------------------
struct DenseDev {
  const int *tile_slot;
  const int *tile_start;
  const int *r0, *c0, *h, *w;
  const long long *off;
  void *out;
  int *sing_slot;           // queued P0 touching entries
  long long *sing_pos;
  unsigned long long *sing_count;
  unsigned long long *stat;
};

template <typename T, bool C, int OP, bool HELM, int NT, int NS>
__global__ void __launch_bounds__(kThreads) k_dense(Prob<T> P, DenseDev D) {
  using N = Num<T, C>;
  using V = typename N::V;
  const int s = D.tile_slot[blockIdx.x];
  const int idx = D.tile_start[blockIdx.x] + threadIdx.x;
  const int h = D.h[s], w = D.w[s];
  if (idx >= h * w) return;
  const int i = idx / w, c = idx - (idx / w) * w;
  const int di = P.rperm[D.r0[s] + i], dj = P.cperm[D.c0[s] + c];
  V *out = static_cast<V *>(D.out) + D.off[s] + idx;
  if constexpr (NT == 1 && NS == 1) {
    if (touching(P.elem[di], P.elem[dj])) {
      const unsigned long long q = atomicAdd(D.sing_count, 1ull);
      D.sing_slot[q] = s;
      D.sing_pos[q] = D.off[s] + idx;
      return;
    }
    T x[18], y[18], na[4], nb[4], re[1][1], im[1][1];
    load_q<T>(P.g.q, di, x);
    load_q<T>(P.g.q, dj, y);
    load_nj<T>(P.g.nj, di, na);
    load_nj<T>(P.g.nj, dj, nb);
    regular_pair<T, OP, HELM, 1, 1>(P.R, x, y, na, nb, nullptr, nullptr, re, im);
    *out = N::mk(re[0][0], im[0][0]);
  } else {
    *out = entry<T, C, OP, HELM, NT, NS>(P, di, dj, D.stat + 1);
  }
}

// warp per queued P0 touching entry
template <typename T, bool C, int OP, bool HELM>
__global__ void __launch_bounds__(kThreads) k_dense_singular(Prob<T> P, DenseDev D) {
  using N = Num<T, C>;
  using V = typename N::V;
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long n = (long long)*D.sing_count;
  for (long long q = warp; q < n; q += nw) {
    const int s = D.sing_slot[q];
    const long long pos = D.sing_pos[q];
    const long long idx = pos - D.off[s];
    const int w = D.w[s];
    const int i = (int)(idx / w), c = (int)(idx - (idx / w) * w);
    const int e = P.rperm[D.r0[s] + i], f = P.cperm[D.c0[s] + c];
    double re[1][1], im[1][1];
    singular_local<OP, HELM, 1, 1, 32>(P.G64, e, f, re, im);
    if (lane == 0) static_cast<V *>(D.out)[pos] = N::mk((T)re[0][0], (T)im[0][0]);
  }
}

// dense u v^T expansion for converged blocks whose compression does not pay
template <typename T, bool C>
__global__ void k_expand(const int *slots, int n, AcaDev S, const long long *off, void *out) {
  using N = Num<T, C>;
  using V = typename N::V;
  const int q = blockIdx.x;
  if (q >= n) return;
  const int b = slots[q];
  const int h = S.h[b], w = S.w[b], k = S.rank[b];
  const V *pool = static_cast<const V *>(S.pool);
  V *o = static_cast<V *>(out) + off[q];
  for (long long idx = threadIdx.x; idx < (long long)h * w; idx += blockDim.x) {
    const int i = (int)(idx / w), c = (int)(idx % w);
    V acc = N::zero();
    for (int l = 0; l < k; ++l) {
      const V *t = pool + S.terms[(long long)b * S.tmax + l];
      acc = N::fma_acc(acc, t[i], t[h + c]);
    }
    o[idx] = acc;
  }
}

// pack the factors of low-rank blocks [first, last) into U/V staging
template <typename V>
__global__ void k_pack_factors(const int *slots, int n, AcaDev S, const long long *uoff,
                               const long long *voff, long long ubase, long long vbase, V *u,
                               V *v) {
  const int q = blockIdx.x;
  if (q >= n) return;
  const int b = slots[q];
  const int h = S.h[b], w = S.w[b], k = S.rank[b];
  const V *pool = static_cast<const V *>(S.pool);
  for (int l = 0; l < k; ++l) {
    const V *t = pool + S.terms[(long long)b * S.tmax + l];
    for (int r = threadIdx.x; r < h; r += blockDim.x)
      u[uoff[q] - ubase + (long long)l * h + r] = t[r];
    for (int c = threadIdx.x; c < w; c += blockDim.x)
      v[voff[q] - vbase + (long long)l * w + c] = t[h + c];
  }
}

}  // namespace hb

using namespace hb;

// ---------------------------------------------------------------------------
// host side: setup (partition upload, state allocation) and execute (waves)
// ---------------------------------------------------------------------------
struct hbem_hmat {
  hbem_ctx *ctx = nullptr;
  int device = 0;
  int64_t n_leaves = 0;
  bool complex_ = false;
  size_t vbytes = 8;
  int nt = 1, ns = 1;
  // per leaf results (host)
  std::vector<int32_t> kind, rank, flags;
  std::vector<int64_t> off_u, off_v, off_dense;
  std::vector<double> resid;
  // partition views (device)
  const int *rperm = nullptr, *cperm = nullptr;
  const int *tptr = nullptr, *tel = nullptr, *sptr = nullptr, *sel = nullptr;
  const signed char *tloc = nullptr, *sloc = nullptr;
  // admissible blocks
  int na = 0;
  std::vector<int> adm_leaf, ah, aw, ar0, ac0;
  int *d_order = nullptr, *listA = nullptr, *listA2 = nullptr;
  longlong2 *needA = nullptr, *needA2 = nullptr, *scanA = nullptr;
  long long *scanC = nullptr;
  void *cub_tmp = nullptr;
  size_t cub_bytes = 0;
  AcaDev S{};
  void *pool = nullptr;
  // near-field leaves
  int nd = 0;
  std::vector<int> den_leaf;
  long long nf_entries = 0;
  DenseDev D{};
  unsigned n_tiles = 0;
  long long nf_max_sing = 0;
  void *dense_nf = nullptr;
  // admissible blocks stored densely (after ACA)
  void *dense_adm = nullptr;
  size_t dense_adm_cap = 0;
  long long dense_entries = 0, u_entries = 0, v_entries = 0;
  std::vector<int> lowrank_slots;
  std::vector<int64_t> lr_uoff, lr_voff;
  cudaStream_t side = nullptr;
  cudaEvent_t side_done = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<void *> dev_allocs;
  hbem_hmat_stats stats{};
  double setup_s = 0.0;
  ~hbem_hmat() {
    cudaSetDevice(device);
    for (void *p : dev_allocs) cudaFree(p);
    cudaFree(pool);
    cudaFree(dense_nf);
    cudaFree(dense_adm);
    if (side) cudaStreamDestroy(side);
    if (side_done) cudaEventDestroy(side_done);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
  }
};

namespace {

using clk = std::chrono::steady_clock;
double secs(clk::time_point a, clk::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

template <typename X> int dalloc(hbem_hmat *H, X **p, size_t n) {
  void *q = nullptr;
  cudaError_t e = cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(X));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(HBEM_ERR_CAPACITY, "device allocation of %zu bytes failed: %s",
                     n * sizeof(X), cudaGetErrorString(e));
  }
  H->dev_allocs.push_back(q);
  *p = static_cast<X *>(q);
  return HBEM_OK;
}

template <typename X> int upload(hbem_hmat *H, X **p, const std::vector<X> &v) {
  HB_CHECK(dalloc(H, p, v.size()));
  if (!v.empty()) HB_CUDA(cudaMemcpy(*p, v.data(), v.size() * sizeof(X), cudaMemcpyHostToDevice));
  return HBEM_OK;
}

struct Incidence {
  std::vector<int> ptr, el;
  std::vector<signed char> loc;
};

// CSR DOF -> (element, local), stable in element order (hmatrix.py:531-541)
Incidence incidence(const int64_t *dofmap, int64_t m, int nl, int64_t n_dofs) {
  Incidence I;
  I.ptr.assign(n_dofs + 1, 0);
  for (int64_t e = 0; e < m; ++e)
    for (int a = 0; a < nl; ++a) I.ptr[dofmap[e * nl + a] + 1]++;
  for (int64_t d = 0; d < n_dofs; ++d) I.ptr[d + 1] += I.ptr[d];
  I.el.resize(m * nl);
  I.loc.resize(m * nl);
  std::vector<int> fill(I.ptr.begin(), I.ptr.end() - 1);
  for (int64_t e = 0; e < m; ++e)
    for (int a = 0; a < nl; ++a) {
      const int64_t d = dofmap[e * nl + a];
      I.el[fill[d]] = (int)e;
      I.loc[fill[d]] = (signed char)a;
      fill[d]++;
    }
  return I;
}

template <typename T> Prob<T> make_prob(const hbem_hmat *H) {
  Prob<T> P{};
  P.g = H->ctx->geo<T>();
  P.R = H->ctx->rule<T>();
  P.G64 = H->ctx->geo64();
  P.elem = H->ctx->elem;
  P.rperm = H->rperm;
  P.cperm = H->cperm;
  P.tptr = H->tptr; P.tel = H->tel; P.tloc = H->tloc;
  P.sptr = H->sptr; P.sel = H->sel; P.sloc = H->sloc;
  return P;
}

// one-time: partition / DOF maps / ACA state / pools on the device
int setup(hbem_hmat *H, const hbem_hmat_desc *d) {
  hbem_ctx *ctx = H->ctx;
  const int64_t m = ctx->m;
  const int nt = ctx->nt, ns = ctx->ns;
  H->nt = nt;
  H->ns = ns;
  {
    std::vector<int> rp(d->n_rows), cp(d->n_cols);
    for (int64_t i = 0; i < d->n_rows; ++i) rp[i] = (int)d->row_perm[i];
    for (int64_t i = 0; i < d->n_cols; ++i) cp[i] = (int)d->col_perm[i];
    int *a, *b;
    HB_CHECK(upload(H, &a, rp));
    HB_CHECK(upload(H, &b, cp));
    H->rperm = a;
    H->cperm = b;
  }
  if (nt == 3) {
    Incidence I = incidence(d->test_dofmap, m, 3, d->n_rows);
    int *p, *e;
    signed char *l;
    HB_CHECK(upload(H, &p, I.ptr));
    HB_CHECK(upload(H, &e, I.el));
    HB_CHECK(upload(H, &l, I.loc));
    H->tptr = p; H->tel = e; H->tloc = l;
  }
  if (ns == 3) {
    Incidence I = incidence(d->trial_dofmap, m, 3, d->n_cols);
    int *p, *e;
    signed char *l;
    HB_CHECK(upload(H, &p, I.ptr));
    HB_CHECK(upload(H, &e, I.el));
    HB_CHECK(upload(H, &l, I.loc));
    H->sptr = p; H->sel = e; H->sloc = l;
  }
  const int64_t L = d->n_leaves;
  H->n_leaves = L;
  H->kind.assign(L, 0);
  H->rank.assign(L, 0);
  H->flags.assign(L, 0);
  H->off_u.assign(L, -1);
  H->off_v.assign(L, -1);
  H->off_dense.assign(L, -1);
  H->resid.assign(L, 0.0);
  for (int64_t q = 0; q < L; ++q)
    (d->leaves[3 * q + 2] ? H->adm_leaf : H->den_leaf).push_back((int)q);
  auto rng = [&](const int64_t *nodes, int64_t n) {
    return std::pair<int, int>((int)nodes[5 * n], (int)(nodes[5 * n + 1] - nodes[5 * n]));
  };
  // ---- admissible blocks --------------------------------------------------------
  const int na = (int)H->adm_leaf.size();
  H->na = na;
  H->ah.resize(na); H->aw.resize(na); H->ar0.resize(na); H->ac0.resize(na);
  std::vector<long long> rmo(na), cmo(na);
  long long rmw = 0, cmw = 0, sum_hw = 0;
  for (int q = 0; q < na; ++q) {
    const int64_t lf = H->adm_leaf[q];
    auto [r0, h] = rng(d->row_nodes, d->leaves[3 * lf]);
    auto [c0, w] = rng(d->col_nodes, d->leaves[3 * lf + 1]);
    H->ar0[q] = r0; H->ah[q] = h; H->ac0[q] = c0; H->aw[q] = w;
    rmo[q] = rmw; rmw += (h + 31) / 32;
    cmo[q] = cmw; cmw += (w + 31) / 32;
    sum_hw += h + w;
  }
  AcaDev &S = H->S;
  int tmax = d->rank_capacity > 0 ? d->rank_capacity : 64;
  S.tmax = std::min(tmax, 256);
  S.kmax_cfg = d->k_max > 0 ? (int)std::min<int64_t>(d->k_max, 1 << 30) : (1 << 30);
  S.eps = d->epsilon;
  {
    int *p;
    HB_CHECK(upload(H, &p, H->ah)); S.h = p;
    HB_CHECK(upload(H, &p, H->aw)); S.w = p;
    HB_CHECK(upload(H, &p, H->ar0)); S.r0 = p;
    HB_CHECK(upload(H, &p, H->ac0)); S.c0 = p;
    long long *pl;
    HB_CHECK(upload(H, &pl, rmo)); S.rmask_off = pl;
    HB_CHECK(upload(H, &pl, cmo)); S.cmask_off = pl;
    // big blocks first (load balance of the CTA-per-block waves)
    std::vector<int> order(na);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return (long long)H->ah[a] * H->aw[a] > (long long)H->ah[b] * H->aw[b];
    });
    HB_CHECK(upload(H, &H->d_order, order));
  }
  HB_CHECK(dalloc(H, &S.rank, na));
  HB_CHECK(dalloc(H, &S.cur, na));
  HB_CHECK(dalloc(H, &S.pcol, na));
  HB_CHECK(dalloc(H, &S.small, na));
  HB_CHECK(dalloc(H, &S.status, na));
  HB_CHECK(dalloc(H, &S.exhausted, na));
  HB_CHECK(dalloc(H, &S.norm2, na));
  HB_CHECK(dalloc(H, &S.resid, na));
  HB_CHECK(dalloc(H, &S.rn2, na));
  HB_CHECK(dalloc(H, &S.piv, 2 * (size_t)na));
  HB_CHECK(dalloc(H, &S.pend, na));
  HB_CHECK(dalloc(H, &S.terms, (size_t)na * S.tmax));
  HB_CHECK(dalloc(H, &S.rmask, rmw));
  HB_CHECK(dalloc(H, &S.cmask, cmw));
  HB_CHECK(dalloc(H, &H->listA, na));
  HB_CHECK(dalloc(H, &H->listA2, na));
  HB_CHECK(dalloc(H, &S.listC, na));
  HB_CHECK(dalloc(H, &H->needA, na));
  HB_CHECK(dalloc(H, &H->needA2, na));
  HB_CHECK(dalloc(H, &H->scanA, na));
  HB_CHECK(dalloc(H, &S.needC, na));
  HB_CHECK(dalloc(H, &H->scanC, na));
  HB_CHECK(dalloc(H, &S.counts, 4));
  HB_CHECK(dalloc(H, &S.stat, 4));
  {
    // chunk map sized for the widest wave: every block's row and column
    long long maxch = 0;
    for (int q = 0; q < na; ++q)
      maxch += std::max(chunks_of(H->ah[q]), chunks_of(H->aw[q]));
    HB_CHECK(dalloc(H, &S.cmap, std::max<long long>(maxch, 1)));
    HB_CHECK(dalloc(H, &S.jobs, na));
    HB_CHECK(dalloc(H, (char **)&S.coef, (size_t)na * S.tmax * H->vbytes));
  }
  S.squeue_cap = 1 << 20;
  HB_CHECK(dalloc(H, &S.squeue, S.squeue_cap));
  {
    size_t b1 = 0, b2 = 0;
    HB_CUDA(cub::DeviceScan::InclusiveScan(nullptr, b1, H->needA, H->scanA, SumLL2(),
                                           std::max(na, 1)));
    HB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, b2, S.needC, H->scanC, std::max(na, 1)));
    H->cub_bytes = std::max(b1, b2);
    HB_CHECK(dalloc(H, (char **)&H->cub_tmp, H->cub_bytes));
  }
  // ---- near-field leaves --------------------------------------------------------
  const int nd = (int)H->den_leaf.size();
  H->nd = nd;
  std::vector<int> dr0(nd), dc0(nd), dh(nd), dw(nd);
  std::vector<long long> doff(nd);
  long long tot = 0;
  for (int q = 0; q < nd; ++q) {
    const int64_t lf = H->den_leaf[q];
    auto [r0, h] = rng(d->row_nodes, d->leaves[3 * lf]);
    auto [c0, w] = rng(d->col_nodes, d->leaves[3 * lf + 1]);
    dr0[q] = r0; dh[q] = h; dc0[q] = c0; dw[q] = w;
    doff[q] = tot;
    H->off_dense[lf] = tot;
    tot += (long long)h * w;
  }
  H->nf_entries = tot;
  {
    std::vector<int> tslot, tstart;
    tslot.reserve(tot / kThreads + nd);
    tstart.reserve(tot / kThreads + nd);
    for (int s = 0; s < nd; ++s) {
      const long long hw = (long long)dh[s] * dw[s];
      for (long long t = 0; t < hw; t += kThreads) {
        tslot.push_back(s);
        tstart.push_back((int)t);
      }
    }
    H->n_tiles = (unsigned)tslot.size();
    DenseDev &D = H->D;
    int *p;
    long long *pl;
    HB_CHECK(upload(H, &p, tslot)); D.tile_slot = p;
    HB_CHECK(upload(H, &p, tstart)); D.tile_start = p;
    HB_CHECK(upload(H, &p, dr0)); D.r0 = p;
    HB_CHECK(upload(H, &p, dc0)); D.c0 = p;
    HB_CHECK(upload(H, &p, dh)); D.h = p;
    HB_CHECK(upload(H, &p, dw)); D.w = p;
    HB_CHECK(upload(H, &pl, doff)); D.off = pl;
    HB_CHECK(dalloc(H, &D.sing_count, 1));
    HB_CHECK(dalloc(H, &D.stat, 2));
    if (nt == 1 && ns == 1) {
      // touching P0 pairs: at most ~13 per element; bound by the entry count
      H->nf_max_sing = std::min<long long>(tot, 32 * (m + 1));
      HB_CHECK(dalloc(H, &D.sing_slot, H->nf_max_sing));
      HB_CHECK(dalloc(H, &D.sing_pos, H->nf_max_sing));
    }
  }
  const size_t vb = H->vbytes;
  HB_CUDA(cudaMalloc(&H->dense_nf, std::max<size_t>((size_t)tot * vb, vb)));
  H->D.out = H->dense_nf;
  // ---- factor pool: what is left after a margin for the admissible-dense arena
  size_t free_b = 0, total_b = 0;
  HB_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const size_t want = (size_t)sum_hw * (size_t)std::min(S.tmax, 24) * vb;
  const size_t reserve = ((size_t)4 << 30) + (size_t)(0.02 * (double)free_b);
  size_t cap_b = free_b > reserve ? free_b - reserve : 0;
  cap_b = std::min(cap_b, std::max(want, (size_t)1 << 20));
  HB_CUDA(cudaMalloc(&H->pool, std::max<size_t>(cap_b, vb)));
  S.pool = H->pool;
  S.pool_cap = (long long)(cap_b / vb);
  HB_CUDA(cudaStreamCreateWithFlags(&H->side, cudaStreamNonBlocking));
  HB_CUDA(cudaEventCreateWithFlags(&H->side_done, cudaEventDisableTiming));
  for (auto &e : H->ev) HB_CUDA(cudaEventCreate(&e));
  return HBEM_OK;
}

template <typename T, bool C> int execute_t(hbem_hmat *H, cudaStream_t st) {
  using V = typename Num<T, C>::V;
  hbem_ctx *ctx = H->ctx;
  const auto t0 = clk::now();
  Prob<T> P = make_prob<T>(H);
  AcaDev &S = H->S;
  const int nt = H->nt, ns = H->ns;
  const int na = H->na;
  int64_t launches = 0;
  hbem_hmat_stats &ST = H->stats;
  const hbem_hmat_stats zero{};
  ST = zero;
  // ---- near-field leaves on the side stream (overlaps the ACA waves) ---------
  cudaEvent_t start_ev;
  HB_CUDA(cudaEventCreateWithFlags(&start_ev, cudaEventDisableTiming));
  HB_CUDA(cudaEventRecord(start_ev, st));
  HB_CUDA(cudaStreamWaitEvent(H->side, start_ev, 0));
  cudaEventDestroy(start_ev);
  HB_CUDA(cudaEventRecord(H->ev[2], H->side));
  if (H->nd > 0) {
    HB_CUDA(cudaMemsetAsync(H->D.sing_count, 0, 8, H->side));
    HB_CUDA(cudaMemsetAsync(H->D.stat, 0, 16, H->side));
    int rc = dispatch_op(ctx->op, ctx->helm, nt, ns, [&](auto OPc, auto Hc, auto NTc,
                                                         auto NSc) -> int {
      constexpr int OP = decltype(OPc)::value;
      constexpr bool HH = decltype(Hc)::value != 0;
      constexpr int NT = decltype(NTc)::value, NS = decltype(NSc)::value;
      k_dense<T, C, OP, HH, NT, NS><<<H->n_tiles, kThreads, 0, H->side>>>(P, H->D);
      HB_CUDA(cudaGetLastError());
      ++launches;
      if constexpr (NT == 1 && NS == 1) {
        k_dense_singular<T, C, OP, HH><<<148 * 16, kThreads, 0, H->side>>>(P, H->D);
        HB_CUDA(cudaGetLastError());
        ++launches;
      }
      return HBEM_OK;
    });
    if (rc != HBEM_OK) return rc;
  }
  HB_CUDA(cudaEventRecord(H->side_done, H->side));
  HB_CUDA(cudaEventRecord(H->ev[3], H->side));
  // ---- ACA waves ------------------------------------------------------------------
  HB_CUDA(cudaMemsetAsync(S.stat, 0, 32, st));
  int waves = 0;
  long long pool_top = 0;
  if (na > 0) {
    k_aca_init<<<(na + 127) / 128, 128, 0, st>>>(S, na, H->d_order, H->listA, H->needA);
    HB_CUDA(cudaGetLastError());
    ++launches;
    int nA = na;
    int *la = H->listA, *la2 = H->listA2;
    longlong2 *na_ = H->needA, *na2 = H->needA2;
    // per wave: scan(row chunks, pool) -> int_row -> singular -> fin_row ->
    // scan(col chunks) -> int_col -> singular -> fin_col; 2 host syncs
    while (nA > 0) {
      S.listA = la;
      S.needA = na_;
      S.scanA = H->scanA;
      S.listA2 = la2;
      S.needA2 = na2;
      S.scanC = H->scanC;
      HB_CUDA(cudaEventRecord(H->ev[0], st));
      size_t tb = H->cub_bytes;
      HB_CUDA(cub::DeviceScan::InclusiveScan(H->cub_tmp, tb, na_, H->scanA, SumLL2(), nA, st));
      longlong2 tot;
      HB_CUDA(cudaMemcpyAsync(&tot, H->scanA + nA - 1, sizeof(tot), cudaMemcpyDeviceToHost, st));
      HB_CUDA(cudaMemsetAsync(S.counts, 0, 16, st));
      k_zero_ll<<<(nA + 255) / 256, 256, 0, st>>>(S.needC, nA);
      k_zero_ll2<<<(nA + 255) / 256, 256, 0, st>>>(na2, nA);
      HB_CUDA(cudaStreamSynchronize(st));
      if (pool_top + tot.y > S.pool_cap)
        return set_error(HBEM_ERR_CAPACITY,
                         "ACA factor pool of %lld values exhausted at wave %d (need %lld more)",
                         (long long)S.pool_cap, waves, (long long)(pool_top + tot.y - S.pool_cap));
      S.pool_base = pool_top;
      pool_top += tot.y;
      const unsigned row_chunks = (unsigned)tot.x;
      int rc = dispatch_op(ctx->op, ctx->helm, nt, ns, [&](auto OPc, auto Hc, auto NTc,
                                                           auto NSc) -> int {
        constexpr int OP = decltype(OPc)::value;
        constexpr bool HH = decltype(Hc)::value != 0;
        constexpr int NT = decltype(NTc)::value, NS = decltype(NSc)::value;
        k_jobs<V><<<(nA + 127) / 128, 128, 0, st>>>(S, la, nA, 0, P.rperm, P.cperm);
        HB_CUDA(cudaGetLastError());
        k_int<T, C, OP, HH, NT, NS, false><<<row_chunks, kThreads, 0, st>>>(P, S);
        HB_CUDA(cudaGetLastError());
        if constexpr (NT == 1 && NS == 1) {
          k_int_singular<T, C, OP, HH><<<148 * 4, kThreads, 0, st>>>(P, S, 0);
          HB_CUDA(cudaGetLastError());
        }
        return HBEM_OK;
      });
      if (rc != HBEM_OK) return rc;
      k_fin_row<T, C><<<(nA + kWarps - 1) / kWarps, kThreads, 0, st>>>(S, nA);
      HB_CUDA(cudaGetLastError());
      size_t tb2 = H->cub_bytes;
      HB_CUDA(cub::DeviceScan::InclusiveSum(H->cub_tmp, tb2, S.needC, H->scanC, nA, st));
      int cnt[3];
      long long col_chunks = 0;
      HB_CUDA(cudaMemcpyAsync(cnt, S.counts, 12, cudaMemcpyDeviceToHost, st));
      HB_CUDA(cudaMemcpyAsync(&col_chunks, H->scanC + nA - 1, 8, cudaMemcpyDeviceToHost, st));
      HB_CUDA(cudaMemsetAsync(S.counts + 2, 0, 4, st));
      HB_CUDA(cudaStreamSynchronize(st));
      if (cnt[2] > S.squeue_cap)
        return set_error(HBEM_ERR_CAPACITY, "singular queue overflow (%d touching pairs)", cnt[2]);
      const int nC = cnt[0];
      if (nC > 0) {
        rc = dispatch_op(ctx->op, ctx->helm, nt, ns, [&](auto OPc, auto Hc, auto NTc,
                                                         auto NSc) -> int {
          constexpr int OP = decltype(OPc)::value;
          constexpr bool HH = decltype(Hc)::value != 0;
          constexpr int NT = decltype(NTc)::value, NS = decltype(NSc)::value;
          k_jobs<V><<<(nC + 127) / 128, 128, 0, st>>>(S, S.listC, nC, 1, P.rperm, P.cperm);
          HB_CUDA(cudaGetLastError());
          k_int<T, C, OP, HH, NT, NS, true><<<(unsigned)col_chunks, kThreads, 0, st>>>(P, S);
          HB_CUDA(cudaGetLastError());
          if constexpr (NT == 1 && NS == 1) {
            k_int_singular<T, C, OP, HH><<<148 * 4, kThreads, 0, st>>>(P, S, 1);
            HB_CUDA(cudaGetLastError());
          }
          return HBEM_OK;
        });
        if (rc != HBEM_OK) return rc;
        k_fin_col<T, C><<<(nC + kWarps - 1) / kWarps, kThreads, 0, st>>>(S, nC);
        HB_CUDA(cudaGetLastError());
      }
      launches += (nt == 1 && ns == 1) ? 10 : 8;
      HB_CUDA(cudaEventRecord(H->ev[1], st));
      HB_CUDA(cudaMemcpyAsync(cnt, S.counts, 12, cudaMemcpyDeviceToHost, st));
      HB_CUDA(cudaStreamSynchronize(st));
      if (cnt[2] > S.squeue_cap)
        return set_error(HBEM_ERR_CAPACITY, "singular queue overflow (%d touching pairs)", cnt[2]);
      float ms = 0.f;
      HB_CUDA(cudaEventElapsedTime(&ms, H->ev[0], H->ev[1]));
      ST.aca_kernel_ms += ms;
      ST.row_jobs += nA;
      ST.col_jobs += nC;
      nA = cnt[1];
      std::swap(la, la2);
      std::swap(na_, na2);
      ++waves;
    }
  }
  const auto t_aca = clk::now();
  // ---- classify admissible blocks (lowrank_leaf, hmatrix.py:721-735) -------------
  std::vector<int> st_h(na), rk_h(na), ex_h(na);
  std::vector<double> rs_h(na);
  if (na > 0) {
    HB_CUDA(cudaMemcpy(st_h.data(), S.status, na * 4, cudaMemcpyDeviceToHost));
    HB_CUDA(cudaMemcpy(rk_h.data(), S.rank, na * 4, cudaMemcpyDeviceToHost));
    HB_CUDA(cudaMemcpy(ex_h.data(), S.exhausted, na * 4, cudaMemcpyDeviceToHost));
    HB_CUDA(cudaMemcpy(rs_h.data(), S.resid, na * 8, cudaMemcpyDeviceToHost));
  }
  H->lowrank_slots.clear();
  H->lr_uoff.clear();
  H->lr_voff.clear();
  H->u_entries = H->v_entries = 0;
  std::vector<int> expand_slots, fb_r0, fb_c0, fb_h, fb_w;
  std::vector<long long> expand_off, fb_off;
  long long adm_dense = 0;
  for (int q = 0; q < na; ++q) {
    const int lf = H->adm_leaf[q];
    const int s = st_h[q];
    const int h = H->ah[q], w = H->aw[q];
    if (s == ST_OVERFLOW)
      return set_error(HBEM_ERR_CAPACITY,
                       "ACA rank capacity %d exceeded for block rows [%d, %d) x cols [%d, %d); "
                       "raise rank_capacity",
                       S.tmax, H->ar0[q], H->ar0[q] + h, H->ac0[q], H->ac0[q] + w);
    if (s == ST_POOL)
      return set_error(HBEM_ERR_CAPACITY, "ACA factor pool of %lld values exhausted",
                       (long long)S.pool_cap);
    H->rank[lf] = rk_h[q];
    H->resid[lf] = rs_h[q];
    H->flags[lf] = (s == ST_CONVERGED ? 1 : 0) | (ex_h[q] ? 2 : 0);
    H->kind[lf] = 0;
    H->off_u[lf] = H->off_v[lf] = -1;
    const long long hw = (long long)h * w;
    if (ex_h[q]) ST.aca_exhausted++;
    if (s == ST_CONVERGED) {
      ST.aca_converged++;
      if ((long long)rk_h[q] * (h + w) < hw) {
        H->kind[lf] = 1;
        H->lowrank_slots.push_back(q);
        H->off_u[lf] = H->u_entries;
        H->off_v[lf] = H->v_entries;
        H->lr_uoff.push_back(H->u_entries);
        H->lr_voff.push_back(H->v_entries);
        H->u_entries += (long long)h * rk_h[q];
        H->v_entries += (long long)w * rk_h[q];
        ST.lowrank_leaves++;
        continue;
      }
      expand_slots.push_back(q);
      expand_off.push_back(adm_dense);
    } else {  // ST_FALLBACK: rank cap without convergence -> exact rows
      ST.aca_fallback_dense++;
      fb_r0.push_back(H->ar0[q]); fb_c0.push_back(H->ac0[q]);
      fb_h.push_back(h); fb_w.push_back(w);
      fb_off.push_back(adm_dense);
    }
    H->off_dense[lf] = H->nf_entries + adm_dense;
    adm_dense += hw;
  }
  ST.dense_leaves = H->nd + (int64_t)expand_slots.size() + (int64_t)fb_r0.size();
  H->dense_entries = H->nf_entries + adm_dense;
  const size_t vb = sizeof(V);
  if ((size_t)adm_dense * vb > H->dense_adm_cap) {
    cudaFree(H->dense_adm);
    H->dense_adm = nullptr;
    H->dense_adm_cap = (size_t)adm_dense * vb;
    HB_CUDA(cudaMalloc(&H->dense_adm, std::max(H->dense_adm_cap, vb)));
  }
  if (!expand_slots.empty()) {
    int *slots;
    long long *offs;
    HB_CHECK(upload(H, &slots, expand_slots));
    HB_CHECK(upload(H, &offs, expand_off));
    k_expand<T, C><<<(unsigned)expand_slots.size(), 128, 0, st>>>(
        slots, (int)expand_slots.size(), S, offs, H->dense_adm);
    HB_CUDA(cudaGetLastError());
    ++launches;
  }
  unsigned long long fb_sing = 0;
  if (!fb_r0.empty()) {
    // exact rows of non-converged blocks: the dense-leaf kernels on a
    // temporary tile list
    DenseDev F{};
    std::vector<int> tslot, tstart;
    long long ent = 0;
    for (size_t s = 0; s < fb_r0.size(); ++s) {
      const long long hw = (long long)fb_h[s] * fb_w[s];
      for (long long t = 0; t < hw; t += kThreads) {
        tslot.push_back((int)s);
        tstart.push_back((int)t);
      }
      ent += hw;
    }
    int *p;
    long long *pl;
    HB_CHECK(upload(H, &p, tslot)); F.tile_slot = p;
    HB_CHECK(upload(H, &p, tstart)); F.tile_start = p;
    HB_CHECK(upload(H, &p, fb_r0)); F.r0 = p;
    HB_CHECK(upload(H, &p, fb_c0)); F.c0 = p;
    HB_CHECK(upload(H, &p, fb_h)); F.h = p;
    HB_CHECK(upload(H, &p, fb_w)); F.w = p;
    HB_CHECK(upload(H, &pl, fb_off)); F.off = pl;
    F.out = H->dense_adm;
    HB_CHECK(dalloc(H, &F.sing_count, 1));
    HB_CHECK(dalloc(H, &F.stat, 2));
    HB_CUDA(cudaMemsetAsync(F.sing_count, 0, 8, st));
    HB_CUDA(cudaMemsetAsync(F.stat, 0, 16, st));
    if (nt == 1 && ns == 1) {
      HB_CHECK(dalloc(H, &F.sing_slot, ent));
      HB_CHECK(dalloc(H, &F.sing_pos, ent));
    }
    const unsigned ntl = (unsigned)tslot.size();
    int rc = dispatch_op(ctx->op, ctx->helm, nt, ns, [&](auto OPc, auto Hc, auto NTc,
                                                         auto NSc) -> int {
      constexpr int OP = decltype(OPc)::value;
      constexpr bool HH = decltype(Hc)::value != 0;
      constexpr int NT = decltype(NTc)::value, NS = decltype(NSc)::value;
      k_dense<T, C, OP, HH, NT, NS><<<ntl, kThreads, 0, st>>>(P, F);
      HB_CUDA(cudaGetLastError());
      if constexpr (NT == 1 && NS == 1) {
        k_dense_singular<T, C, OP, HH><<<148 * 16, kThreads, 0, st>>>(P, F);
        HB_CUDA(cudaGetLastError());
      }
      return HBEM_OK;
    });
    if (rc != HBEM_OK) return rc;
    launches += (nt == 1 && ns == 1) ? 2 : 1;
    unsigned long long fs[2] = {0, 0};
    HB_CUDA(cudaMemcpyAsync(&fb_sing, F.sing_count, 8, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaMemcpyAsync(fs, F.stat, 16, cudaMemcpyDeviceToHost, st));
    HB_CUDA(cudaStreamSynchronize(st));
    fb_sing += fs[1];
    ST.regular_pairs += ent;
  }
  HB_CUDA(cudaStreamWaitEvent(st, H->side_done, 0));
  unsigned long long nf_sing = 0, nf_stat[2] = {0, 0}, aca_stat[2] = {0, 0};
  HB_CUDA(cudaMemcpyAsync(&nf_sing, H->D.sing_count, 8, cudaMemcpyDeviceToHost, st));
  HB_CUDA(cudaMemcpyAsync(nf_stat, H->D.stat, 16, cudaMemcpyDeviceToHost, st));
  HB_CUDA(cudaMemcpyAsync(aca_stat, S.stat, 16, cudaMemcpyDeviceToHost, st));
  HB_CUDA(cudaStreamSynchronize(st));
  const auto t_end = clk::now();
  {
    float ms = 0.f;
    HB_CUDA(cudaEventElapsedTime(&ms, H->ev[2], H->ev[3]));
    ST.nearfield_kernel_ms = ms;
  }
  ST.aca_entries = (int64_t)aca_stat[0];
  // pair accounting: ACA jobs |T(dof)| |col_elems| (P0: the job
  // width), near-field |rows| |cols|; singular pairs counted separately
  const int64_t sing = (int64_t)(nf_sing + nf_stat[1] + aca_stat[1] + fb_sing);
  ST.singular_pairs = sing;
  ST.regular_pairs += (int64_t)aca_stat[0] + H->nf_entries - sing;
  ST.waves = waves;
  ST.u_entries = H->u_entries;
  ST.v_entries = H->v_entries;
  ST.dense_entries = H->dense_entries;
  ST.seconds = secs(t0, t_end);
  ST.seconds_setup = H->setup_s;
  ST.seconds_aca = secs(t0, t_aca);
  ST.seconds_finalize = secs(t_aca, t_end);
  ST.launches = launches;
  return HBEM_OK;
}

int execute(hbem_hmat *H, cudaStream_t st) {
  hbem_ctx *ctx = H->ctx;
  if (ctx->precision == HBEM_DOUBLE)
    return ctx->helm ? execute_t<double, true>(H, st) : execute_t<double, false>(H, st);
  return ctx->helm ? execute_t<float, true>(H, st) : execute_t<float, false>(H, st);
}

}  // namespace

// ---------------------------------------------------------------------------
// FP64 / FP32 FMA throughput probes (roofline denominators measured live)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_fma_probe(T *out, int iters, T a) {
  T x0 = (T)threadIdx.x, x1 = x0 + T(1), x2 = x0 + T(2), x3 = x0 + T(3);
  T x4 = x0 + T(4), x5 = x0 + T(5), x6 = x0 + T(6), x7 = x0 + T(7);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = x0 * a + a; x1 = x1 * a + a; x2 = x2 * a + a; x3 = x3 * a + a;
      x4 = x4 * a + a; x5 = x5 * a + a; x6 = x6 * a + a; x7 = x7 * a + a;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

extern "C" {

int hbem_hmat_assemble(hbem_ctx *ctx, const hbem_hmat_desc *d, void *stream, hbem_hmat **out) {
  clear_error();
  if (!ctx || !d || !out) return set_error(HBEM_ERR_ARG, "null argument");
  *out = nullptr;
  if (d->pointers_on_device)
    return set_error(HBEM_ERR_ARG, "device-resident partition descriptors not supported yet");
  if (d->epsilon <= 0.0) return set_error(HBEM_ERR_CONFIG, "epsilon must be > 0, got %g", d->epsilon);
  HB_CUDA(cudaSetDevice(ctx->device));
  hbem_hmat *H = new hbem_hmat();
  H->ctx = ctx;
  H->device = ctx->device;
  H->complex_ = ctx->helm;
  H->vbytes = (size_t)ctx->real_bytes() * (ctx->helm ? 2 : 1);
  const auto t0 = clk::now();
  int rc = setup(H, d);
  H->setup_s = secs(t0, clk::now());
  if (rc == HBEM_OK) rc = execute(H, (cudaStream_t)stream);
  if (rc != HBEM_OK) {
    delete H;
    return rc;
  }
  *out = H;
  return HBEM_OK;
}

int hbem_hmat_execute(hbem_hmat *h, void *stream) {
  clear_error();
  if (!h) return set_error(HBEM_ERR_ARG, "null hmat");
  HB_CUDA(cudaSetDevice(h->device));
  return execute(h, (cudaStream_t)stream);
}

int hbem_hmat_stats_get(const hbem_hmat *h, hbem_hmat_stats *s) {
  if (!h || !s) return set_error(HBEM_ERR_ARG, "null argument");
  *s = h->stats;
  return HBEM_OK;
}

int hbem_hmat_leaf_meta(const hbem_hmat *h, int32_t *kind, int32_t *rank, int32_t *flags,
                        int64_t *off_u, int64_t *off_v, int64_t *off_dense) {
  if (!h) return set_error(HBEM_ERR_ARG, "null hmat");
  if (kind) std::copy(h->kind.begin(), h->kind.end(), kind);
  if (rank) std::copy(h->rank.begin(), h->rank.end(), rank);
  if (flags) std::copy(h->flags.begin(), h->flags.end(), flags);
  if (off_u) std::copy(h->off_u.begin(), h->off_u.end(), off_u);
  if (off_v) std::copy(h->off_v.begin(), h->off_v.end(), off_v);
  if (off_dense) std::copy(h->off_dense.begin(), h->off_dense.end(), off_dense);
  return HBEM_OK;
}

int hbem_hmat_copy_arenas(const hbem_hmat *hc, void *u, void *v, void *dense) {
  clear_error();
  hbem_hmat *h = const_cast<hbem_hmat *>(hc);
  if (!h) return set_error(HBEM_ERR_ARG, "null hmat");
  HB_CUDA(cudaSetDevice(h->device));
  const size_t vb = h->vbytes;
  if (dense) {
    if (h->nf_entries > 0)
      HB_CUDA(cudaMemcpy(dense, h->dense_nf, (size_t)h->nf_entries * vb, cudaMemcpyDeviceToHost));
    const long long adm = h->dense_entries - h->nf_entries;
    if (adm > 0)
      HB_CUDA(cudaMemcpy((char *)dense + (size_t)h->nf_entries * vb, h->dense_adm, (size_t)adm * vb,
                         cudaMemcpyDeviceToHost));
  }
  if ((u || v) && !h->lowrank_slots.empty()) {
    // gather the factor records of the low-rank blocks in chunks
    const size_t n = h->lowrank_slots.size();
    const long long chunk_vals = 64ll << 20;
    void *su = nullptr, *sv = nullptr;
    HB_CUDA(cudaMalloc(&su, chunk_vals * vb));
    HB_CUDA(cudaMalloc(&sv, chunk_vals * vb));
    int *d_slots = nullptr;
    long long *d_uo = nullptr, *d_vo = nullptr;
    HB_CUDA(cudaMalloc(&d_slots, n * 4));
    HB_CUDA(cudaMalloc(&d_uo, n * 8));
    HB_CUDA(cudaMalloc(&d_vo, n * 8));
    HB_CUDA(cudaMemcpy(d_slots, h->lowrank_slots.data(), n * 4, cudaMemcpyHostToDevice));
    HB_CUDA(cudaMemcpy(d_uo, h->lr_uoff.data(), n * 8, cudaMemcpyHostToDevice));
    HB_CUDA(cudaMemcpy(d_vo, h->lr_voff.data(), n * 8, cudaMemcpyHostToDevice));
    size_t q0 = 0;
    while (q0 < n) {
      const long long ub = h->lr_uoff[q0], vbase = h->lr_voff[q0];
      size_t q1 = q0 + 1;
      while (q1 < n && h->lr_uoff[q1] - ub < chunk_vals && h->lr_voff[q1] - vbase < chunk_vals &&
             (q1 + 1 < n ? h->lr_uoff[q1 + 1] : h->u_entries) - ub <= chunk_vals &&
             (q1 + 1 < n ? h->lr_voff[q1 + 1] : h->v_entries) - vbase <= chunk_vals)
        ++q1;
      const long long ue = q1 < n ? h->lr_uoff[q1] : h->u_entries;
      const long long ve = q1 < n ? h->lr_voff[q1] : h->v_entries;
      if (ue - ub > chunk_vals || ve - vbase > chunk_vals) {
        cudaFree(su); cudaFree(sv);
        HB_CUDA(cudaMalloc(&su, (ue - ub) * vb));
        HB_CUDA(cudaMalloc(&sv, (ve - vbase) * vb));
      }
      const int cnt = (int)(q1 - q0);
      if (h->vbytes == 16)
        k_pack_factors<Cx<double>><<<cnt, 128>>>(d_slots + q0, cnt, h->S, d_uo + q0, d_vo + q0,
                                                 ub, vbase, (Cx<double> *)su, (Cx<double> *)sv);
      else if (h->vbytes == 8 && h->complex_)
        k_pack_factors<Cx<float>><<<cnt, 128>>>(d_slots + q0, cnt, h->S, d_uo + q0, d_vo + q0, ub,
                                                vbase, (Cx<float> *)su, (Cx<float> *)sv);
      else if (h->vbytes == 8)
        k_pack_factors<double><<<cnt, 128>>>(d_slots + q0, cnt, h->S, d_uo + q0, d_vo + q0, ub,
                                             vbase, (double *)su, (double *)sv);
      else
        k_pack_factors<float><<<cnt, 128>>>(d_slots + q0, cnt, h->S, d_uo + q0, d_vo + q0, ub,
                                            vbase, (float *)su, (float *)sv);
      HB_CUDA(cudaGetLastError());
      if (u)
        HB_CUDA(cudaMemcpy((char *)u + ub * vb, su, (ue - ub) * vb, cudaMemcpyDeviceToHost));
      if (v)
        HB_CUDA(cudaMemcpy((char *)v + vbase * vb, sv, (ve - vbase) * vb, cudaMemcpyDeviceToHost));
      q0 = q1;
    }
    cudaFree(su);
    cudaFree(sv);
    cudaFree(d_slots);
    cudaFree(d_uo);
    cudaFree(d_vo);
  }
  return HBEM_OK;
}

int hbem_hmat_matvec(const hbem_hmat *, const void *, void *) {
  return set_error(HBEM_ERR_CONFIG, "device matvec not available in this build");
}

int hbem_hmat_destroy(hbem_hmat *h) {
  delete h;
  return HBEM_OK;
}

int hbem_host_alloc(int64_t bytes, void **out) {
  clear_error();
  if (!out) return set_error(HBEM_ERR_ARG, "null argument");
  *out = nullptr;
  HB_CUDA(cudaHostAlloc(out, (size_t)std::max<int64_t>(bytes, 1), cudaHostAllocDefault));
  return HBEM_OK;
}

int hbem_host_free(void *p) {
  if (p) cudaFreeHost(p);
  return HBEM_OK;
}

int hbem_probe_fma(int32_t device, int32_t precision, double *flops_per_s) {
  clear_error();
  if (!flops_per_s) return set_error(HBEM_ERR_ARG, "null argument");
  HB_CUDA(cudaSetDevice(device));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int threads = 256, blocks = sms * 8, iters = 4096;
  void *out = nullptr;
  HB_CUDA(cudaMalloc(&out, (size_t)blocks * threads * 8));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    if (precision == HBEM_DOUBLE)
      k_fma_probe<double><<<blocks, threads>>>((double *)out, iters, 0.999999);
    else
      k_fma_probe<float><<<blocks, threads>>>((float *)out, iters, 0.999999f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (rep > 0) best = std::min(best, ms);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  HB_CUDA(cudaGetLastError());
  const double fmas = (double)blocks * threads * iters * 16.0 * 8.0;
  *flops_per_s = 2.0 * fmas / (best * 1e-3);
  return HBEM_OK;
}

}  // extern "C"
