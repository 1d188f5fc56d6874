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

struct AcaDev {
  const int *h, *w, *r0, *c0;
  int *rank, *cur, *pcol, *small, *status, *exhausted;
  double *norm2, *resid, *rn2, *piv;  // piv: 2 doubles (re, im)
  long long *pend, *terms;
  int tmax;
  unsigned *rmask, *cmask;
  const long long *rmask_off, *cmask_off;
  void *pool;
  long long pool_cap;
  unsigned long long *pool_top;
  int kmax_cfg;
  double eps;
  const int *listA;
  int *listB, *listA2, *counts;  // counts[0] = |B|, counts[1] = |A2|
  unsigned long long *stat;      // [0] entries, [1] singular pairs
};

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kTmaxSmem = 96;

__device__ __forceinline__ bool better(double a, int ia, double b, int ib) {
  return a > b || (a == b && ia < ib);
}

// block-wide argmax (first index on ties) and sum; result valid in thread 0
__device__ __forceinline__ void block_reduce(double &best, int &bidx, double &sum, double *s_v,
                                             int *s_i, double *s_s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (better(ob, oi, best, bidx)) { best = ob; bidx = oi; }
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { s_v[warp] = best; s_i[warp] = bidx; s_s[warp] = sum; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < kWarps; ++k) {
      if (better(s_v[k], s_i[k], best, bidx)) { best = s_v[k]; bidx = s_i[k]; }
      sum += s_s[k];
    }
  }
}

__device__ __forceinline__ bool bit(const unsigned *m, int i) { return (m[i >> 5] >> (i & 31)) & 1u; }
__device__ __forceinline__ void set_bit(unsigned *m, int i) { atomicOr(m + (i >> 5), 1u << (i & 31)); }

// lowest row without its bit set (padding bits are preset), or -1
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

// ---------------------------------------------------------------------------
// K3a: ACA row phase.  One CTA per active block.
// ---------------------------------------------------------------------------
template <typename T, bool C, int OP, bool HELM, int NT, int NS>
__global__ void __launch_bounds__(kThreads) k_aca_row(Prob<T> P, AcaDev S) {
  using N = Num<T, C>;
  using V = typename N::V;
  __shared__ V s_u[kTmaxSmem];
  __shared__ long long s_term[kTmaxSmem];
  __shared__ double s_v[kWarps], s_s[kWarps];
  __shared__ int s_i[kWarps];
  __shared__ int s_stop;
  __shared__ long long s_pend;
  const int b = S.listA[blockIdx.x];
  const int h = S.h[b], w = S.w[b];
  const int k = S.rank[b];
  const int i = S.cur[b];
  V *pool = static_cast<V *>(S.pool);
  if (threadIdx.x == 0) {
    int stop = 0;
    const int kmax_b = min(S.kmax_cfg, min(h, w));
    if (k >= kmax_b) {                   // rank cap without convergence
      S.status[b] = ST_FALLBACK;
      stop = 1;
    } else if (k >= S.tmax) {            // term table exhausted: retry bigger
      S.status[b] = ST_OVERFLOW;
      stop = 1;
    } else if (i < 0) {                  // rows exhausted (hmatrix.py:319-322)
      S.status[b] = ST_CONVERGED;
      S.exhausted[b] = 1;
      stop = 1;
    } else {
      long long pe = S.pend[b];
      if (pe < 0) {
        const unsigned long long o = atomicAdd(S.pool_top, (unsigned long long)(h + w));
        if ((long long)o + h + w > S.pool_cap) {
          S.status[b] = ST_POOL;
          stop = 1;
        } else {
          pe = (long long)o;
          S.pend[b] = pe;
        }
      }
      s_pend = pe;
      atomicAdd(S.stat, (unsigned long long)w);
    }
    s_stop = stop;
  }
  if (i >= 0)
    for (int l = threadIdx.x; l < k && l < S.tmax; l += kThreads) {
      const long long t = S.terms[(long long)b * S.tmax + l];
      s_term[l] = t;
      s_u[l] = pool[t + i];
    }
  __syncthreads();
  if (s_stop) return;
  const long long pe = s_pend;
  V *row = pool + pe + h;
  const unsigned *cm = S.cmask + S.cmask_off[b];
  const int r0 = S.r0[b], c0 = S.c0[b];
  const int di = P.rperm[r0 + i];
  double best = -1.0, ss = 0.0;
  int bidx = 0x7fffffff;

  if constexpr (NT == 1 && NS == 1) {
    // P0: the test element is fixed for the whole row
    T x[18], na[4];
    load_q<T>(P.g.q, di, x);
    load_nj<T>(P.g.nj, di, na);
    const int4 ea = P.elem[di];
    for (int c = threadIdx.x; c < w; c += kThreads) {
      const int f = P.cperm[c0 + c];
      V val;
      if (touching(ea, P.elem[f])) {
        val = entry<T, C, OP, HELM, 1, 1>(P, di, f, S.stat + 1);
      } else {
        T y[18], nb[4], re[1][1], im[1][1];
        load_q<T>(P.g.q, f, y);
        load_nj<T>(P.g.nj, f, nb);
        regular_pair<T, OP, HELM, 1, 1>(P.R, x, y, na, nb, nullptr, nullptr, re, im);
        val = N::mk(re[0][0], im[0][0]);
      }
      for (int l = 0; l < k; ++l) val = N::fms(val, s_u[l], pool[s_term[l] + h + c]);
      row[c] = val;
      const double a = N::abs(val);
      ss += N::nrm(val);
      if (!bit(cm, c) && a > best) { best = a; bidx = c; }
    }
  } else {
    for (int c = threadIdx.x; c < w; c += kThreads) {
      const int dj = P.cperm[c0 + c];
      V val = entry<T, C, OP, HELM, NT, NS>(P, di, dj, S.stat + 1);
      for (int l = 0; l < k; ++l) val = N::fms(val, s_u[l], pool[s_term[l] + h + c]);
      row[c] = val;
      const double a = N::abs(val);
      ss += N::nrm(val);
      if (!bit(cm, c) && a > best) { best = a; bidx = c; }
    }
  }
  block_reduce(best, bidx, ss, s_v, s_i, s_s);
  if (threadIdx.x == 0) {
    if (best <= 0.0) {
      // residual row vanished: retire it to Z, restart from the lowest
      // unused row (hmatrix.py:334-338); no column job this wave
      unsigned *rm = S.rmask + S.rmask_off[b];
      set_bit(rm, i);
      __threadfence_block();
      S.cur[b] = first_clear(rm, h);
      S.listA2[atomicAdd(S.counts + 1, 1)] = b;
    } else {
      const V pv = row[bidx];
      S.pcol[b] = bidx;
      if constexpr (C) {
        S.piv[2 * b] = pv.re;
        S.piv[2 * b + 1] = pv.im;
      } else {
        S.piv[2 * b] = pv;
        S.piv[2 * b + 1] = 0.0;
      }
      S.rn2[b] = ss;
      S.listB[atomicAdd(S.counts, 1)] = b;
    }
  }
}

// ---------------------------------------------------------------------------
// K3b: ACA column phase + stopping test + Frobenius update + next pivot.
// ---------------------------------------------------------------------------
template <typename T, bool C, int OP, bool HELM, int NT, int NS>
__global__ void __launch_bounds__(kThreads) k_aca_col(Prob<T> P, AcaDev S) {
  using N = Num<T, C>;
  using V = typename N::V;
  __shared__ V s_v[kTmaxSmem];
  __shared__ long long s_term[kTmaxSmem];
  __shared__ double s_bv[kWarps], s_ss[kWarps];
  __shared__ int s_bi[kWarps];
  __shared__ double s_dot[kTmaxSmem][kWarps][4];
  __shared__ int s_accept;
  if ((int)blockIdx.x >= S.counts[0]) return;
  const int b = S.listB[blockIdx.x];
  const int h = S.h[b], w = S.w[b];
  const int k = S.rank[b];
  const int i = S.cur[b];
  const int j = S.pcol[b];
  const long long pe = S.pend[b];
  V *pool = static_cast<V *>(S.pool);
  for (int l = threadIdx.x; l < k; l += kThreads) {
    const long long t = S.terms[(long long)b * S.tmax + l];
    s_term[l] = t;
    s_v[l] = pool[t + h + j];
  }
  if (threadIdx.x == 0) atomicAdd(S.stat, (unsigned long long)h);
  __syncthreads();
  V *col = pool + pe;
  unsigned *rm = S.rmask + S.rmask_off[b];
  const int r0 = S.r0[b], c0 = S.c0[b];
  const int dj = P.cperm[c0 + j];
  double best = -1.0, ss = 0.0;
  int bidx = 0x7fffffff;
  if constexpr (NT == 1 && NS == 1) {
    T y[18], nb[4];
    load_q<T>(P.g.q, dj, y);
    load_nj<T>(P.g.nj, dj, nb);
    const int4 eb = P.elem[dj];
    for (int r = threadIdx.x; r < h; r += kThreads) {
      const int e = P.rperm[r0 + r];
      V val;
      if (touching(P.elem[e], eb)) {
        val = entry<T, C, OP, HELM, 1, 1>(P, e, dj, S.stat + 1);
      } else {
        T x[18], na[4], re[1][1], im[1][1];
        load_q<T>(P.g.q, e, x);
        load_nj<T>(P.g.nj, e, na);
        regular_pair<T, OP, HELM, 1, 1>(P.R, x, y, na, nb, nullptr, nullptr, re, im);
        val = N::mk(re[0][0], im[0][0]);
      }
      for (int l = 0; l < k; ++l) val = N::fms(val, s_v[l], pool[s_term[l] + r]);
      col[r] = val;
      const double a = N::abs(val);
      ss += N::nrm(val);
      if (r != i && !bit(rm, r) && a > best) { best = a; bidx = r; }
    }
  } else {
    for (int r = threadIdx.x; r < h; r += kThreads) {
      const int di = P.rperm[r0 + r];
      V val = entry<T, C, OP, HELM, NT, NS>(P, di, dj, S.stat + 1);
      for (int l = 0; l < k; ++l) val = N::fms(val, s_v[l], pool[s_term[l] + r]);
      col[r] = val;
      const double a = N::abs(val);
      ss += N::nrm(val);
      if (r != i && !bit(rm, r) && a > best) { best = a; bidx = r; }
    }
  }
  block_reduce(best, bidx, ss, s_bv, s_bi, s_ss);
  const int next = best >= 0.0 ? bidx : -1;
  if (threadIdx.x == 0) {
    const double nu = sqrt(ss);
    const double pr = S.piv[2 * b], pim = S.piv[2 * b + 1];
    const double nv = sqrt(S.rn2[b]) / hypot(pr, pim);
    const double upd = nu * nv;
    const double n2 = S.norm2[b];
    int accept = 1;
    if (n2 > 0.0 && upd <= S.eps * sqrt(n2)) {
      // negligible update: dropped; two in a row stop (hmatrix.py:347-357)
      accept = 0;
      S.resid[b] = upd / sqrt(n2);
      const int sm = S.small[b] + 1;
      S.small[b] = sm;
      if (sm >= 2) {
        S.status[b] = ST_CONVERGED;
      } else {
        set_bit(rm, i);
        S.cur[b] = next;
        S.listA2[atomicAdd(S.counts + 1, 1)] = b;
      }
    }
    s_accept = accept;
    S.rn2[b] = upd;  // stash the update size for the accept path
  }
  __syncthreads();
  if (!s_accept) return;
  // cross terms sum_l Re(vdot(u_l, u) * vdot(v_l, v)) (hmatrix.py:359-361)
  const V *row = pool + pe + h;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int l = 0; l < k; ++l) {
    double ur = 0, ui = 0, vr = 0, vi = 0;
    const V *ul = pool + s_term[l];
    const V *vl = ul + h;
    for (int r = threadIdx.x; r < h; r += kThreads) N::cdot(ur, ui, ul[r], col[r]);
    for (int c = threadIdx.x; c < w; c += kThreads) N::cdot(vr, vi, vl[c], row[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ur += __shfl_xor_sync(0xffffffffu, ur, o);
      ui += __shfl_xor_sync(0xffffffffu, ui, o);
      vr += __shfl_xor_sync(0xffffffffu, vr, o);
      vi += __shfl_xor_sync(0xffffffffu, vi, o);
    }
    if (lane == 0) {
      s_dot[l][warp][0] = ur;
      s_dot[l][warp][1] = ui;
      s_dot[l][warp][2] = vr;
      s_dot[l][warp][3] = vi;
    }
  }
  __syncthreads();
  const double pr = S.piv[2 * b], pim = S.piv[2 * b + 1];
  if (threadIdx.x == 0) {
    double cross = 0.0;
    const double pd = pr * pr + pim * pim;
    for (int l = 0; l < k; ++l) {
      double ur = 0, ui = 0, vr = 0, vi = 0;
      for (int q = 0; q < kWarps; ++q) {
        ur += s_dot[l][q][0];
        ui += s_dot[l][q][1];
        vr += s_dot[l][q][2];
        vi += s_dot[l][q][3];
      }
      // vdot(v_l, v) = (sum conj(v_l) row) / pivot
      const double dr = (vr * pr + vi * pim) / pd, di = (vi * pr - vr * pim) / pd;
      cross += ur * dr - ui * di;
    }
    const double upd = S.rn2[b];
    double n2 = S.norm2[b] + 2.0 * cross + upd * upd;
    S.norm2[b] = n2;
    S.small[b] = 0;
    S.terms[(long long)b * S.tmax + k] = pe;
    S.pend[b] = -1;
    S.rank[b] = k + 1;
    set_bit(rm, i);
    set_bit(S.cmask + S.cmask_off[b], j);
    if (n2 > 0.0) {
      S.resid[b] = upd / sqrt(n2);
      if (upd <= S.eps * sqrt(n2)) S.small[b] = 1;
    }
    S.cur[b] = next;
    S.listA2[atomicAdd(S.counts + 1, 1)] = b;
  }
  // v = row / pivot, in place (hmatrix.py:339)
  V pv;
  if constexpr (C) pv = V{(T)pr, (T)pim};
  else pv = (T)pr;
  V *rw = pool + pe + h;
  for (int c = threadIdx.x; c < w; c += kThreads) rw[c] = N::div(rw[c], pv);
}

__global__ void k_aca_init(AcaDev S, int n) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n) return;
  S.rank[b] = 0;
  S.cur[b] = 0;
  S.small[b] = 0;
  S.status[b] = ST_ACTIVE;
  S.exhausted[b] = 0;
  S.norm2[b] = 0.0;
  S.resid[b] = INFINITY;
  S.pend[b] = -1;
  // row mask padding bits preset (blocked), everything else clear
  const int h = S.h[b], w = S.w[b];
  unsigned *rm = S.rmask + S.rmask_off[b];
  for (int k = 0; k < (h + 31) / 32; ++k) {
    const int lo = k * 32;
    const int valid = min(32, h - lo);
    rm[k] = valid == 32 ? 0u : ~((1u << valid) - 1u);
  }
  unsigned *cm = S.cmask + S.cmask_off[b];
  for (int k = 0; k < (w + 31) / 32; ++k) cm[k] = 0u;
}

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
// host side
// ---------------------------------------------------------------------------
struct hbem_hmat {
  hbem_ctx *ctx = nullptr;
  int device = 0;
  int64_t n_leaves = 0;
  bool complex_ = false;
  size_t vbytes = 8;  // bytes per value
  // per leaf (host)
  std::vector<int32_t> kind, rank, flags;
  std::vector<int64_t> off_u, off_v, off_dense;
  std::vector<double> resid;
  // device
  void *pool = nullptr;
  void *dense = nullptr;
  long long dense_entries = 0, u_entries = 0, v_entries = 0;
  // ACA block arrays needed for packing (device)
  std::vector<void *> dev_allocs;
  AcaDev S{};
  std::vector<int> lowrank_slots;   // adm slot per low-rank leaf
  std::vector<int64_t> lr_uoff, lr_voff;
  hbem_hmat_stats stats{};
  ~hbem_hmat() {
    cudaSetDevice(device);
    for (void *p : dev_allocs) cudaFree(p);
    cudaFree(pool);
    cudaFree(dense);
  }
};

namespace {

template <typename X> int dalloc(hbem_hmat *H, X **p, size_t n) {
  void *q = nullptr;
  cudaError_t e = cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(X));
  if (e != cudaSuccess)
    return set_error(HBEM_ERR_CAPACITY, "device allocation of %zu bytes failed: %s",
                     n * sizeof(X), cudaGetErrorString(e));
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

template <typename T, bool C>
int assemble_t(hbem_ctx *ctx, const hbem_hmat_desc *d, cudaStream_t st, hbem_hmat *H) {
  using V = typename Num<T, C>::V;
  const auto t_start = std::chrono::steady_clock::now();
  const int64_t m = ctx->m;
  const int nt = ctx->nt, ns = ctx->ns;
  // ---- partition / DOF maps on device ------------------------------------
  std::vector<int> rperm(d->n_rows), cperm(d->n_cols);
  for (int64_t i = 0; i < d->n_rows; ++i) rperm[i] = (int)d->row_perm[i];
  for (int64_t i = 0; i < d->n_cols; ++i) cperm[i] = (int)d->col_perm[i];
  Prob<T> P{};
  P.g = ctx->geo<T>();
  P.R = ctx->rule<T>();
  P.G64 = ctx->geo64();
  P.elem = ctx->elem;
  int *d_rperm, *d_cperm;
  HB_CHECK(upload(H, &d_rperm, rperm));
  HB_CHECK(upload(H, &d_cperm, cperm));
  P.rperm = d_rperm;
  P.cperm = d_cperm;
  if (nt == 3) {
    Incidence I = incidence(d->test_dofmap, m, 3, d->n_rows);
    int *p, *e;
    signed char *l;
    HB_CHECK(upload(H, &p, I.ptr));
    HB_CHECK(upload(H, &e, I.el));
    HB_CHECK(upload(H, &l, I.loc));
    P.tptr = p; P.tel = e; P.tloc = l;
  }
  if (ns == 3) {
    Incidence I = incidence(d->trial_dofmap, m, 3, d->n_cols);
    int *p, *e;
    signed char *l;
    HB_CHECK(upload(H, &p, I.ptr));
    HB_CHECK(upload(H, &e, I.el));
    HB_CHECK(upload(H, &l, I.loc));
    P.sptr = p; P.sel = e; P.sloc = l;
  }
  // ---- split leaves ----------------------------------------------------------
  const int64_t L = d->n_leaves;
  H->n_leaves = L;
  H->kind.assign(L, 0);
  H->rank.assign(L, 0);
  H->flags.assign(L, 0);
  H->off_u.assign(L, -1);
  H->off_v.assign(L, -1);
  H->off_dense.assign(L, -1);
  H->resid.assign(L, 0.0);
  std::vector<int> adm_leaf, den_leaf;
  for (int64_t q = 0; q < L; ++q) (d->leaves[3 * q + 2] ? adm_leaf : den_leaf).push_back((int)q);
  auto node_rng = [&](const int64_t *nodes, int64_t n) {
    return std::pair<int, int>((int)nodes[5 * n], (int)(nodes[5 * n + 1] - nodes[5 * n]));
  };
  const int na = (int)adm_leaf.size();
  std::vector<int> ah(na), aw(na), ar0(na), ac0(na);
  std::vector<long long> rmo(na), cmo(na);
  long long rmw = 0, cmw = 0, sum_hw = 0;
  for (int q = 0; q < na; ++q) {
    const int64_t lf = adm_leaf[q];
    auto [r0, h] = node_rng(d->row_nodes, d->leaves[3 * lf]);
    auto [c0, w] = node_rng(d->col_nodes, d->leaves[3 * lf + 1]);
    ar0[q] = r0; ah[q] = h; ac0[q] = c0; aw[q] = w;
    rmo[q] = rmw; rmw += (h + 31) / 32;
    cmo[q] = cmw; cmw += (w + 31) / 32;
    sum_hw += h + w;
  }
  const int kmax_cfg = d->k_max > 0 ? (int)std::min<int64_t>(d->k_max, 1 << 30) : (1 << 30);
  int tmax = d->rank_capacity > 0 ? d->rank_capacity : 64;
  tmax = std::min(tmax, kTmaxSmem);
  AcaDev &S = H->S;
  S.tmax = tmax;
  S.kmax_cfg = kmax_cfg;
  S.eps = d->epsilon;
  {
    int *p;
    HB_CHECK(upload(H, &p, ah)); S.h = p;
    HB_CHECK(upload(H, &p, aw)); S.w = p;
    HB_CHECK(upload(H, &p, ar0)); S.r0 = p;
    HB_CHECK(upload(H, &p, ac0)); S.c0 = p;
    long long *pl;
    HB_CHECK(upload(H, &pl, rmo)); S.rmask_off = pl;
    HB_CHECK(upload(H, &pl, cmo)); S.cmask_off = pl;
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
  HB_CHECK(dalloc(H, &S.terms, (size_t)na * tmax));
  HB_CHECK(dalloc(H, &S.rmask, rmw));
  HB_CHECK(dalloc(H, &S.cmask, cmw));
  int *listA, *listB, *listA2, *counts;
  HB_CHECK(dalloc(H, &listA, na));
  HB_CHECK(dalloc(H, &listB, na));
  HB_CHECK(dalloc(H, &listA2, na));
  HB_CHECK(dalloc(H, &counts, 4));
  S.counts = counts;
  S.listB = listB;
  unsigned long long *stat, *pool_top;
  HB_CHECK(dalloc(H, &stat, 4));
  HB_CHECK(dalloc(H, &pool_top, 1));
  HB_CUDA(cudaMemsetAsync(stat, 0, 32, st));
  HB_CUDA(cudaMemsetAsync(pool_top, 0, 8, st));
  S.stat = stat;
  S.pool_top = pool_top;
  // dense leaves: exact sizes known now
  const int nd = (int)den_leaf.size();
  std::vector<int> dr0, dc0, dh, dw;
  std::vector<long long> doff;
  long long dense_total = 0;
  for (int q = 0; q < nd; ++q) {
    const int64_t lf = den_leaf[q];
    auto [r0, h] = node_rng(d->row_nodes, d->leaves[3 * lf]);
    auto [c0, w] = node_rng(d->col_nodes, d->leaves[3 * lf + 1]);
    dr0.push_back(r0); dh.push_back(h); dc0.push_back(c0); dw.push_back(w);
    doff.push_back(dense_total);
    H->off_dense[lf] = dense_total;
    dense_total += (long long)h * w;
  }
  // pool: what is left of device memory after a margin for the dense arena
  size_t free_b = 0, total_b = 0;
  HB_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const size_t vb = sizeof(V);
  const size_t want = (size_t)sum_hw * (size_t)std::min(tmax, 24) * vb;
  const size_t reserve = (size_t)dense_total * vb * 2 + ((size_t)2 << 30);
  size_t cap_b = free_b > reserve ? free_b - reserve : 0;
  cap_b = std::min(cap_b, std::max(want, (size_t)1 << 20));
  cap_b = std::min(cap_b, (size_t)(free_b * 0.85));
  HB_CUDA(cudaMalloc(&H->pool, std::max<size_t>(cap_b, vb)));
  S.pool = H->pool;
  S.pool_cap = (long long)(cap_b / vb);

  const auto t_setup = std::chrono::steady_clock::now();
  // ---- ACA waves ---------------------------------------------------------------
  int waves = 0;
  if (na > 0) {
    k_aca_init<<<(na + 127) / 128, 128, 0, st>>>(S, na);
    HB_CUDA(cudaGetLastError());
    // large blocks first for load balance
    std::vector<int> order(na);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return (long long)ah[a] * aw[a] > (long long)ah[b] * aw[b];
    });
    HB_CUDA(cudaMemcpyAsync(listA, order.data(), na * sizeof(int), cudaMemcpyHostToDevice, st));
    int nA = na;
    int *la = listA, *la2 = listA2;
    int h_counts[2];
    while (nA > 0) {
      S.listA = la;
      S.listA2 = la2;
      HB_CUDA(cudaMemsetAsync(counts, 0, 16, st));
      int rc = dispatch_op(ctx->op, ctx->helm, nt, ns, [&](auto OPc, auto Hc, auto NTc, auto NSc) -> int {
        constexpr int OP = decltype(OPc)::value;
        constexpr bool HH = decltype(Hc)::value != 0;
        constexpr int NT = decltype(NTc)::value, NS = decltype(NSc)::value;
        k_aca_row<T, C, OP, HH, NT, NS><<<nA, kThreads, 0, st>>>(P, S);
        HB_CUDA(cudaGetLastError());
        k_aca_col<T, C, OP, HH, NT, NS><<<nA, kThreads, 0, st>>>(P, S);
        HB_CUDA(cudaGetLastError());
        return HBEM_OK;
      });
      if (rc != HBEM_OK) return rc;
      HB_CUDA(cudaMemcpyAsync(h_counts, counts, 8, cudaMemcpyDeviceToHost, st));
      HB_CUDA(cudaStreamSynchronize(st));
      H->stats.row_jobs += nA;
      H->stats.col_jobs += h_counts[0];
      nA = h_counts[1];
      std::swap(la, la2);
      ++waves;
    }
  }
  const auto t_aca = std::chrono::steady_clock::now();
  // ---- classify admissible blocks --------------------------------------------
  std::vector<int> st_h(na), rk_h(na), ex_h(na);
  std::vector<double> rs_h(na);
  if (na > 0) {
    HB_CUDA(cudaMemcpy(st_h.data(), S.status, na * 4, cudaMemcpyDeviceToHost));
    HB_CUDA(cudaMemcpy(rk_h.data(), S.rank, na * 4, cudaMemcpyDeviceToHost));
    HB_CUDA(cudaMemcpy(ex_h.data(), S.exhausted, na * 4, cudaMemcpyDeviceToHost));
    HB_CUDA(cudaMemcpy(rs_h.data(), S.resid, na * 8, cudaMemcpyDeviceToHost));
  }
  std::vector<int> expand_slots, fallback_slots;
  std::vector<long long> expand_off;
  for (int q = 0; q < na; ++q) {
    const int lf = adm_leaf[q];
    const int s = st_h[q];
    if (s == ST_OVERFLOW)
      return set_error(HBEM_ERR_CAPACITY,
                       "ACA rank capacity %d exceeded for block rows [%d, %d) x cols [%d, %d); "
                       "raise rank_capacity",
                       tmax, ar0[q], ar0[q] + ah[q], ac0[q], ac0[q] + aw[q]);
    if (s == ST_POOL)
      return set_error(HBEM_ERR_CAPACITY, "ACA factor pool of %lld values exhausted",
                       (long long)S.pool_cap);
    H->rank[lf] = rk_h[q];
    H->resid[lf] = rs_h[q];
    H->flags[lf] = (s == ST_CONVERGED ? 1 : 0) | (ex_h[q] ? 2 : 0);
    const long long hw = (long long)ah[q] * aw[q];
    if (s == ST_CONVERGED) {
      H->stats.aca_converged++;
      if (ex_h[q]) H->stats.aca_exhausted++;
      if ((long long)rk_h[q] * (ah[q] + aw[q]) < hw) {
        H->kind[lf] = 1;
        H->lowrank_slots.push_back(q);
        H->off_u[lf] = H->u_entries;
        H->off_v[lf] = H->v_entries;
        H->lr_uoff.push_back(H->u_entries);
        H->lr_voff.push_back(H->v_entries);
        H->u_entries += (long long)ah[q] * rk_h[q];
        H->v_entries += (long long)aw[q] * rk_h[q];
        H->stats.lowrank_leaves++;
        continue;
      }
      expand_slots.push_back(q);
      expand_off.push_back(dense_total);
    } else {  // ST_FALLBACK: rank cap without convergence -> exact rows
      if (ex_h[q]) H->stats.aca_exhausted++;
      H->stats.aca_fallback_dense++;
      fallback_slots.push_back(q);
      dr0.push_back(ar0[q]); dh.push_back(ah[q]); dc0.push_back(ac0[q]); dw.push_back(aw[q]);
      doff.push_back(dense_total);
    }
    H->off_dense[lf] = dense_total;
    dense_total += hw;
  }
  H->stats.dense_leaves = nd + (int64_t)expand_slots.size() + (int64_t)fallback_slots.size();
  H->dense_entries = dense_total;
  // ---- dense arena -------------------------------------------------------------
  HB_CUDA(cudaMalloc(&H->dense, std::max<size_t>((size_t)dense_total * vb, vb)));
  const int nds = (int)dr0.size();
  if (nds > 0) {
    std::vector<int> tslot, tstart;
    long long maxq = 0;
    for (int s = 0; s < nds; ++s) {
      const long long hw = (long long)dh[s] * dw[s];
      for (long long t = 0; t < hw; t += kThreads) {
        tslot.push_back(s);
        tstart.push_back((int)t);
      }
      maxq += hw;
    }
    DenseDev D{};
    int *p;
    long long *pl;
    HB_CHECK(upload(H, &p, tslot)); D.tile_slot = p;
    HB_CHECK(upload(H, &p, tstart)); D.tile_start = p;
    HB_CHECK(upload(H, &p, dr0)); D.r0 = p;
    HB_CHECK(upload(H, &p, dc0)); D.c0 = p;
    HB_CHECK(upload(H, &p, dh)); D.h = p;
    HB_CHECK(upload(H, &p, dw)); D.w = p;
    HB_CHECK(upload(H, &pl, doff)); D.off = pl;
    D.out = H->dense;
    D.stat = stat;
    unsigned long long *scount;
    HB_CHECK(dalloc(H, &scount, 1));
    HB_CUDA(cudaMemsetAsync(scount, 0, 8, st));
    D.sing_count = scount;
    if (nt == 1 && ns == 1) {
      // touching P0 pairs <= 13 per element; bound by the entry count
      const long long cap = std::min<long long>(maxq, 16 * (m + 1));
      HB_CHECK(dalloc(H, &D.sing_slot, cap));
      HB_CHECK(dalloc(H, &D.sing_pos, cap));
    }
    const unsigned ntiles = (unsigned)tslot.size();
    int rc = dispatch_op(ctx->op, ctx->helm, nt, ns, [&](auto OPc, auto Hc, auto NTc, auto NSc) -> int {
      constexpr int OP = decltype(OPc)::value;
      constexpr bool HH = decltype(Hc)::value != 0;
      constexpr int NT = decltype(NTc)::value, NS = decltype(NSc)::value;
      k_dense<T, C, OP, HH, NT, NS><<<ntiles, kThreads, 0, st>>>(P, D);
      HB_CUDA(cudaGetLastError());
      if constexpr (NT == 1 && NS == 1) {
        k_dense_singular<T, C, OP, HH><<<148 * 16, kThreads, 0, st>>>(P, D);
        HB_CUDA(cudaGetLastError());
      }
      return HBEM_OK;
    });
    if (rc != HBEM_OK) return rc;
    if (nt == 1 && ns == 1) {
      unsigned long long ns_h = 0;
      HB_CUDA(cudaMemcpyAsync(&ns_h, scount, 8, cudaMemcpyDeviceToHost, st));
      HB_CUDA(cudaStreamSynchronize(st));
      H->stats.singular_pairs += (int64_t)ns_h;
    }
    H->stats.regular_pairs += maxq;
  }
  if (!expand_slots.empty()) {
    int *slots;
    long long *offs;
    HB_CHECK(upload(H, &slots, expand_slots));
    HB_CHECK(upload(H, &offs, expand_off));
    k_expand<T, C><<<(unsigned)expand_slots.size(), 128, 0, st>>>(slots, (int)expand_slots.size(), S, offs, H->dense);
    HB_CUDA(cudaGetLastError());
  }
  HB_CUDA(cudaStreamSynchronize(st));
  const auto t_end = std::chrono::steady_clock::now();
  unsigned long long stat_h[2] = {0, 0};
  HB_CUDA(cudaMemcpy(stat_h, stat, 16, cudaMemcpyDeviceToHost));
  // entries evaluated by ACA jobs + dense; singular counted separately
  H->stats.singular_pairs += (int64_t)stat_h[1];
  H->stats.regular_pairs += (int64_t)stat_h[0];
  H->stats.regular_pairs -= H->stats.singular_pairs;
  H->stats.waves = waves;
  H->stats.u_entries = H->u_entries;
  H->stats.v_entries = H->v_entries;
  H->stats.dense_entries = H->dense_entries;
  H->stats.seconds = std::chrono::duration<double>(t_end - t_start).count();
  (void)t_setup;
  (void)t_aca;
  return HBEM_OK;
}

}  // namespace

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
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if (ctx->precision == HBEM_DOUBLE)
    rc = ctx->helm ? assemble_t<double, true>(ctx, d, st, H) : assemble_t<double, false>(ctx, d, st, H);
  else
    rc = ctx->helm ? assemble_t<float, true>(ctx, d, st, H) : assemble_t<float, false>(ctx, d, st, H);
  if (rc != HBEM_OK) {
    delete H;
    return rc;
  }
  *out = H;
  return HBEM_OK;
}

int hbem_hmat_stats_get(const hbem_hmat *h, hbem_hmat_stats *s) {
  if (!h || !s) return set_error(HBEM_ERR_ARG, "null argument");
  *s = h->stats;
  return HBEM_OK;
}

int hbem_hmat_leaf_meta(const hbem_hmat *h, int32_t *kind, int32_t *rank, int32_t *flags,
                        int64_t *off_u, int64_t *off_v, int64_t *off_dense) {
  if (!h) return set_error(HBEM_ERR_ARG, "null hmat");
  const size_t L = (size_t)h->n_leaves;
  if (kind) std::copy(h->kind.begin(), h->kind.end(), kind);
  if (rank) std::copy(h->rank.begin(), h->rank.end(), rank);
  if (flags) std::copy(h->flags.begin(), h->flags.end(), flags);
  if (off_u) std::copy(h->off_u.begin(), h->off_u.end(), off_u);
  if (off_v) std::copy(h->off_v.begin(), h->off_v.end(), off_v);
  if (off_dense) std::copy(h->off_dense.begin(), h->off_dense.end(), off_dense);
  (void)L;
  return HBEM_OK;
}

int hbem_hmat_copy_arenas(const hbem_hmat *hc, void *u, void *v, void *dense) {
  clear_error();
  hbem_hmat *h = const_cast<hbem_hmat *>(hc);
  if (!h) return set_error(HBEM_ERR_ARG, "null hmat");
  HB_CUDA(cudaSetDevice(h->device));
  if (dense && h->dense_entries > 0)
    HB_CUDA(cudaMemcpy(dense, h->dense, (size_t)h->dense_entries * h->vbytes,
                       cudaMemcpyDeviceToHost));
  if ((u || v) && !h->lowrank_slots.empty()) {
    // pack in chunks of blocks through a staging buffer
    const size_t n = h->lowrank_slots.size();
    const long long chunk_vals = 64ll << 20;  // values per staging half
    void *su = nullptr, *sv = nullptr;
    HB_CUDA(cudaMalloc(&su, chunk_vals * h->vbytes));
    HB_CUDA(cudaMalloc(&sv, chunk_vals * h->vbytes));
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
      size_t q1 = q0;
      const long long ub = h->lr_uoff[q0], vbase = h->lr_voff[q0];
      long long ue = ub, ve = vbase;
      while (q1 < n) {
        const long long nu = (q1 + 1 < n ? h->lr_uoff[q1 + 1] : h->u_entries) - ub;
        const long long nv = (q1 + 1 < n ? h->lr_voff[q1 + 1] : h->v_entries) - vbase;
        if ((nu > chunk_vals || nv > chunk_vals) && q1 > q0) break;
        ue = ub + nu;
        ve = vbase + nv;
        ++q1;
        if (nu > chunk_vals || nv > chunk_vals) break;
      }
      const int cnt = (int)(q1 - q0);
      const unsigned grid = (unsigned)cnt;
      if (h->vbytes == 16)
        k_pack_factors<Cx<double>><<<grid, 128>>>(d_slots + q0, cnt, h->S, d_uo + q0, d_vo + q0,
                                                  ub, vbase, (Cx<double> *)su, (Cx<double> *)sv);
      else if (h->vbytes == 8 && h->complex_)
        k_pack_factors<Cx<float>><<<grid, 128>>>(d_slots + q0, cnt, h->S, d_uo + q0, d_vo + q0, ub,
                                                 vbase, (Cx<float> *)su, (Cx<float> *)sv);
      else if (h->vbytes == 8)
        k_pack_factors<double><<<grid, 128>>>(d_slots + q0, cnt, h->S, d_uo + q0, d_vo + q0, ub,
                                              vbase, (double *)su, (double *)sv);
      else
        k_pack_factors<float><<<grid, 128>>>(d_slots + q0, cnt, h->S, d_uo + q0, d_vo + q0, ub,
                                             vbase, (float *)su, (float *)sv);
      HB_CUDA(cudaGetLastError());
      if (u)
        HB_CUDA(cudaMemcpy((char *)u + ub * h->vbytes, su, (ue - ub) * h->vbytes,
                           cudaMemcpyDeviceToHost));
      if (v)
        HB_CUDA(cudaMemcpy((char *)v + vbase * h->vbytes, sv, (ve - vbase) * h->vbytes,
                           cudaMemcpyDeviceToHost));
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

}  // extern "C"
