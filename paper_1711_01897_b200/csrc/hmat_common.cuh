// Shared device-side types of the H-matrix assembler (hmat.cu host side,
// aca_impl.cuh lock-step ACA waves, near_impl.cuh near-field leaves).
//
// Reference: /root/reference/pkg/src/hbem/hmatrix.py
//   aca                 271-382   (pivoting, stopping, Frobenius update)
//   _row_job/_col_job   625-672   (entry = sum over carrying element pairs)
//   dense_leaf          676-699
//   assemble_hmatrix    759-811
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "hbem_internal.h"

#ifndef HB_INNER_UNROLL2
#define HB_INNER_UNROLL2 6  // fixed-point loop unroll of the two-job quadrature
#endif
#ifndef HB_ACA_MINB
#define HB_ACA_MINB 3  // k_aca_p0 / k_near_p0 resident CTAs per SM (register cap)
#endif

namespace hb {

constexpr int kInnerUnroll2 = HB_INNER_UNROLL2;

// ---------------------------------------------------------------------------
// value arithmetic (real T or complex as (re, im) pairs, numpy layout)
// ---------------------------------------------------------------------------
template <typename T> struct Cx { T re, im; };

template <typename T, bool C> struct Num;
template <typename T, bool C> struct NumV;
template <typename T> struct Num<T, false> {
  using V = T;
  static constexpr int NC = 1;
  __device__ static V mk(T r, T) { return r; }
  __device__ static V fms(V a, V b, V c) { return a - b * c; }
  __device__ static double abs(V a) { return fabs((double)a); }
  __device__ static double nrm(V a) { return (double)a * (double)a; }
  __device__ static void cdot(double &re, double &, V a, V b) { re += (double)a * (double)b; }
  __device__ static V div(V a, V b) { return a / b; }
  __device__ static V zero() { return T(0); }
  __device__ static V fma_acc(V acc, V a, V b) { return acc + a * b; }
  __device__ static T re(V a) { return a; }
  __device__ static T im(V) { return T(0); }
};
template <typename T> struct Num<T, true> {
  using V = Cx<T>;
  static constexpr int NC = 2;
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
  __device__ static T re(V a) { return a.re; }
  __device__ static T im(V a) { return a.im; }
};

template <typename T, bool C> using V_t = typename Num<T, C>::V;

// ---------------------------------------------------------------------------
// Tree-ordered element records (P0 spaces: DOF = element).  Record tp holds
// the element at cluster-tree position tp, so a cluster [start, start + n)
// is n consecutive records: warps read a varying cluster coalesced and keep
// one element per lane in registers.  Layout (T units): qpoints 18 | nx ny
// nz |J| | (v0, v1, v2, element id) as 4 x int32, padded to 16-byte vectors.
// ---------------------------------------------------------------------------
template <typename T> struct RecLen;
template <> struct RecLen<double> { static constexpr int value = 24; };  // 192 B
template <> struct RecLen<float> { static constexpr int value = 28; };   // 112 B

template <typename T> struct ElemRec {
  T q[18];
  T n[4];       // nx, ny, nz, |J|
  int4 ev;      // vertex ids, element id
};

template <typename T> __device__ __forceinline__ void load_rec(const T *recs, int64_t tp,
                                                               ElemRec<T> &r);
template <> __device__ __forceinline__ void load_rec<double>(const double *recs, int64_t tp,
                                                             ElemRec<double> &r) {
  const double2 *p = reinterpret_cast<const double2 *>(recs + tp * 24);
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const double2 v = __ldg(p + i);
    r.q[2 * i] = v.x;
    r.q[2 * i + 1] = v.y;
  }
  const double2 a = __ldg(p + 9), b = __ldg(p + 10);
  r.n[0] = a.x; r.n[1] = a.y; r.n[2] = b.x; r.n[3] = b.y;
  r.ev = __ldg(reinterpret_cast<const int4 *>(p + 11));
}
template <> __device__ __forceinline__ void load_rec<float>(const float *recs, int64_t tp,
                                                            ElemRec<float> &r) {
  const float4 *p = reinterpret_cast<const float4 *>(recs + tp * 28);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float4 v = __ldg(p + i);
    r.q[4 * i] = v.x; r.q[4 * i + 1] = v.y; r.q[4 * i + 2] = v.z; r.q[4 * i + 3] = v.w;
  }
  const float4 v4 = __ldg(p + 4);
  r.q[16] = v4.x; r.q[17] = v4.y; r.n[0] = v4.z; r.n[1] = v4.w;
  const float4 v5 = __ldg(p + 5);
  r.n[2] = v5.x; r.n[3] = v5.y;
  r.ev = __ldg(reinterpret_cast<const int4 *>(p + 6));
}

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
  // P0: tree-ordered element records (test / trial tree; may alias)
  const T *trec, *srec;
  const Geo64 *G64p;  // device copy of G64 (rarely used paths)
  // singular table (k_sing_table): touching element pairs -> NT x NS block
  const int *nb_ptr, *nb_idx;
  const void *stab;
};

// Point kernel of kernel_planes (kernels.py:129-158) for d = x - y:
// SLP 1/r, DLP <d, n_y>/r^3, ADLP -<d, n_x>/r^3, Helmholtz factors e^{ikr}
// (SLP) and (cos kr + kr sin kr, sin kr - kr cos kr) (DLP/ADLP); 1/(4 pi)
// is applied by the caller.  nt / nf: normal of the test / trial element.
template <typename T, int OP, bool HELM>
__device__ __forceinline__ void point_kernel(const RuleTab<T> &R, T d0, T d1, T d2,
                                             const T *ntest, const T *ntrial, T &gr, T &gi) {
  const T r2 = d0 * d0 + d1 * d1 + d2 * d2;
  const T ri = rsqrt_t<T>(r2);
  gi = T(0);
  if (OP == HBEM_SLP) {
    if (!HELM) {
      gr = ri;
    } else {
      const T kr = R.k * (r2 * ri);
      T s, c;
      sincos_t<T>(kr, &s, &c);
      gr = ri * c;
      gi = ri * s;
    }
  } else {
    const T dot = OP == HBEM_DLP ? d0 * ntrial[0] + d1 * ntrial[1] + d2 * ntrial[2]
                                 : -(d0 * ntest[0] + d1 * ntest[1] + d2 * ntest[2]);
    const T amp = dot * (ri * ri * ri);
    if (!HELM) {
      gr = amp;
    } else {
      const T kr = R.k * (r2 * ri);
      T s, c;
      sincos_t<T>(kr, &s, &c);
      gr = amp * (c + kr * s);
      gi = amp * (s - kr * c);
    }
  }
}

// block of one element pair (any adjacency), thread-level
template <typename T, int OP, bool HELM, int NT, int NS>
__device__ __forceinline__ void pair_block(const Prob<T> &P, int e, int f, T (&re)[NT][NS],
                                           T (&im)[NT][NS], unsigned long long *nsing) {
  if (touching(P.elem[e], P.elem[f])) {
    if (P.stab) {
      // Sauter-Schwab block from the singular table (one integration per
      // touching element pair and execute, warp-cooperative)
      int j = P.nb_ptr[e];
      while (P.nb_idx[j] != f) ++j;
      const T *blk = static_cast<const T *>(P.stab) + (long long)j * NT * NS * (HELM ? 2 : 1);
#pragma unroll
      for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int jj = 0; jj < NS; ++jj) {
          const int o = i * NS + jj;
          re[i][jj] = HELM ? blk[2 * o] : blk[o];
          im[i][jj] = HELM ? blk[2 * o + 1] : T(0);
        }
      if (nsing) atomicAdd(nsing, 1ull);
      return;
    }
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
    T x[18], na[4];
    if (OP != HBEM_HYPS) {
      load_q<T>(P.g.q, e, x);
      load_nj<T>(P.g.nj, e, na);
    }
    for (int s = s0; s < s1; ++s) {
      const int f = NS == 1 ? dj : P.sel[s];
      const int b = NS == 1 ? 0 : P.sloc[s];
      if (OP != HBEM_HYPS && !touching(P.elem[e], P.elem[f])) {
        // only the (a, b) basis pair of the block is needed: one weighted
        // accumulation per quadrature-point pair instead of the 3 x 3 block
        T y[18], nb[4];
        load_q<T>(P.g.q, f, y);
        load_nj<T>(P.g.nj, f, nb);
        T sr = T(0), si = T(0);
#pragma unroll
        for (int pp = 0; pp < 6; ++pp) {
          T ar = T(0), ai = T(0);
#pragma unroll
          for (int qq = 0; qq < 6; ++qq) {
            T gr, gi;
            point_kernel<T, OP, HELM>(P.R, x[3 * pp] - y[3 * qq], x[3 * pp + 1] - y[3 * qq + 1],
                                      x[3 * pp + 2] - y[3 * qq + 2], na, nb, gr, gi);
            ar += P.R.wb[b][qq] * gr;
            if (HELM) ai += P.R.wb[b][qq] * gi;
          }
          sr += P.R.wa[a][pp] * ar;
          if (HELM) si += P.R.wa[a][pp] * ai;
        }
        const T scale = (na[3] * nb[3]) * T(kInv4Pi);
        const typename N::V val = N::mk(scale * sr, HELM ? scale * si : T(0));
        if constexpr (C) { acc.re += val.re; acc.im += val.im; }
        else acc += val;
        continue;
      }
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

// regular P0 pair from two element records (test x, trial y)
template <typename T, bool C, int OP, bool HELM>
__device__ __forceinline__ typename Num<T, C>::V p0_regular(const RuleTab<T> &R,
                                                             const T (&x)[18], const T (&na)[4],
                                                             const T (&y)[18], const T (&nb)[4]) {
  T re[1][1], im[1][1];
  regular_pair<T, OP, HELM, 1, 1>(R, x, y, na, nb, nullptr, nullptr, re, im);
  return Num<T, C>::mk(re[0][0], im[0][0]);
}

// Regular P0 pairs of NJ fixed elements (points read from shared memory in
// the inner loop, broadcast to the warp) against the lane's element in
// registers (outer loop).  The NJ pairs are independent dependency chains
// that share the lane's points, which doubles the instruction-level
// parallelism at the cost of a few accumulators.  FIXED_TEST: the fixed
// elements are test elements x (row jobs, near-field rows); otherwise trial
// elements y (column jobs).  The double sum runs lane-side outer.
template <typename T, bool C, int OP, bool HELM, bool FIXED_TEST, int NJ>
__device__ __forceinline__ void p0_pairs_fx(const RuleTab<T> &R, const ElemRec<T> *const (&F)[NJ],
                                            const T (&y)[18], const T (&nl)[4],
                                            typename Num<T, C>::V (&out)[NJ]) {
  T sr[NJ], si[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) { sr[j] = T(0); si[j] = T(0); }
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const T y0 = y[3 * i], y1 = y[3 * i + 1], y2 = y[3 * i + 2];
    T ar[NJ], ai[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) { ar[j] = T(0); ai[j] = T(0); }
#pragma unroll(NJ == 1 ? 2 : (HELM ? 2 : kInnerUnroll2))
    for (int o = 0; o < 6; ++o) {
      const T wo = FIXED_TEST ? R.wa[0][o] : R.wb[0][o];
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const ElemRec<T> &G = *F[j];
        const T d0 = FIXED_TEST ? G.q[3 * o] - y0 : y0 - G.q[3 * o];
        const T d1 = FIXED_TEST ? G.q[3 * o + 1] - y1 : y1 - G.q[3 * o + 1];
        const T d2 = FIXED_TEST ? G.q[3 * o + 2] - y2 : y2 - G.q[3 * o + 2];
        T gr, gi;
        point_kernel<T, OP, HELM>(R, d0, d1, d2, FIXED_TEST ? G.n : nl, FIXED_TEST ? nl : G.n,
                                  gr, gi);
        ar[j] += wo * gr;
        if (HELM) ai[j] += wo * gi;
      }
    }
    const T wi = FIXED_TEST ? R.wb[0][i] : R.wa[0][i];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      sr[j] += wi * ar[j];
      if (HELM) si[j] += wi * ai[j];
    }
  }
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const T scale = (F[j]->n[3] * nl[3]) * T(kInv4Pi);
    out[j] = Num<T, C>::mk(scale * sr[j], HELM ? scale * si[j] : T(0));
  }
}

// warp-cooperative Sauter-Schwab value of the touching pair (e test, f
// trial) in float64 (local_matrix, kernels.py:330-347), kept out of line so
// its registers do not bound the occupancy of the regular path
template <int OP, bool HELM>
__device__ __noinline__ double2 singular_warp(const Geo64 *__restrict__ Gp, int e, int f) {
  // the geometry view is read from global memory here, on the rare
  // touching path, instead of being held in registers by every caller
  const Geo64 G = *Gp;
  double re[1][1], im[1][1];
  singular_local<OP, HELM, 1, 1, 32>(G, e, f, re, im);
  return make_double2(re[0][0], im[0][0]);
}

__device__ __forceinline__ bool touching4(const int4 &a, const int4 &b) {
  return a.x == b.x || a.x == b.y || a.x == b.z || a.y == b.x || a.y == b.y || a.y == b.z ||
         a.z == b.x || a.z == b.y || a.z == b.z;
}

// ---------------------------------------------------------------------------
// warp helpers
// ---------------------------------------------------------------------------
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
__device__ __forceinline__ int first_clear(const unsigned *m, int n) {
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
// ACA state (one entry per admissible block b)
// ---------------------------------------------------------------------------
enum : int { ST_ACTIVE = 0, ST_CONVERGED = 1, ST_FALLBACK = 2, ST_OVERFLOW = 3 };

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kNeedThreads = 256;  // k_need block size (block-scan width)
constexpr size_t kStageRecMax = 512;  // bytes per job of the P0 stage records (StageRec)
constexpr long long kPoolSlack = 64;  // factor-pool values kept mapped past the last record
constexpr int kFinRegs = 8;  // terms gathered per job by k_jobs and held in registers by k_fin

// One ACA job of the current phase: the next row (row phase) or pivot column
// (column phase) of block b.  The "fixed" index is the row i / column j; the
// "varying" side is the column / row cluster the entries run over.
struct Job {
  int b, key;       // block, grouping key (varying-side cluster node)
  int fix;          // row i / column j within the block
  int h, w, k;      // block shape, accepted rank so far
  int nfix;         // tree position of the fixed DOF
  int vstart, nvar; // varying cluster start (tree position) and length
  int cur;          // column phase: the block's current row i (excluded from the next pivot)
  long long pe;     // pool record of the pending term [u (h) | v (w)]
  long long part;   // first partial record of this job (doubles)
  long long rsc;    // linear spaces: element-row values of this job (V units)
  long long mofs;   // used-index mask words of the varying side (rmask / cmask offset)
};

// partial record per (job, 32-wide tile): best |val| over unmasked entries,
// its index, sum |val|^2, then k dots (re, im for complex) with the factor
// the residual used: row phase vdot(v_l, row), column phase vdot(u_l, col).
// per job: nt tile statistics records of 4 doubles (best |val| over unmasked,
// its index, sum |val|^2, pad) followed by nt dot records of k*nc doubles
// (record length rounded up to an even number of doubles: 16-byte aligned records)
__host__ __device__ __forceinline__ long long part_len(int k, int nc) {
  return (4 + (long long)k * nc + 1) & ~1ll;
}
__host__ __device__ __forceinline__ long long part_dots(int nt) { return 4ll * nt; }
__host__ __device__ __forceinline__ int tiles_of(int n) { return (n + 31) >> 5; }

// per-position allocation need: pool values, dot-record doubles, DOF-tile warp
// items, element-tile warp items (linear spaces) and element-row values
// (linear spaces: NT or NS per element of the varying cluster's union)
struct Need {
  long long pool, part, items, eitems, rsc;
};
struct SumNeed {
  __device__ __forceinline__ Need operator()(const Need &a, const Need &b) const {
    return Need{a.pool + b.pool, a.part + b.part, a.items + b.items, a.eitems + b.eitems,
                a.rsc + b.rsc};
  }
};

// static per-block fields in one record: a job's block costs one or two
// sectors instead of one per field array
struct BlockInfo {
  int h, w, r0, c0, rnode, cnode;
  long long rmo, cmo;  // used-index mask word offsets (rows, columns)
};

struct AcaDev {
  // static per block
  const int *h, *w, *r0, *c0, *rnode, *cnode;
  // iteration state
  int *rank, *cur, *pcol, *small, *status, *exhausted;
  double *norm2, *resid, *rn2, *piv;  // piv: pivot of the pending row (re, im)
  long long *pend, *terms;            // pending record, accepted term records (tmax per block)
  long long *rowpart;                 // row-phase partial record 0 of the block's pending row
  double *rsum;                       // row-phase dots of the first kFinRegs terms summed over
                                      // the tiles (kFinRegs x 2 per block, k_fin_row)
  int tmax;
  unsigned *rmask, *cmask;
  const long long *rmask_off, *cmask_off;
  const struct BlockInfo *binfo;  // the static fields above, one record per block (k_jobs)
  void *pool;
  long long pool_cap, pool_base;
  int kmax_cfg;
  double eps;
  unsigned char *flagA, *flagC;  // block needs a row job next wave / a column job this wave
  // current phase
  const int *list;   // positions -> block (sorted by key)
  const int *nlist;  // device count of list
  Need *need, *scan;
  int *pkey;         // per list position: the grouping key (k_need)
  Job *jobs;
  int4 *items;       // (head position, tile, varying start, varying length)
  int *iglen;        // per item: jobs in its group
  void *stage;       // P0: per job position, its StageRec (k_jobs -> k_aca_p0)
  int2 *eitems;      // linear spaces: (head position, element tile)
  void *rsc;         // linear spaces: element-row values of the current phase
  // linear spaces: per cluster node, the sorted union of the elements that
  // carry its DOFs (row tree / column tree CSR)
  const long long *recl_ptr, *cecl_ptr;
  const int *recl, *cecl;
  double *part;      // dot records of the current phase (k values per job)
  void *tpiv;        // per block and term: the term's pivot value (V), contiguous per block
  long long *jt;     // per job: record offsets of its first kFinRegs terms
  void *jc;          // per job: their residual coefficients (u_l[i] / p_l or r_l[j] / p_l)
  const double *rpart;  // row-phase partial records (read by the column finalize)
  unsigned long long *stat;  // [0] entries evaluated, [1] singular pairs
};

// ---------------------------------------------------------------------------
// dense entries (near-field leaves and ACA fallback blocks)
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
  // P0 warp items: (slot, column tile)
  const int2 *items;
  long long n_items;
  // P0 singular table: element -> sorted touching elements (CSR) and the
  // Sauter-Schwab value of every (element, neighbour) entry
  const int *nb_ptr, *nb_idx;
  void *stab;
  const int4 *spairs;  // (test e, trial f, slot of (e,f), slot of (f,e) or -1)
  long long n_spairs;
  long long skind[4];  // sorted by touching class: pairs of class c at [skind[c-1], skind[c])
};

// P0 singular-table construction (setup) and evaluation (execute)
struct SingTable {
  int *nb_ptr = nullptr, *nb_idx = nullptr;
  int4 *pairs = nullptr;
  long long nnz = 0, n_pairs = 0;
  long long kind_n[4] = {0, 0, 0, 0};  // pairs per touching class after sort_sing_pairs
};
int build_sing_table(const int4 *d_elem, int m, int nv, bool symmetric, SingTable &out,
                     std::vector<void *> &allocs, cudaStream_t st);
// keep only the touching pairs some near-field leaf of this handle reads
// (P0: row element in the leaf's row cluster, trial element in its column
// cluster), so a rank assembling a slice of the leaves integrates only its
// share of the Sauter-Schwab table
// order the pairs by touching class (vertex, edge, identical; stable), so a
// warp's 32 pairs share one Sauter-Schwab rule (lane-per-pair table kernel)
int sort_sing_pairs(SingTable &tab, const int4 *d_elem, std::vector<void *> &allocs,
                    cudaStream_t st);
int restrict_sing_pairs(SingTable &tab, const int *rperm, const int *cinv,
                        const long long *rowbase, int nd, long long nrows, const int *r0,
                        const int *c0, const int *w, std::vector<void *> &allocs,
                        cudaStream_t st);

// ---------------------------------------------------------------------------
// launchers (aca_f64.cu / aca_f32.cu, near_f64.cu / near_f32.cu)
// ---------------------------------------------------------------------------
struct PhaseArgs {
  int na;             // admissible blocks
  int col_phase;
  const int *order;   // static block order of this phase (sorted by key)
  void *cub_tmp;
  size_t cub_bytes;
  int *sel_tmp;       // na flags scratch for the compaction
  int nt, ns;         // basis functions per element (test, trial)
  cudaEvent_t int_beg, int_end;  // recorded around the integration launch (may be null)
};

template <typename T, bool C>
int aca_init(const Prob<T> &P, AcaDev &S, int na, cudaStream_t st);
// list selection + need scan (no host sync)
template <typename T, bool C>
int aca_select(const Prob<T> &P, AcaDev &S, const PhaseArgs &A, cudaStream_t st);
// jobs + items + integration + finalize for a phase of n jobs and n_items items
template <typename T, bool C>
int aca_phase(const Prob<T> &P, AcaDev &S, const PhaseArgs &A, int op, bool helm, int nt, int ns,
              int n, long long n_items, long long n_eitems, cudaStream_t st);
size_t aca_cub_bytes(int na);

template <typename T>
int build_recs(const Geo<T> &g, const int4 *elem, const int *perm, int n, T *recs, cudaStream_t st);
struct MatvecArgs {
  int n_rows, n_cols;
  const int *rperm, *cperm;
  const void *x;  // device, original DOF order
  void *y;        // device, original DOF order
  void *xt, *yt;  // device scratch, tree order
  struct Dense {
    int n;
    const int *r0, *c0, *h, *w;
    const long long *off, *rowbase;
    long long nrows;
    const void *arena;
    long long part_base;  // first partial slot of this list (leaf row g -> part_base + g)
  } dense[2];     // near-field leaves, admissible blocks stored densely
  int n_lowrank;
  const int *lowrank;  // admissible block slots
  // packed factors (U h x k, V w x k per block, v = r / p applied): the
  // matvec streams these instead of the scattered pool terms
  const void *ua, *va;
  const long long *uoff, *voff;  // per admissible block
  // work items (low-rank list position, chunk start), <= kMvChunk rows or
  // columns each, so one huge block does not serialise on one warp
  long long n_ditems, n_ritems;
  const int2 *ditems, *ritems;
  const long long *sbase;   // per list position: offset of its k dots in s
  const long long *ifirst;  // per list position: first dots item (n_lowrank + 1)
  const long long *ibase;   // per dots item: offset of its k partial dots in dpart
  const long long *rbase;   // per list position: first partial slot of its rows
  void *s;                  // per-block dots
  void *dpart;              // per-chunk partial dots
  long long n_s;
  // deterministic reduction: every leaf's row contributions in private slots
  // (part), summed per row over the covering leaves in the reference's
  // (row start, column start) order, one warp per row cluster of the tree
  void *part;
  int n_clusters;
  const int *cstart;        // n_clusters + 1 row-cluster starts
  const long long *cptr;    // n_clusters + 1 offsets into cover
  const long long *cover;   // slot base minus the leaf's first row
};
constexpr int kMvChunk = 512;
template <typename T, bool C>
int matvec_launch(const MatvecArgs &M, const AcaDev &S, cudaStream_t st);
template <typename T, bool C>
int sing_table_launch(const Prob<T> &P, const DenseDev &D, int op, bool helm, int nt, int ns,
                      cudaStream_t st);
template <typename T, bool C>
int near_p0_launch(const Prob<T> &P, const DenseDev &D, int op, bool helm, cudaStream_t st);

}  // namespace hb
