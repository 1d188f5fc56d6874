// Near-field (inadmissible) dense leaves for P0 spaces (dense_leaf,
// hmatrix.py:676-699) and the tree-ordered element record gather.
//
// One warp per (leaf, 32-column tile): lane l keeps the trial element of
// leaf column 32 t + l in registers, test elements of 32 rows at a time are
// staged in shared memory and broadcast; rows are stored coalesced.
// Touching pairs (shared vertex / edge / identical) are integrated by the
// whole warp with the Sauter-Schwab rules (kernels.py:249-347) and handed
// back to the owning lane, so no element integral leaves the device.
#pragma once
#include <algorithm>

#include "aca_impl.cuh"

namespace hb {

// record tp <- element perm[tp] (ctx geometry, element-indexed)
template <typename T>
__global__ void k_build_recs(Geo<T> g, const int4 *elem, const int *perm, int n, T *recs) {
  const int tp = blockIdx.x * blockDim.x + threadIdx.x;
  if (tp >= n) return;
  const int e = perm[tp];
  constexpr int L = RecLen<T>::value;
  T q[18], nj[4];
  load_q<T>(g.q, e, q);
  load_nj<T>(g.nj, e, nj);
  T *r = recs + (int64_t)tp * L;
#pragma unroll
  for (int i = 0; i < 18; ++i) r[i] = q[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) r[18 + i] = nj[i];
  const int4 v = elem[e];
  int4 *ev = reinterpret_cast<int4 *>(r + L - 16 / sizeof(T));
  *ev = make_int4(v.x, v.y, v.z, e);
}

template <typename T, bool C, int OP, bool HELM>
__global__ void __launch_bounds__(kThreads, HB_ACA_MINB) k_near_p0(Prob<T> P, DenseDev D) {
  using N = Num<T, C>;
  using V = typename N::V;
  constexpr unsigned kAll = 0xffffffffu;
  __shared__ FixRec<T> sr[kWarps][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long item = (long long)blockIdx.x * kWarps + wid;
  if (item >= D.n_items) return;
  const int2 it = D.items[item];
  const int s = it.x, t = it.y;
  const int h = D.h[s], w = D.w[s], r0 = D.r0[s], c0 = D.c0[s];
  const int c = t * 32 + lane;
  const bool valid = c < w;
  ElemRec<T> my;
  load_rec<T>(P.srec, c0 + (valid ? c : w - 1), my);
  T ny[6] = {T(0), T(0), T(0), T(0), T(0), T(0)};
  V *out = static_cast<V *>(D.out) + D.off[s];
  unsigned long long nsing = 0;
  for (int seg = 0; seg < h; seg += 32) {
    const int nseg = min(32, h - seg);
    if (lane < nseg) {
      ElemRec<T> r;
      load_rec<T>(P.trec, r0 + seg + lane, r);
      FixRec<T> f;
      fix_from_rec<T, false>(r, T(0), T(0), T(0), f);
      sr[wid][lane] = f;
    }
    __syncwarp();
    for (int i = 0; i < nseg; i += 2) {
      const int nj = i + 1 < nseg ? 2 : 1;
      V val[2];
      if (nj == 2) {
        const FixRec<T> *const F2[2] = {&sr[wid][i], &sr[wid][i + 1]};
        p0_quad<T, C, OP, HELM, true, 2, true>(P.R, F2, my.q, ny, my.n, val);
      } else {
        const FixRec<T> *const F1[1] = {&sr[wid][i]};
        V v1[1];
        p0_quad<T, C, OP, HELM, true, 1, true>(P.R, F1, my.q, ny, my.n, v1);
        val[0] = v1[0];
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (u < nj) {
          const int4 fev = sr[wid][i + u].ev;
          if (valid && touching4(fev, my.ev)) {
            // Sauter-Schwab value from the singular table (computed once per
            // touching element pair, k_sing_table)
            const int b0 = D.nb_ptr[fev.w], b1 = D.nb_ptr[fev.w + 1];
            int j = b0;
            while (j < b1 && D.nb_idx[j] != my.ev.w) ++j;
            val[u] = static_cast<const V *>(D.stab)[j];
            ++nsing;
          }
          if (valid) out[(long long)(seg + i + u) * w + c] = val[u];
        }
      }
    }
    __syncwarp();
  }
  nsing = (unsigned long long)__reduce_add_sync(kAll, (unsigned)nsing);
  if (lane == 0 && nsing) atomicAdd(D.stat + 1, nsing);
}


// ---------------------------------------------------------------------------
// Singular table (P0): one warp per touching element pair (e, f) computes
// local_matrix(e, f) (kernels.py:330-347, canonical test>trial transpose
// included) in float64 and stores it at the (e, f) entry of e's neighbour
// list; for the single layer the value is symmetric bit for bit
// (S = S^T, kernels.py:340-344), so it is also stored at (f, e) and each
// unordered pair is integrated once.
// ---------------------------------------------------------------------------
#ifndef HB_SING_LANES
#define HB_SING_LANES 1
#endif
#ifndef HB_SING_PPW
#define HB_SING_PPW 8
#endif
constexpr int kSingPerWarp = HB_SING_PPW;

template <typename T, bool C, int OP, bool HELM, int NT, int NS>
__global__ void __launch_bounds__(kThreads) k_sing_table(Prob<T> P, DenseDev D) {
  using N = Num<T, C>;
  using V = typename N::V;
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  V *tab = static_cast<V *>(D.stab);
  for (long long q = warp; q < D.n_spairs; q += nw) {
    const int4 pr = D.spairs[q];
    double re[NT][NS], im[NT][NS];
    singular_local<OP, HELM, NT, NS, 32>(P.G64, pr.x, pr.y, re, im);
    // lane o < NT NS stores entry o of the block (and of its transpose at
    // the back slot: the symmetric operators give S(f,e) = S(e,f)^T)
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        if (lane == i * NS + j) {
          const V v = N::mk((T)re[i][j], (T)im[i][j]);
          tab[(long long)pr.z * NT * NS + i * NS + j] = v;
          if (pr.w >= 0) tab[(long long)pr.w * NT * NS + j * NT + i] = v;
        }
      }
  }
}

// Singular table, single layer on P0 (the C1/C3/C5 near field): one lane per
// touching pair, the pairs of one launch all of one touching class (sorted at
// setup, sort_sing_pairs), so every lane walks the same Sauter-Schwab rule and
// the rule loads are warp-uniform broadcasts; no cross-lane reduction.  The
// single layer is symmetric, so the pair is integrated in its canonical
// orientation (lower element index as test, kernels.py:340-344) and stored
// at both slots.
template <typename T, bool C, bool HELM>
__global__ void __launch_bounds__(kThreads) k_sing_lanes(Prob<T> P, DenseDev D, long long q0,
                                                         long long q1) {
  using N = Num<T, C>;
  using V = typename N::V;
  const long long q = q0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool act = q < q1;
  const int4 pr = D.spairs[act ? q : q0];  // idle lanes repeat a pair of the same class
  const int a = min(pr.x, pr.y), b = max(pr.x, pr.y);
  const int4 ea = P.G64.elem[a], eb = P.G64.elem[b];
  const int ta[3] = {ea.x, ea.y, ea.z}, tb[3] = {eb.x, eb.y, eb.z};
  int pa[3], pb[3];
  const int kind = classify_pair(ta, tb, pa, pb);
  double re[1][1], im[1][1];
  singular_pair_warp<HBEM_SLP, HELM, 1, 1, 1>(P.G64, a, b, kind, pa, pb, re, im);
  if (!act) return;
  const V v = N::mk((T)re[0][0], (T)im[0][0]);
  V *tab = static_cast<V *>(D.stab);
  tab[pr.z] = v;
  if (pr.w >= 0) tab[pr.w] = v;
}

template <typename T, bool C>
int sing_table_launch(const Prob<T> &P, const DenseDev &D, int op, bool helm, int nt, int ns,
                      cudaStream_t st) {
  if (D.n_spairs <= 0) return HBEM_OK;
  // short-lived CTAs (kSingPerWarp pairs per warp): the table runs on the
  // low-priority stream and must hand SM slots back to the ACA phases within
  // tens of microseconds, not hold them for the whole table
  const long long per_cta = (long long)kWarps * kSingPerWarp;
  const unsigned grid = (unsigned)std::min<long long>((D.n_spairs + per_cta - 1) / per_cta, 0x7fffffffll);
  if (op == HBEM_SLP && nt == 1 && ns == 1 && D.skind[3] == D.n_spairs && HB_SING_LANES) {
    // pairs sorted by touching class: one launch per class
    for (int c = 1; c < 4; ++c) {
      const long long q0 = D.skind[c - 1], q1 = D.skind[c];
      if (q1 <= q0) continue;
      const unsigned g = (unsigned)((q1 - q0 + kThreads - 1) / kThreads);
      if (helm != C) return set_error(HBEM_ERR_KERNEL, "value type does not match the equation");
      k_sing_lanes<T, C, C><<<g, kThreads, 0, st>>>(P, D, q0, q1);
      HB_CUDA(cudaGetLastError());
    }
    return HBEM_OK;
  }
  return dispatch_op(op, helm, nt, ns, [&](auto OPc, auto Hc, auto NTc, auto NSc) -> int {
    constexpr int OP = decltype(OPc)::value;
    constexpr bool HH = decltype(Hc)::value != 0;
    constexpr int NT = decltype(NTc)::value, NS = decltype(NSc)::value;
    if constexpr (HH == C) {
      k_sing_table<T, C, OP, HH, NT, NS><<<grid, kThreads, 0, st>>>(P, D);
      HB_CUDA(cudaGetLastError());
      return HBEM_OK;
    } else {
      return set_error(HBEM_ERR_KERNEL, "value type does not match the equation");
    }
  });
}

template <typename T, bool C>
int near_p0_launch(const Prob<T> &P, const DenseDev &D, int op, bool helm, cudaStream_t st) {
  if (D.n_items <= 0) return HBEM_OK;
  const unsigned grid = (unsigned)((D.n_items + kWarps - 1) / kWarps);
  return dispatch_op(op, helm, 1, 1, [&](auto OPc, auto Hc, auto, auto) -> int {
    constexpr int OP = decltype(OPc)::value;
    constexpr bool HH = decltype(Hc)::value != 0;
    if constexpr (HH == C && OP != HBEM_HYPS) {
      k_near_p0<T, C, OP, HH><<<grid, kThreads, 0, st>>>(P, D);
      HB_CUDA(cudaGetLastError());
      return HBEM_OK;
    } else {
      return set_error(HBEM_ERR_KERNEL, "unsupported P0 near-field operator");
    }
  });
}

template <typename T>
int build_recs(const Geo<T> &g, const int4 *elem, const int *perm, int n, T *recs,
               cudaStream_t st) {
  if (n <= 0) return HBEM_OK;
  k_build_recs<T><<<(n + 127) / 128, 128, 0, st>>>(g, elem, perm, n, recs);
  HB_CUDA(cudaGetLastError());
  return HBEM_OK;
}

}  // namespace hb
