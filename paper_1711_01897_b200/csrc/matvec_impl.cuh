// Device H-matrix matvec y = H x (hmat_matvec, hmatrix.py:441-470) straight
// from the device arenas: dense leaves row by row, low-rank blocks from the
// packed U / V arenas (contiguous per block; the ACA pool scatters a block's
// terms over one region per wave, which costs a TLB miss per term).
//
// Bit-reproducible like the reference ("leaves are applied sequentially in a
// fixed (row, column) order, so the result is reproducible bit for bit
// between calls"): no float atomics.  Every leaf writes its own row
// contributions into a private slot range (partials), chunked low-rank dots
// are summed per block in chunk order, and one warp per row cluster of the
// tree adds, for each of its rows, the contributions of the leaves covering
// it in the reference's (row start, column start) order.
#pragma once
#include "hmat_common.cuh"

namespace hb {

template <typename T, bool C>
__device__ __forceinline__ typename Num<T, C>::V warp_sum_v(typename Num<T, C>::V v) {
  using N = Num<T, C>;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    if constexpr (C) {
      v.re += __shfl_xor_sync(0xffffffffu, v.re, o);
      v.im += __shfl_xor_sync(0xffffffffu, v.im, o);
    } else {
      v += __shfl_xor_sync(0xffffffffu, v, o);
    }
  }
  (void)sizeof(N);
  return v;
}

// one warp per dense-leaf row; rowbase: exclusive prefix of leaf heights
template <typename T, bool C>
__global__ void k_mv_dense(int nl, const int *r0, const int *c0, const int *h, const int *w,
                           const long long *off, const long long *rowbase, long long nrows,
                           const void *arena, const void *xt, void *part) {
  using N = Num<T, C>;
  using V = typename N::V;
  const long long g = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= nrows) return;
  int lo = 0, hi = nl;  // last leaf with rowbase <= g
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (rowbase[mid] <= g) lo = mid;
    else hi = mid;
  }
  const int s = lo, i = (int)(g - rowbase[s]), ww = w[s];
  const V *A = static_cast<const V *>(arena) + off[s] + (long long)i * ww;
  const V *x = static_cast<const V *>(xt) + c0[s];
  V acc = N::zero();
  for (int c = lane; c < ww; c += 32) acc = N::fma_acc(acc, A[c], x[c]);
  acc = warp_sum_v<T, C>(acc);
  if (lane == 0) static_cast<V *>(part)[g] = acc;  // slot: leaf row g of this list
}

template <typename T, bool C>
__device__ __forceinline__ typename Num<T, C>::V shfl_v(typename Num<T, C>::V v, int src) {
  if constexpr (C) {
    v.re = __shfl_sync(0xffffffffu, v.re, src);
    v.im = __shfl_sync(0xffffffffu, v.im, src);
    return v;
  } else {
    return __shfl_sync(0xffffffffu, v, src);
  }
}

// one warp per dense leaf (near field: at most 32 x 32): lane r owns row r and
// streams it (each row's 32 values are one 256-byte run, so every DRAM sector
// is used once through L1), x of the leaf's columns is broadcast by shuffles;
// no per-row warp reduction and no leaf search.  The sum order per row is the
// column order, fixed.
template <typename T, bool C>
__global__ void k_mv_dense_leaf(int nl, const int *c0, const int *h, const int *w,
                                const long long *off, const long long *rowbase,
                                const void *arena, const void *xt, void *part) {
  using N = Num<T, C>;
  using V = typename N::V;
  const long long s = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= nl) return;
  const int hh = h[s], ww = w[s];
  const V *A = static_cast<const V *>(arena) + off[s];
  const V *x = static_cast<const V *>(xt) + c0[s];
  V *out = static_cast<V *>(part) + rowbase[s];
  for (int r0 = 0; r0 < hh; r0 += 32) {
    const int r = r0 + lane;
    const V *row = A + (long long)(r < hh ? r : 0) * ww;
    V acc = N::zero();
    for (int c0_ = 0; c0_ < ww; c0_ += 32) {
      const V xv = c0_ + lane < ww ? x[c0_ + lane] : N::zero();
      const int cn = min(32, ww - c0_);
#pragma unroll 8
      for (int c = 0; c < cn; ++c) acc = N::fma_acc(acc, row[c0_ + c], shfl_v<T, C>(xv, c));
    }
    if (r < hh) out[r] = acc;
  }
}

// one warp per low-rank block: s_l = v_l . x, y += sum_l u_l s_l.  The term
// offsets and pivots are fetched lane-parallel (lane l holds term l) and
// broadcast by shuffles, so every factor load is independent of the others
// (no per-term dependent global load); dots run four terms at a time.

// low-rank blocks in two passes over (block, chunk) work items:
//   dots: warp per (block, <= kMvChunk columns): s_l += v_l[chunk] . x[chunk]
//   rows: warp per (block, <= kMvChunk rows):    y[chunk] += sum_l u_l[chunk] s_l
template <typename T, bool C>
__global__ void k_mv_dots(long long n, const int2 *items, const int *slots, AcaDev S,
                          const void *va, const long long *voff, const long long *ibase,
                          const void *xt, void *dpart) {
  using N = Num<T, C>;
  using V = typename N::V;
  const long long it = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (it >= n) return;
  const int2 wi = items[it];
  const int b = slots[wi.x];
  const int w = S.w[b], k = S.rank[b];
  const int c0 = wi.y, c1 = min(w, c0 + kMvChunk);
  const V *W = static_cast<const V *>(va) + voff[b];  // column l: W[l * w + c]
  const V *x = static_cast<const V *>(xt) + S.c0[b];
  V *sd = static_cast<V *>(dpart) + ibase[it];  // this chunk's k partial dots
  for (int l = 0; l < k; l += 4) {
    V acc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u] = N::zero();
    for (int c = c0 + lane; c < c1; c += 32) {
      const V xc = x[c];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (l + u < k) acc[u] = N::fma_acc(acc[u], W[(long long)(l + u) * w + c], xc);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const V d = warp_sum_v<T, C>(acc[u]);
      if (lane == 0 && l + u < k) sd[l + u] = d;
    }
  }
}

// dots of list position p: sum of its chunks' partial dots in chunk order
template <typename T, bool C>
__global__ void k_mv_dots_sum(int nl, const int *slots, AcaDev S, const long long *sbase,
                              const long long *ifirst, const long long *ibase,
                              const void *dpart, void *s) {
  using N = Num<T, C>;
  using V = typename N::V;
  const int p = blockIdx.x * (blockDim.x / 8) + threadIdx.x / 8;
  if (p >= nl) return;
  const int k = S.rank[slots[p]];
  const V *dp = static_cast<const V *>(dpart);
  for (int l = threadIdx.x % 8; l < k; l += 8) {
    V acc = N::zero();
    for (long long it = ifirst[p]; it < ifirst[p + 1]; ++it) {
      const V d = dp[ibase[it] + l];
      if constexpr (C) { acc.re += d.re; acc.im += d.im; }
      else acc += d;
    }
    static_cast<V *>(s)[sbase[p] + l] = acc;
  }
}

template <typename T, bool C>
__global__ void k_mv_rows(long long n, const int2 *items, const int *slots, AcaDev S,
                          const void *ua, const long long *uoff, const long long *sbase,
                          const void *s, const long long *rbase, void *part) {
  using N = Num<T, C>;
  using V = typename N::V;
  const long long it = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (it >= n) return;
  const int2 wi = items[it];
  const int b = slots[wi.x];
  const int h = S.h[b], k = S.rank[b];
  const int r0 = wi.y, r1 = min(h, r0 + kMvChunk);
  const V *U = static_cast<const V *>(ua) + uoff[b];  // column l: U[l * h + i]
  const V *sd = static_cast<const V *>(s) + sbase[wi.x];
  V *y = static_cast<V *>(part) + rbase[wi.x];  // this block's row slots
  for (int i0 = r0; i0 < r1; i0 += 32) {  // warp-uniform trip count (shuffles)
    const int i = i0 + lane;
    V acc = N::zero();
    for (int l0 = 0; l0 < k; l0 += 32) {
      const int lk = min(32, k - l0);
      const V mine = lane < lk ? sd[l0 + lane] : N::zero();
#pragma unroll 4
      for (int l = 0; l < lk; ++l) {
        const V sl = shfl_v<T, C>(mine, l);
        if (i < r1) acc = N::fma_acc(acc, U[(long long)(l0 + l) * h + i], sl);
      }
    }
    if (i < r1) y[i] = acc;
  }
}

// one warp per row cluster [cs, ce) of the tree (<= 32 rows): row r adds the
// contributions of the leaves covering it, cover list = slot bases minus the
// leaf's first row, in the reference's (row start, column start) order
template <typename T, bool C>
__global__ void k_mv_reduce(int ncl, const int *cstart, const long long *cptr,
                            const long long *cover, const void *part, void *yt) {
  using N = Num<T, C>;
  using V = typename N::V;
  const long long g = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= ncl) return;
  const int r = cstart[g] + lane;
  if (r >= cstart[g + 1]) return;
  const V *pp = static_cast<const V *>(part);
  V acc = N::zero();
  for (long long j = cptr[g]; j < cptr[g + 1]; ++j) {
    const V d = pp[cover[j] + r];
    if constexpr (C) { acc.re += d.re; acc.im += d.im; }
    else acc += d;
  }
  static_cast<V *>(yt)[r] = acc;
}

template <typename T, bool C>
__global__ void k_mv_gather(int n, const int *perm, const void *x, void *xt) {
  using V = typename Num<T, C>::V;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) static_cast<V *>(xt)[j] = static_cast<const V *>(x)[perm[j]];
}
template <typename T, bool C>
__global__ void k_mv_scatter(int n, const int *perm, const void *yt, void *y) {
  using V = typename Num<T, C>::V;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) static_cast<V *>(y)[perm[i]] = static_cast<const V *>(yt)[i];
}

template <typename T, bool C>
int matvec_launch(const MatvecArgs &M, const AcaDev &S, cudaStream_t st) {
  using V = typename Num<T, C>::V;
  k_mv_gather<T, C><<<(M.n_cols + 255) / 256, 256, 0, st>>>(M.n_cols, M.cperm, M.x, M.xt);
  for (int a = 0; a < 2; ++a) {
    const MatvecArgs::Dense &D = M.dense[a];
    if (D.n <= 0 || D.nrows <= 0) continue;
    if (a == 0) {  // near-field leaves: warp per leaf, lane per row
      k_mv_dense_leaf<T, C><<<(unsigned)((D.n + 3) / 4), 128, 0, st>>>(
          D.n, D.c0, D.h, D.w, D.off, D.rowbase, D.arena, M.xt,
          static_cast<V *>(M.part) + D.part_base);
    } else {  // admissible blocks stored densely (any width): warp per row
      const long long warps = D.nrows;
      k_mv_dense<T, C><<<(unsigned)((warps + 3) / 4), 128, 0, st>>>(
          D.n, D.r0, D.c0, D.h, D.w, D.off, D.rowbase, D.nrows, D.arena, M.xt,
          static_cast<V *>(M.part) + D.part_base);
    }
  }
  if (M.n_lowrank > 0) {
    k_mv_dots<T, C><<<(unsigned)((M.n_ditems + 3) / 4), 128, 0, st>>>(
        M.n_ditems, M.ditems, M.lowrank, S, M.va, M.voff, M.ibase, M.xt, M.dpart);
    k_mv_dots_sum<T, C><<<(unsigned)((M.n_lowrank + 15) / 16), 128, 0, st>>>(
        M.n_lowrank, M.lowrank, S, M.sbase, M.ifirst, M.ibase, M.dpart, M.s);
    k_mv_rows<T, C><<<(unsigned)((M.n_ritems + 3) / 4), 128, 0, st>>>(
        M.n_ritems, M.ritems, M.lowrank, S, M.ua, M.uoff, M.sbase, M.s, M.rbase, M.part);
  }
  k_mv_reduce<T, C><<<(unsigned)((M.n_clusters + 3) / 4), 128, 0, st>>>(
      M.n_clusters, M.cstart, M.cptr, M.cover, M.part, M.yt);
  k_mv_scatter<T, C><<<(M.n_rows + 255) / 256, 256, 0, st>>>(M.n_rows, M.rperm, M.yt, M.y);
  HB_CUDA(cudaGetLastError());
  return HBEM_OK;
}

}  // namespace hb
