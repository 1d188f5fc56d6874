// Device H-matrix matvec y = H x (hmat_matvec, hmatrix.py:441-470) straight
// from the device arenas: dense leaves row by row, low-rank blocks from the
// ACA factor pool (v = r / p applied on the fly).  Leaf contributions are
// accumulated with atomics (the sum order over leaves is not fixed, so
// results agree with the host matvec to rounding, not bitwise).
#pragma once
#include "hmat_common.cuh"

namespace hb {

template <typename V> __device__ __forceinline__ void atomic_add_v(V *p, V v);
template <> __device__ __forceinline__ void atomic_add_v<double>(double *p, double v) { atomicAdd(p, v); }
template <> __device__ __forceinline__ void atomic_add_v<float>(float *p, float v) { atomicAdd(p, v); }
template <> __device__ __forceinline__ void atomic_add_v<Cx<double>>(Cx<double> *p, Cx<double> v) {
  atomicAdd(&p->re, v.re);
  atomicAdd(&p->im, v.im);
}
template <> __device__ __forceinline__ void atomic_add_v<Cx<float>>(Cx<float> *p, Cx<float> v) {
  atomicAdd(&p->re, v.re);
  atomicAdd(&p->im, v.im);
}

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
                           const void *arena, const void *xt, void *yt) {
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
  if (lane == 0) atomic_add_v<V>(static_cast<V *>(yt) + r0[s] + i, acc);
}

// one warp per low-rank block: s_l = v_l . x, y += sum_l u_l s_l
template <typename T, bool C>
__global__ void k_mv_lowrank(int n, const int *slots, AcaDev S, const void *xt, void *yt) {
  using N = Num<T, C>;
  using V = typename N::V;
  const int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= n) return;
  const int b = slots[q];
  const int h = S.h[b], w = S.w[b], k = S.rank[b];
  const V *pool = static_cast<const V *>(S.pool);
  const V *x = static_cast<const V *>(xt) + S.c0[b];
  V *y = static_cast<V *>(yt) + S.r0[b];
  const long long *tl = S.terms + (long long)b * S.tmax;
  for (int l0 = 0; l0 < k; l0 += 32) {
    const int lk = min(32, k - l0);
    V mine = N::zero();
    for (int l = 0; l < lk; ++l) {
      const V *t = pool + tl[l0 + l];
      V acc = N::zero();
      for (int c = lane; c < w; c += 32) acc = N::fma_acc(acc, t[h + c], x[c]);
      acc = warp_sum_v<T, C>(acc);
      if (lane == l) mine = N::div(acc, t[h + w]);
    }
    for (int i0 = 0; i0 < h; i0 += 32) {  // warp-uniform trip count (shuffles below)
      const int i = i0 + lane;
      V acc = N::zero();
      for (int l = 0; l < lk; ++l) {
        V sl;
        if constexpr (C) {
          sl.re = __shfl_sync(0xffffffffu, mine.re, l);
          sl.im = __shfl_sync(0xffffffffu, mine.im, l);
        } else {
          sl = __shfl_sync(0xffffffffu, mine, l);
        }
        if (i < h) acc = N::fma_acc(acc, pool[tl[l0 + l] + i], sl);
      }
      if (i < h) atomic_add_v<V>(y + i, acc);
    }
  }
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
  const size_t vb = sizeof(typename Num<T, C>::V);
  HB_CUDA(cudaMemsetAsync(M.yt, 0, (size_t)M.n_rows * vb, st));
  k_mv_gather<T, C><<<(M.n_cols + 255) / 256, 256, 0, st>>>(M.n_cols, M.cperm, M.x, M.xt);
  for (int a = 0; a < 2; ++a) {
    const MatvecArgs::Dense &D = M.dense[a];
    if (D.n <= 0 || D.nrows <= 0) continue;
    const long long warps = D.nrows;
    k_mv_dense<T, C><<<(unsigned)((warps + 3) / 4), 128, 0, st>>>(
        D.n, D.r0, D.c0, D.h, D.w, D.off, D.rowbase, D.nrows, D.arena, M.xt, M.yt);
  }
  if (M.n_lowrank > 0)
    k_mv_lowrank<T, C><<<(unsigned)((M.n_lowrank + 3) / 4), 128, 0, st>>>(M.n_lowrank, M.lowrank,
                                                                         S, M.xt, M.yt);
  k_mv_scatter<T, C><<<(M.n_rows + 255) / 256, 256, 0, st>>>(M.n_rows, M.rperm, M.yt, M.y);
  HB_CUDA(cudaGetLastError());
  return HBEM_OK;
}

}  // namespace hb
