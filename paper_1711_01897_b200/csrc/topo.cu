// Mesh topology on the device (setup only): element -> touching elements
// (elements sharing at least one vertex index, classify_pair's
// quadrature.py:155-181 notion of adjacency), and the list of element pairs
// the singular table integrates.
//
//   corners (v, e) sorted by (v, e)  ->  vertex -> element CSR
//   per element: union of its three vertex lists, sorted, deduplicated
//   per element e: pairs (e, f) for f in nb(e) (symmetric operators: f >= e),
//                  with the table slot of (e, f) and of (f, e)
#include <cub/cub.cuh>

#include "hmat_common.cuh"

namespace hb {
namespace {

constexpr int kMaxNb = 1024;  // touching elements per element (setup scratch bound)

__global__ void k_corner_keys(const int4 *elem, int m, unsigned long long *keys) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  const int4 t = elem[e];
  keys[3ll * e + 0] = ((unsigned long long)(unsigned)t.x << 32) | (unsigned)e;
  keys[3ll * e + 1] = ((unsigned long long)(unsigned)t.y << 32) | (unsigned)e;
  keys[3ll * e + 2] = ((unsigned long long)(unsigned)t.z << 32) | (unsigned)e;
}

// vptr[v] = first sorted corner of vertex v (vertices without elements get
// the next start), vptr[nv] = 3m
__global__ void k_vertex_ptr(const unsigned long long *keys, long long nc, int nv, int *vptr) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q > nc) return;
  const int v = q < nc ? (int)(keys[q] >> 32) : nv;
  const int vp = q > 0 ? (int)(keys[q - 1] >> 32) : -1;
  for (int u = vp + 1; u <= v; ++u) vptr[u] = (int)q;
}

__device__ int gather_nb(const unsigned long long *keys, const int *vptr, int4 t, int *buf) {
  int n = 0;
  const int vs[3] = {t.x, t.y, t.z};
  for (int a = 0; a < 3; ++a)
    for (int q = vptr[vs[a]]; q < vptr[vs[a] + 1]; ++q) {
      const int f = (int)(keys[q] & 0xffffffffull);
      // insertion into the sorted unique buffer
      int j = n;
      bool dup = false;
      while (j > 0 && buf[j - 1] >= f) {
        if (buf[j - 1] == f) { dup = true; break; }
        --j;
      }
      if (dup) continue;
      if (n >= kMaxNb) return -1;
      for (int r = n; r > j; --r) buf[r] = buf[r - 1];
      buf[j] = f;
      ++n;
    }
  return n;
}

__global__ void k_nb_count(const int4 *elem, int m, const unsigned long long *keys,
                           const int *vptr, int *cnt, int *overflow) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  int buf[kMaxNb];
  const int n = gather_nb(keys, vptr, elem[e], buf);
  if (n < 0) {
    atomicExch(overflow, 1);
    cnt[e] = 0;
  } else {
    cnt[e] = n;
  }
}

__global__ void k_nb_fill(const int4 *elem, int m, const unsigned long long *keys,
                          const int *vptr, const int *ptr, int *idx) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  int buf[kMaxNb];
  const int n = gather_nb(keys, vptr, elem[e], buf);
  for (int j = 0; j < n; ++j) idx[ptr[e] + j] = buf[j];
}

__global__ void k_pair_count(int m, const int *ptr, const int *idx, int sym, int *cnt) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  int c = 0;
  for (int j = ptr[e]; j < ptr[e + 1]; ++j) c += (!sym || idx[j] >= e) ? 1 : 0;
  cnt[e] = c;
}

__global__ void k_pair_fill(int m, const int *ptr, const int *idx, int sym, const int *pptr,
                            int4 *pairs) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  int o = pptr[e];
  for (int j = ptr[e]; j < ptr[e + 1]; ++j) {
    const int f = idx[j];
    if (sym && f < e) continue;
    int back = -1;
    if (sym && f != e) {
      // slot of e in f's sorted list (binary search)
      int lo = ptr[f], hi = ptr[f + 1];
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (idx[mid] < e) lo = mid + 1;
        else hi = mid;
      }
      back = lo;
    }
    pairs[o++] = make_int4(e, f, j, back);
  }
}

// touching class of a pair = number of shared vertex indices (1 vertex, 2
// edge, 3 identical: classify_pair's kinds, quadrature.py:155-181)
__global__ void k_pair_kind(const int4 *elem, const int4 *pairs, long long n,
                            unsigned char *key, unsigned long long *cnt) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int ns = -1;
  if (q < n) {
    const int4 pr = pairs[q];
    const int4 a = elem[pr.x], b = elem[pr.y];
    const int ta[3] = {a.x, a.y, a.z};
    ns = 0;
#pragma unroll
    for (int i = 0; i < 3; ++i) ns += (ta[i] == b.x || ta[i] == b.y || ta[i] == b.z) ? 1 : 0;
    key[q] = (unsigned char)ns;
  }
  // warp-aggregated counts (one atomic per class per warp)
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const unsigned m = __ballot_sync(0xffffffffu, ns == c);
    if (lane == 0 && m) atomicAdd(cnt + c, (unsigned long long)__popc(m));
  }
}

template <typename X> int alloc(std::vector<void *> &allocs, X **p, size_t n) {
  void *q = nullptr;
  cudaError_t err = cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(X));
  if (err != cudaSuccess) {
    cudaGetLastError();
    return set_error(HBEM_ERR_CAPACITY, "device allocation of %zu bytes failed: %s",
                     n * sizeof(X), cudaGetErrorString(err));
  }
  allocs.push_back(q);
  *p = static_cast<X *>(q);
  return HBEM_OK;
}

// exclusive scan of n counts into ptr[0..n] (ptr[n] = total), returns total
int scan_counts(const int *cnt, int *ptr, int n, cudaStream_t st, long long *total) {
  size_t tb = 0;
  HB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, ptr, n + 1, st));
  void *tmp = nullptr;
  HB_CUDA(cudaMalloc(&tmp, std::max<size_t>(tb, 1)));
  cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, ptr, n + 1, st);
  cudaFree(tmp);
  HB_CUDA(e);
  int t = 0;
  HB_CUDA(cudaMemcpyAsync(&t, ptr + n, sizeof(int), cudaMemcpyDeviceToHost, st));
  HB_CUDA(cudaStreamSynchronize(st));
  *total = t;
  return HBEM_OK;
}

// one thread per near-field leaf row: mark the neighbour slots (e, f) whose
// trial element f lies in the leaf's column cluster
__global__ void k_mark_rows(const int *nb_ptr, const int *nb_idx, const int *rperm,
                            const int *cinv, const long long *rowbase, int nd, long long nrows,
                            const int *r0, const int *c0, const int *w, unsigned char *mark) {
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= nrows) return;
  int lo = 0, hi = nd;  // leaf s with rowbase[s] <= g < rowbase[s + 1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (rowbase[mid] <= g) lo = mid;
    else hi = mid;
  }
  const int s = lo;
  const int e = rperm[r0[s] + (int)(g - rowbase[s])];
  const int cb = c0[s], ce = c0[s] + w[s];
  for (int j = nb_ptr[e]; j < nb_ptr[e + 1]; ++j) {
    const int tp = cinv[nb_idx[j]];
    if (tp >= cb && tp < ce) mark[j] = 1;
  }
}

__global__ void k_pair_flags(const int4 *pairs, long long np, const unsigned char *mark,
                             unsigned char *flag) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= np) return;
  const int4 p = pairs[q];
  flag[q] = mark[p.z] || (p.w >= 0 && mark[p.w]);
}

}  // namespace

int restrict_sing_pairs(SingTable &tab, const int *rperm, const int *cinv,
                        const long long *rowbase, int nd, long long nrows, const int *r0,
                        const int *c0, const int *w, std::vector<void *> &allocs,
                        cudaStream_t st) {
  if (tab.n_pairs <= 0) return HBEM_OK;
  unsigned char *mark = nullptr, *flag = nullptr;
  int *cnt = nullptr;
  HB_CUDA(cudaMalloc(&mark, (size_t)std::max<long long>(tab.nnz, 1)));
  HB_CUDA(cudaMalloc(&flag, (size_t)tab.n_pairs));
  HB_CUDA(cudaMalloc(&cnt, 4));
  HB_CUDA(cudaMemsetAsync(mark, 0, (size_t)std::max<long long>(tab.nnz, 1), st));
  if (nrows > 0)
    k_mark_rows<<<(unsigned)((nrows + 255) / 256), 256, 0, st>>>(
        tab.nb_ptr, tab.nb_idx, rperm, cinv, rowbase, nd, nrows, r0, c0, w, mark);
  k_pair_flags<<<(unsigned)((tab.n_pairs + 255) / 256), 256, 0, st>>>(tab.pairs, tab.n_pairs,
                                                                      mark, flag);
  int4 *kept = nullptr;
  HB_CHECK(alloc(allocs, &kept, (size_t)tab.n_pairs));
  size_t tb = 0;
  HB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, tab.pairs, flag, kept, cnt, tab.n_pairs, st));
  void *tmp = nullptr;
  HB_CUDA(cudaMalloc(&tmp, std::max<size_t>(tb, 1)));
  cudaError_t e = cub::DeviceSelect::Flagged(tmp, tb, tab.pairs, flag, kept, cnt, tab.n_pairs, st);
  int h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, cnt, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(tmp);
  cudaFree(mark);
  cudaFree(flag);
  cudaFree(cnt);
  HB_CUDA(e);
  tab.pairs = kept;
  tab.n_pairs = h;
  return HBEM_OK;
}

int sort_sing_pairs(SingTable &tab, const int4 *d_elem, std::vector<void *> &allocs,
                    cudaStream_t st) {
  for (long long &c : tab.kind_n) c = 0;
  if (tab.n_pairs <= 0) return HBEM_OK;
  const long long n = tab.n_pairs;
  unsigned char *key = nullptr, *key2 = nullptr;
  unsigned long long *cnt = nullptr;
  HB_CUDA(cudaMalloc(&key, (size_t)n));
  HB_CUDA(cudaMalloc(&key2, (size_t)n));
  HB_CUDA(cudaMalloc(&cnt, 4 * sizeof(unsigned long long)));
  auto cleanup = [&]() { cudaFree(key); cudaFree(key2); cudaFree(cnt); };
  HB_CUDA(cudaMemsetAsync(cnt, 0, 4 * sizeof(unsigned long long), st));
  k_pair_kind<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_elem, tab.pairs, n, key, cnt);
  int4 *sorted = nullptr;
  HB_CHECK(alloc(allocs, &sorted, (size_t)n));
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, tab.pairs, sorted, n, 0, 2, st);
  void *tmp = nullptr;
  HB_CUDA(cudaMalloc(&tmp, std::max<size_t>(tb, 1)));
  cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, tb, key, key2, tab.pairs, sorted, n, 0, 2, st);
  unsigned long long h[4] = {0, 0, 0, 0};
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(tmp);
  cleanup();
  HB_CUDA(e);
  if (h[0] != 0) return set_error(HBEM_ERR_KERNEL, "singular table holds a non-touching pair");
  for (int k = 0; k < 4; ++k) tab.kind_n[k] = (long long)h[k];
  tab.pairs = sorted;
  return HBEM_OK;
}

int build_sing_table(const int4 *d_elem, int m, int nv, bool symmetric, SingTable &out,
                     std::vector<void *> &allocs, cudaStream_t st) {
  const long long nc = 3ll * m;
  unsigned long long *keys = nullptr, *keys2 = nullptr;
  int *vptr = nullptr, *cnt = nullptr, *ovf = nullptr;
  HB_CUDA(cudaMalloc(&keys, nc * 8));
  HB_CUDA(cudaMalloc(&keys2, nc * 8));
  HB_CUDA(cudaMalloc(&vptr, (size_t)(nv + 1) * 4));
  HB_CUDA(cudaMalloc(&cnt, (size_t)(m + 1) * 4));
  HB_CUDA(cudaMalloc(&ovf, 4));
  auto cleanup = [&]() {
    cudaFree(keys); cudaFree(keys2); cudaFree(vptr); cudaFree(cnt); cudaFree(ovf);
  };
  const unsigned g = (unsigned)((m + 127) / 128);
  k_corner_keys<<<g, 128, 0, st>>>(d_elem, m, keys);
  {
    size_t tb = 0;
    int bits = 64;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, keys2, (int)nc, 0, bits, st);
    void *tmp = nullptr;
    HB_CUDA(cudaMalloc(&tmp, std::max<size_t>(tb, 1)));
    cudaError_t e = cub::DeviceRadixSort::SortKeys(tmp, tb, keys, keys2, (int)nc, 0, bits, st);
    cudaFree(tmp);
    if (e != cudaSuccess) { cleanup(); HB_CUDA(e); }
  }
  k_vertex_ptr<<<(unsigned)((nc + 1 + 255) / 256), 256, 0, st>>>(keys2, nc, nv, vptr);
  HB_CUDA(cudaMemsetAsync(ovf, 0, 4, st));
  HB_CUDA(cudaMemsetAsync(cnt + m, 0, 4, st));
  k_nb_count<<<g, 128, 0, st>>>(d_elem, m, keys2, vptr, cnt, ovf);
  int h_ovf = 0;
  HB_CUDA(cudaMemcpyAsync(&h_ovf, ovf, 4, cudaMemcpyDeviceToHost, st));
  HB_CHECK(alloc(allocs, &out.nb_ptr, (size_t)m + 1));
  long long nnz = 0;
  HB_CHECK(scan_counts(cnt, out.nb_ptr, m, st, &nnz));
  if (h_ovf) {
    cleanup();
    return set_error(HBEM_ERR_CAPACITY, "an element touches more than %d elements", kMaxNb);
  }
  out.nnz = nnz;
  HB_CHECK(alloc(allocs, &out.nb_idx, (size_t)nnz));
  k_nb_fill<<<g, 128, 0, st>>>(d_elem, m, keys2, vptr, out.nb_ptr, out.nb_idx);
  k_pair_count<<<g, 128, 0, st>>>(m, out.nb_ptr, out.nb_idx, symmetric ? 1 : 0, cnt);
  int *pptr = nullptr;
  HB_CHECK(alloc(allocs, &pptr, (size_t)m + 1));
  long long np = 0;
  HB_CHECK(scan_counts(cnt, pptr, m, st, &np));
  out.n_pairs = np;
  HB_CHECK(alloc(allocs, &out.pairs, (size_t)np));
  k_pair_fill<<<g, 128, 0, st>>>(m, out.nb_ptr, out.nb_idx, symmetric ? 1 : 0, pptr, out.pairs);
  HB_CUDA(cudaGetLastError());
  HB_CUDA(cudaStreamSynchronize(st));
  cleanup();
  return HBEM_OK;
}

}  // namespace hb
