// Context staging (init_device, backend.py:77-122) and the batched pair
// integrators: K1 regular (integrate_batch, backend.py:200-255) and K2
// Sauter-Schwab (local_matrix on touching pairs, kernels.py:330-347).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "hbem_internal.h"

namespace hb {

static thread_local std::string g_err;

int set_error(int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
void clear_error() { g_err.clear(); }

// ---------------------------------------------------------------------------
// geometry staging
// ---------------------------------------------------------------------------

// precompute_geometry (mesh.py:344-359) + element_curls (spaces.py:138-143)
// in float64 with the numpy operation order (no FMA contraction):
// cross = a1*b2 - a2*b1 ...; |J| = sqrt((c0^2 + c1^2) + c2^2); n = c/|J|;
// q = (v0 + xi*e1) + eta*e2; curl_l = (v_{l+1} - v_{l+2}) / |J|.
__global__ void k_geometry(const double *vtx, const int4 *elem, int64_t m, int nq,
                           const double *rp /* nq x 2 */, double *q64 /* m x nq x 3 */,
                           double *nj64, double *curl64) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  const int4 t = elem[e];
  double v0[3], v1[3], v2[3];
  for (int c = 0; c < 3; ++c) {
    v0[c] = vtx[3 * (int64_t)t.x + c];
    v1[c] = vtx[3 * (int64_t)t.y + c];
    v2[c] = vtx[3 * (int64_t)t.z + c];
  }
  double e1[3], e2[3];
  for (int c = 0; c < 3; ++c) {
    e1[c] = __dsub_rn(v1[c], v0[c]);
    e2[c] = __dsub_rn(v2[c], v0[c]);
  }
  double cr[3];
  cr[0] = __dsub_rn(__dmul_rn(e1[1], e2[2]), __dmul_rn(e1[2], e2[1]));
  cr[1] = __dsub_rn(__dmul_rn(e1[2], e2[0]), __dmul_rn(e1[0], e2[2]));
  cr[2] = __dsub_rn(__dmul_rn(e1[0], e2[1]), __dmul_rn(e1[1], e2[0]));
  const double jac = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(cr[0], cr[0]),
                                                    __dmul_rn(cr[1], cr[1])),
                                          __dmul_rn(cr[2], cr[2])));
  nj64[4 * e + 0] = __ddiv_rn(cr[0], jac);
  nj64[4 * e + 1] = __ddiv_rn(cr[1], jac);
  nj64[4 * e + 2] = __ddiv_rn(cr[2], jac);
  nj64[4 * e + 3] = jac;
  for (int p = 0; p < nq; ++p) {
    const double xi = rp[2 * p], eta = rp[2 * p + 1];
    for (int c = 0; c < 3; ++c)
      q64[(e * nq + p) * 3 + c] =
          __dadd_rn(__dadd_rn(v0[c], __dmul_rn(xi, e1[c])), __dmul_rn(eta, e2[c]));
  }
  if (curl64) {
    const double *vv[3] = {v0, v1, v2};
    for (int l = 0; l < 3; ++l)
      for (int c = 0; c < 3; ++c)
        curl64[9 * e + 3 * l + c] = __ddiv_rn(__dsub_rn(vv[(l + 1) % 3][c], vv[(l + 2) % 3][c]), jac);
  }
}

// Pack float64 caches into the working-precision device layout (the
// astype(real_dtype) of init_device, backend.py:104-121).  Rules with fewer
// than 6 points are padded with zero-weight copies of point 0.
template <typename T>
__global__ void k_pack(const double *q64, const double *nj64, const double *curl64, int64_t m,
                       int nq, T *q, T *nj, T *curl) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  constexpr int QS = QStride<T>::value;
  for (int p = 0; p < 6; ++p) {
    const int src = p < nq ? p : 0;
    for (int c = 0; c < 3; ++c) q[e * QS + 3 * p + c] = (T)q64[(e * nq + src) * 3 + c];
  }
  for (int i = 18; i < QS; ++i) q[e * QS + i] = T(0);
  for (int c = 0; c < 4; ++c) nj[4 * e + c] = (T)nj64[4 * e + c];
  if (curl)
    for (int c = 0; c < 9; ++c) curl[9 * e + c] = (T)curl64[9 * e + c];
}

__global__ void k_elem(const int64_t *el, int64_t m, int4 *out) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  out[e] = make_int4((int)el[3 * e], (int)el[3 * e + 1], (int)el[3 * e + 2], 0);
}

// ---------------------------------------------------------------------------
// K1: one thread per pair, 6x6 regular rule.
// mode 0: trust the caller (device API); 1: validate (range + disjoint,
// reference contract), skipping bad pairs; 2: classify, appending touching
// pairs to sing_list for K2.
// flags[0] min index, [1] max index, [2] first touching pair, [3] #touching
// ---------------------------------------------------------------------------
template <typename T, int OP, bool HELM, int NT, int NS>
__global__ void __launch_bounds__(128)
    k_regular(Geo<T> g, RuleTab<T> R, const int4 *elem, const int64_t *pairs, int64_t p, T *re,
              T *im, int mode, int *sing_list, unsigned long long *flags) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool active = i < p;
  int64_t a = 0, b = 0;
  if (active) {
    const longlong2 ab = *reinterpret_cast<const longlong2 *>(pairs + 2 * i);
    a = ab.x;
    b = ab.y;
  }
  if (mode != 0) {
    long long lo = active ? (long long)min(a, b) : LLONG_MAX;
    long long hi = active ? (long long)max(a, b) : LLONG_MIN;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(reinterpret_cast<long long *>(flags + 0), lo);
      atomicMax(reinterpret_cast<long long *>(flags + 1), hi);
    }
    if (active && (a < 0 || b < 0 || a >= g.m || b >= g.m)) active = false;
    if (active && touching(elem[a], elem[b])) {
      if (mode == 1) {
        atomicMin(reinterpret_cast<long long *>(flags + 2), (long long)i);
      } else {
        const unsigned long long slot = atomicAdd(flags + 3, 1ull);
        sing_list[slot] = (int)i;
      }
      active = false;
    }
  }
  if (!active) return;
  T x[18], y[18], na[4], nb[4];
  load_q<T>(g.q, a, x);
  load_q<T>(g.q, b, y);
  load_nj<T>(g.nj, a, na);
  load_nj<T>(g.nj, b, nb);
  T ore[NT][NS], oim[NT][NS];
  const T *ca = nullptr, *cb = nullptr;
  if (OP == HBEM_HYPS) {
    ca = g.curl + 9 * a;
    cb = g.curl + 9 * b;
  }
  regular_pair<T, OP, HELM, NT, NS>(R, x, y, na, nb, ca, cb, ore, oim);
  T *o = re + i * (NT * NS);
#pragma unroll
  for (int u = 0; u < NT; ++u)
#pragma unroll
    for (int v = 0; v < NS; ++v) o[u * NS + v] = ore[u][v];
  if (HELM) {
    T *oi = im + i * (NT * NS);
#pragma unroll
    for (int u = 0; u < NT; ++u)
#pragma unroll
      for (int v = 0; v < NS; ++v) oi[u * NS + v] = oim[u][v];
  }
}

// K2: one warp per touching pair from sing_list; float64, cast on store.
template <typename T, int OP, bool HELM, int NT, int NS>
__global__ void __launch_bounds__(128)
    k_singular(Geo64 G, const int64_t *pairs, const int *sing_list,
               const unsigned long long *flags, T *re, T *im) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n = (int64_t)flags[3];
  for (int64_t w = warp; w < n; w += nw) {
    const int64_t i = sing_list[w];
    const int64_t a = pairs[2 * i], b = pairs[2 * i + 1];
    double ore[NT][NS], oim[NT][NS];
    singular_local<OP, HELM, NT, NS>(G, a, b, ore, oim);
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < NT; ++u)
#pragma unroll
        for (int v = 0; v < NS; ++v) {
          re[i * NT * NS + u * NS + v] = (T)ore[u][v];
          if (HELM) im[i * NT * NS + u * NS + v] = (T)oim[u][v];
        }
    }
  }
}

__global__ void k_init_flags(unsigned long long *f) {
  f[0] = (unsigned long long)LLONG_MAX;
  f[1] = (unsigned long long)LLONG_MIN;
  f[2] = (unsigned long long)LLONG_MAX;
  f[3] = 0ull;
}

static int sm_count(int dev) {
  static int cached[64] = {0};
  if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cached[dev] = n;
  return n;
}

template <typename T>
static int launch_pairs(hbem_ctx *ctx, const int64_t *d_pairs, int64_t p, T *re, T *im, int mode,
                        int *sing_list, unsigned long long *flags, cudaStream_t st) {
  return dispatch_op(ctx->op, ctx->helm, ctx->nt, ctx->ns, [&](auto OPc, auto Hc, auto NTc,
                                                               auto NSc) -> int {
    constexpr int OP = decltype(OPc)::value;
    constexpr bool H = decltype(Hc)::value != 0;
    constexpr int NT = decltype(NTc)::value, NS = decltype(NSc)::value;
    if (p > 0) {
      const int bs = 128;
      const int64_t grid = (p + bs - 1) / bs;
      k_regular<T, OP, H, NT, NS><<<(unsigned)grid, bs, 0, st>>>(
          ctx->geo<T>(), ctx->rule<T>(), ctx->elem, d_pairs, p, re, im, mode, sing_list, flags);
      HB_CUDA(cudaGetLastError());
      if (mode == 2) {
        const int64_t need = (p + 3) / 4;
        const int64_t cap = (int64_t)sm_count(ctx->device) * 16;
        const unsigned g2 = (unsigned)std::max<int64_t>(1, std::min(need, cap));
        k_singular<T, OP, H, NT, NS><<<g2, 128, 0, st>>>(ctx->geo64(), d_pairs, sing_list, flags,
                                                         re, im);
        HB_CUDA(cudaGetLastError());
      }
    }
    return HBEM_OK;
  });
}

int integrate_pairs_device(hbem_ctx *ctx, const int64_t *d_pairs, int64_t p, void *d_re,
                           void *d_im, int mode, int *d_sing_list, unsigned long long *d_flags,
                           cudaStream_t st) {
  if (mode != 0) {
    k_init_flags<<<1, 1, 0, st>>>(d_flags);
    HB_CUDA(cudaGetLastError());
  }
  if (ctx->precision == HBEM_DOUBLE)
    return launch_pairs<double>(ctx, d_pairs, p, (double *)d_re, (double *)d_im, mode,
                                d_sing_list, d_flags, st);
  return launch_pairs<float>(ctx, d_pairs, p, (float *)d_re, (float *)d_im, mode, d_sing_list,
                             d_flags, st);
}

// host-buffer integrate with validation (mode 1) or classification (mode 2)
static int integrate_host(hbem_ctx *ctx, const int64_t *pairs, int64_t p, void *re, void *im,
                          int mode, int64_t *n_singular) {
  if (!ctx) return set_error(HBEM_ERR_ARG, "null context");
  if (p < 0) return set_error(HBEM_ERR_ARG, "negative pair count");
  if (ctx->helm && p > 0 && !im)
    return set_error(HBEM_ERR_ARG, "Helmholtz result needs an imaginary plane");
  if (p == 0) {
    if (n_singular) *n_singular = 0;
    return HBEM_OK;
  }
  HB_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = cudaStreamPerThread;
  const size_t out_bytes = (size_t)p * ctx->nt * ctx->ns * ctx->real_bytes();
  int64_t *d_pairs = nullptr;
  void *d_re = nullptr, *d_im = nullptr;
  int *d_list = nullptr;
  unsigned long long *d_flags = nullptr;
  HB_CUDA(cudaMallocAsync((void **)&d_pairs, (size_t)p * 16, st));
  HB_CUDA(cudaMallocAsync(&d_re, out_bytes, st));
  if (ctx->helm) HB_CUDA(cudaMallocAsync(&d_im, out_bytes, st));
  HB_CUDA(cudaMallocAsync((void **)&d_flags, 64, st));
  if (mode == 2) HB_CUDA(cudaMallocAsync((void **)&d_list, (size_t)p * sizeof(int), st));
  HB_CUDA(cudaMemcpyAsync(d_pairs, pairs, (size_t)p * 16, cudaMemcpyHostToDevice, st));
  int rc = integrate_pairs_device(ctx, d_pairs, p, d_re, d_im, mode, d_list, d_flags, st);
  unsigned long long flags[4] = {0, 0, 0, 0};
  if (rc == HBEM_OK) {
    cudaMemcpyAsync(flags, d_flags, sizeof(flags), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(re, d_re, out_bytes, cudaMemcpyDeviceToHost, st);
    if (ctx->helm) cudaMemcpyAsync(im, d_im, out_bytes, cudaMemcpyDeviceToHost, st);
  }
  cudaFreeAsync(d_pairs, st);
  cudaFreeAsync(d_re, st);
  if (d_im) cudaFreeAsync(d_im, st);
  cudaFreeAsync(d_flags, st);
  if (d_list) cudaFreeAsync(d_list, st);
  HB_CUDA(cudaStreamSynchronize(st));
  if (rc != HBEM_OK) return rc;
  const long long lo = (long long)flags[0], hi = (long long)flags[1];
  if (lo < 0 || hi >= ctx->m)
    return set_error(HBEM_ERR_CONTRACT, "pair indices must lie in [0, %lld), found [%lld, %lld]",
                     (long long)ctx->m, lo, hi);
  if (mode == 1 && (long long)flags[2] != LLONG_MAX) {
    const long long i = (long long)flags[2];
    return set_error(HBEM_ERR_CONTRACT,
                     "request pair %lld = (%lld, %lld) is not disjoint; touching pairs must take "
                     "the singular path",
                     i, (long long)pairs[2 * i], (long long)pairs[2 * i + 1]);
  }
  if (n_singular) *n_singular = (int64_t)flags[3];
  return HBEM_OK;
}

template <typename T> static void fill_rule(RuleTab<T> &R, const hbem_ctx_desc *d,
                                            const std::vector<double> &ta,
                                            const std::vector<double> &tb, int nt, int ns) {
  std::memset(&R, 0, sizeof(R));
  for (int p = 0; p < 6; ++p) {
    const double w = p < d->n_q ? d->rule_weights[p] : 0.0;
    R.w[p] = (T)w;
    for (int i = 0; i < 3; ++i) {
      R.wa[i][p] = i < nt ? (T)(w * ta[i * 6 + p]) : T(0);
      R.wb[i][p] = i < ns ? (T)(w * tb[i * 6 + p]) : T(0);
    }
  }
  R.k = (T)d->wavenumber;
  R.k2 = (T)(d->wavenumber * d->wavenumber);
  for (int o = 0; o < 6; ++o)
    for (int i = 0; i < 6; ++i) R.w2[o][i] = R.wa[0][o] * R.wb[0][i];
  R.k38 = (T)(0.375 * d->wavenumber);
}

}  // namespace hb

using namespace hb;

extern "C" {

int hbem_abi_version(void) { return HBEM_ABI_VERSION; }
const char *hbem_last_error(void) { return g_err.c_str(); }

int hbem_device_count(int32_t *count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  *count = n;
  return HBEM_OK;
}

int hbem_ctx_create(const hbem_ctx_desc *d, hbem_ctx **out) {
  clear_error();
  if (!d || !out) return set_error(HBEM_ERR_ARG, "null argument");
  *out = nullptr;
  if (d->n_q > HBEM_MAX_WEIGHTS)
    return set_error(HBEM_ERR_CAPACITY,
                     "quadrature rule has %d weights, device capacity is %d", d->n_q,
                     HBEM_MAX_WEIGHTS);
  if (d->n_q < 1) return set_error(HBEM_ERR_CAPACITY, "quadrature rule has no points");
  if (d->op < 0 || d->op > 3) return set_error(HBEM_ERR_KERNEL, "unknown operator %d", d->op);
  if (d->equation != HBEM_LAPLACE && d->equation != HBEM_HELMHOLTZ)
    return set_error(HBEM_ERR_KERNEL, "unknown equation %d", d->equation);
  if (d->op == HBEM_HYPS && (d->test_family == HBEM_P0 || d->trial_family == HBEM_P0))
    return set_error(HBEM_ERR_KERNEL, "hyps requires linear test and trial spaces");
  if (d->n_elements <= 0 || d->n_vertices <= 0)
    return set_error(HBEM_ERR_ARG, "empty mesh");
  if (d->n_elements >= (int64_t)1 << 31 || d->n_vertices >= (int64_t)1 << 31)
    return set_error(HBEM_ERR_CAPACITY, "mesh exceeds 2^31 elements/vertices");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return set_error(HBEM_ERR_CUDA, "no CUDA device available");
  }
  if (d->device < 0 || d->device >= ndev)
    return set_error(HBEM_ERR_ARG, "device %d out of range (%d devices)", d->device, ndev);
  HB_CUDA(cudaSetDevice(d->device));

  hbem_ctx *c = new hbem_ctx();
  auto fail_early = [&](int rc) {
    delete c;
    return rc;
  };
  c->device = d->device;
  c->equation = d->equation;
  c->op = d->op;
  c->precision = d->precision;
  c->wavenumber = d->wavenumber;
  c->helm = d->equation == HBEM_HELMHOLTZ;
  c->test_family = d->test_family;
  c->trial_family = d->trial_family;
  c->nt = d->test_family == HBEM_P0 ? 1 : 3;
  c->ns = d->trial_family == HBEM_P0 ? 1 : 3;
  c->m = d->n_elements;
  c->nv = d->n_vertices;
  const int64_t m = c->m;
  const int nq = d->n_q;

  // basis tables at the rule points (spaces.py:112-125)
  std::vector<double> ta(18, 0.0), tb(18, 0.0);
  if (!d->rule_weights) return fail_early(set_error(HBEM_ERR_ARG, "missing rule weights"));
  if ((!d->test_values || !d->trial_values) && !d->rule_points)
    return fail_early(set_error(HBEM_ERR_ARG, "need basis tables or rule points"));
  for (int p = 0; p < nq; ++p) {
    double bary[3] = {1.0, 0.0, 0.0};
    if (d->rule_points) {
      const double xi = d->rule_points[2 * p], eta = d->rule_points[2 * p + 1];
      bary[0] = 1.0 - xi - eta;
      bary[1] = xi;
      bary[2] = eta;
    }
    for (int i = 0; i < 3; ++i) {
      if (i < c->nt)
        ta[i * 6 + p] = d->test_values ? d->test_values[i * nq + p] : (c->nt == 1 ? 1.0 : bary[i]);
      if (i < c->ns)
        tb[i * 6 + p] = d->trial_values ? d->trial_values[i * nq + p]
                                         : (c->ns == 1 ? 1.0 : bary[i]);
    }
  }
  fill_rule<double>(c->rd, d, ta, tb, c->nt, c->ns);
  fill_rule<float>(c->rf, d, ta, tb, c->nt, c->ns);

  auto fail = [&](int rc) {
    hbem_ctx_destroy(c);
    return rc;
  };
#define HB_CUDA_C(call)                                                                     \
  do {                                                                                      \
    cudaError_t _e = (call);                                                                \
    if (_e != cudaSuccess)                                                                  \
      return fail(set_error(HBEM_ERR_CUDA, "CUDA error %s at %s:%d", cudaGetErrorName(_e),  \
                            __FILE__, __LINE__));                                           \
  } while (0)

  const bool hyps = d->op == HBEM_HYPS;
  const size_t rb = c->real_bytes();
  const int QS = c->precision == HBEM_DOUBLE ? 18 : 20;
  HB_CUDA_C(cudaMalloc(&c->vtx, (size_t)c->nv * 3 * 8));
  HB_CUDA_C(cudaMalloc(&c->elem, (size_t)m * sizeof(int4)));
  HB_CUDA_C(cudaMalloc(&c->q, (size_t)m * QS * rb));
  HB_CUDA_C(cudaMalloc(&c->nj, (size_t)m * 4 * rb));
  if (hyps) HB_CUDA_C(cudaMalloc(&c->curl, (size_t)m * 9 * rb));
  if (c->precision == HBEM_DOUBLE) {
    c->nj64 = (double *)c->nj;
    c->curl64 = (double *)c->curl;
  } else {
    HB_CUDA_C(cudaMalloc(&c->nj64, (size_t)m * 4 * 8));
    if (hyps) HB_CUDA_C(cudaMalloc(&c->curl64, (size_t)m * 9 * 8));
  }
  HB_CUDA_C(cudaMemcpy(c->vtx, d->vertices, (size_t)c->nv * 3 * 8, cudaMemcpyHostToDevice));
  {
    int64_t *del = nullptr;
    HB_CUDA_C(cudaMalloc(&del, (size_t)m * 3 * 8));
    HB_CUDA_C(cudaMemcpy(del, d->elements, (size_t)m * 3 * 8, cudaMemcpyHostToDevice));
    k_elem<<<(unsigned)((m + 255) / 256), 256>>>(del, m, c->elem);
    HB_CUDA_C(cudaGetLastError());
    HB_CUDA_C(cudaDeviceSynchronize());
    cudaFree(del);
  }
  // float64 staging of the geometry caches
  double *q64 = nullptr, *nj64 = nullptr, *curl64 = nullptr, *rp = nullptr;
  HB_CUDA_C(cudaMalloc(&q64, (size_t)m * nq * 3 * 8));
  nj64 = c->precision == HBEM_DOUBLE ? nullptr : c->nj64;
  double *nj_stage = nullptr;
  HB_CUDA_C(cudaMalloc(&nj_stage, (size_t)m * 4 * 8));
  if (hyps) HB_CUDA_C(cudaMalloc(&curl64, (size_t)m * 9 * 8));
  (void)nj64;
  if (d->qpoints && d->normals && d->jacobians) {
    HB_CUDA_C(cudaMemcpy(q64, d->qpoints, (size_t)m * nq * 3 * 8, cudaMemcpyHostToDevice));
    std::vector<double> njh((size_t)m * 4);
    for (int64_t e = 0; e < m; ++e) {
      njh[4 * e + 0] = d->normals[3 * e + 0];
      njh[4 * e + 1] = d->normals[3 * e + 1];
      njh[4 * e + 2] = d->normals[3 * e + 2];
      njh[4 * e + 3] = d->jacobians[e];
    }
    HB_CUDA_C(cudaMemcpy(nj_stage, njh.data(), (size_t)m * 4 * 8, cudaMemcpyHostToDevice));
    if (hyps) {
      if (d->curls) {
        HB_CUDA_C(cudaMemcpy(curl64, d->curls, (size_t)m * 9 * 8, cudaMemcpyHostToDevice));
      } else {
        if (!d->rule_points) return fail(set_error(HBEM_ERR_ARG, "curls need rule points"));
        double *scratch_q = nullptr, *scratch_nj = nullptr;
        HB_CUDA_C(cudaMalloc(&scratch_q, (size_t)m * nq * 3 * 8));
        HB_CUDA_C(cudaMalloc(&scratch_nj, (size_t)m * 4 * 8));
        HB_CUDA_C(cudaMalloc(&rp, (size_t)nq * 2 * 8));
        HB_CUDA_C(cudaMemcpy(rp, d->rule_points, (size_t)nq * 2 * 8, cudaMemcpyHostToDevice));
        k_geometry<<<(unsigned)((m + 127) / 128), 128>>>(c->vtx, c->elem, m, nq, rp, scratch_q,
                                                          scratch_nj, curl64);
        HB_CUDA_C(cudaGetLastError());
        HB_CUDA_C(cudaDeviceSynchronize());
        cudaFree(scratch_q);
        cudaFree(scratch_nj);
      }
    }
  } else {
    if (!d->rule_points) return fail(set_error(HBEM_ERR_ARG, "device geometry needs rule points"));
    HB_CUDA_C(cudaMalloc(&rp, (size_t)nq * 2 * 8));
    HB_CUDA_C(cudaMemcpy(rp, d->rule_points, (size_t)nq * 2 * 8, cudaMemcpyHostToDevice));
    k_geometry<<<(unsigned)((m + 127) / 128), 128>>>(c->vtx, c->elem, m, nq, rp, q64, nj_stage,
                                                      curl64);
    HB_CUDA_C(cudaGetLastError());
  }
  if (c->precision == HBEM_DOUBLE) {
    k_pack<double><<<(unsigned)((m + 127) / 128), 128>>>(q64, nj_stage, curl64, m, nq,
                                                          (double *)c->q, (double *)c->nj,
                                                          (double *)c->curl);
  } else {
    k_pack<float><<<(unsigned)((m + 127) / 128), 128>>>(q64, nj_stage, curl64, m, nq,
                                                         (float *)c->q, (float *)c->nj,
                                                         (float *)c->curl);
    HB_CUDA_C(cudaMemcpy(c->nj64, nj_stage, (size_t)m * 4 * 8, cudaMemcpyDeviceToDevice));
    if (hyps)
      HB_CUDA_C(cudaMemcpy(c->curl64, curl64, (size_t)m * 9 * 8, cudaMemcpyDeviceToDevice));
  }
  HB_CUDA_C(cudaGetLastError());
  HB_CUDA_C(cudaDeviceSynchronize());
  cudaFree(q64);
  cudaFree(nj_stage);
  if (curl64) cudaFree(curl64);
  if (rp) cudaFree(rp);

  // singular rules
  for (int k = 0; k < 3; ++k) {
    const int64_t n = d->sing_n[k];
    c->sn[k] = (int)n;
    if (n <= 0) continue;
    if (!d->sing_points[k] || !d->sing_weights[k]) {
      return fail(set_error(HBEM_ERR_ARG, "missing singular rule %d", k));
    }
    HB_CUDA_C(cudaMalloc(&c->sp[k], (size_t)n * 4 * 8));
    HB_CUDA_C(cudaMalloc(&c->sw[k], (size_t)n * 8));
    HB_CUDA_C(cudaMemcpy(c->sp[k], d->sing_points[k], (size_t)n * 32, cudaMemcpyHostToDevice));
    HB_CUDA_C(cudaMemcpy(c->sw[k], d->sing_weights[k], (size_t)n * 8, cudaMemcpyHostToDevice));
  }
#undef HB_CUDA_C
  *out = c;
  return HBEM_OK;
}

int hbem_ctx_destroy(hbem_ctx *c) {
  if (!c) return HBEM_OK;
  cudaSetDevice(c->device);
  cudaFree(c->q);
  cudaFree(c->nj);
  cudaFree(c->curl);
  if (c->precision != HBEM_DOUBLE) {
    cudaFree(c->nj64);
    cudaFree(c->curl64);
  }
  cudaFree(c->vtx);
  cudaFree(c->elem);
  for (int k = 0; k < 3; ++k) {
    cudaFree(c->sp[k]);
    cudaFree(c->sw[k]);
  }
  delete c;
  return HBEM_OK;
}

int hbem_ctx_info(const hbem_ctx *c, int32_t *nt, int32_t *ns, int32_t *is_complex,
                  int32_t *real_bytes) {
  if (!c) return set_error(HBEM_ERR_ARG, "null context");
  if (nt) *nt = c->nt;
  if (ns) *ns = c->ns;
  if (is_complex) *is_complex = c->helm ? 1 : 0;
  if (real_bytes) *real_bytes = c->real_bytes();
  return HBEM_OK;
}

int hbem_ctx_geometry(const hbem_ctx *c, double *qpoints, double *normals, double *jacobians) {
  if (!c) return set_error(HBEM_ERR_ARG, "null context");
  HB_CUDA(cudaSetDevice(c->device));
  const int64_t m = c->m;
  std::vector<double> nj((size_t)m * 4);
  HB_CUDA(cudaMemcpy(nj.data(), c->nj64, (size_t)m * 32, cudaMemcpyDeviceToHost));
  for (int64_t e = 0; e < m; ++e) {
    if (normals)
      for (int k = 0; k < 3; ++k) normals[3 * e + k] = nj[4 * e + k];
    if (jacobians) jacobians[e] = nj[4 * e + 3];
  }
  if (qpoints) {
    const int QS = c->precision == HBEM_DOUBLE ? 18 : 20;
    if (c->precision == HBEM_DOUBLE) {
      std::vector<double> q((size_t)m * QS);
      HB_CUDA(cudaMemcpy(q.data(), c->q, q.size() * 8, cudaMemcpyDeviceToHost));
      for (int64_t e = 0; e < m; ++e)
        for (int k = 0; k < 18; ++k) qpoints[18 * e + k] = q[QS * e + k];
    } else {
      std::vector<float> q((size_t)m * QS);
      HB_CUDA(cudaMemcpy(q.data(), c->q, q.size() * 4, cudaMemcpyDeviceToHost));
      for (int64_t e = 0; e < m; ++e)
        for (int k = 0; k < 18; ++k) qpoints[18 * e + k] = q[QS * e + k];
    }
  }
  return HBEM_OK;
}

int hbem_integrate_regular(hbem_ctx *ctx, const int64_t *pairs, int64_t p, void *re, void *im) {
  clear_error();
  return integrate_host(ctx, pairs, p, re, im, 1, nullptr);
}

int hbem_integrate_any(hbem_ctx *ctx, const int64_t *pairs, int64_t p, void *re, void *im,
                       int64_t *n_singular) {
  clear_error();
  return integrate_host(ctx, pairs, p, re, im, 2, n_singular);
}

int hbem_integrate_regular_device(hbem_ctx *ctx, const int64_t *d_pairs, int64_t p, void *d_re,
                                  void *d_im, void *stream) {
  clear_error();
  if (!ctx) return set_error(HBEM_ERR_ARG, "null context");
  HB_CUDA(cudaSetDevice(ctx->device));
  return integrate_pairs_device(ctx, d_pairs, p, d_re, d_im, 0, nullptr, nullptr,
                                (cudaStream_t)stream);
}

int hbem_integrate_any_device(hbem_ctx *ctx, const int64_t *d_pairs, int64_t p, void *d_re,
                              void *d_im, void *stream) {
  clear_error();
  if (!ctx) return set_error(HBEM_ERR_ARG, "null context");
  HB_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = (cudaStream_t)stream;
  int *list = nullptr;
  unsigned long long *flags = nullptr;
  HB_CUDA(cudaMallocAsync((void **)&list, (size_t)std::max<int64_t>(p, 1) * 4, st));
  HB_CUDA(cudaMallocAsync((void **)&flags, 64, st));
  int rc = integrate_pairs_device(ctx, d_pairs, p, d_re, d_im, 2, list, flags, st);
  cudaFreeAsync(list, st);
  cudaFreeAsync(flags, st);
  return rc;
}

}  // extern "C"
