// Far-field potential of a surface density (evaluate_far_field,
// scatter.py:362-408): u(x) = sum_{elements, rule points} K_dlp(x, y_q) dens_q,
// dens_q = (sum_l phi[dofmap[e, l]] table[l, q]) * (|J_e| w_q), K_dlp the
// (Helmholtz or Laplace) double-layer kernel of kernel_planes
// (kernels.py:129-158) with n_trial = n_e.
//
//   k_far_dens : one thread per element: geometry in the numpy operation
//                order of precompute_geometry (mesh.py:344-359, no FMA
//                contraction), rule points mapped, densities formed
//   k_far      : CTA = 64 points x 4 element lanes over one element chunk;
//                the chunk's points (x, y, z, dens) stream through shared
//                memory; partial sums per (chunk, point), minimum distance
//   k_far_sum  : partials summed over the chunks in chunk order (fixed
//                reduction order: bitwise reproducible for a given device)
//
// FP64 (the reference path is float64); FP64-pipe bound: per evaluation
// 3 sub + 5 (r^2) + sqrt/div + 5 (dot) + amp 2 + sincos (Helmholtz) + 8 (complex
// kernel x density).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "hbem_internal.h"

namespace hb {
namespace {

constexpr int kFarPts = 64;    // points per CTA
constexpr int kFarLanes = 4;   // element lanes per point
constexpr int kFarStage = 256; // rule points staged per smem round
constexpr int kMaxQ = 6;
constexpr double kInv4Pi = 0.07957747154594767;  // 1 / (4 pi), kernels.py INV_4PI

struct FarSoA {
  double *qx, *qy, *qz, *nx, *ny, *nz, *dre, *dim;  // (m*nq) except n (m)
};

__global__ void k_far_dens(const double *vtx, const long long *elem, long long m, int nq,
                           const double *rp, const double *rw, int ld, const double *table,
                           const long long *dofmap, const double *phr, const double *phi,
                           FarSoA S) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= m) return;
  double v[3][3];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c) v[a][c] = vtx[3 * elem[3 * e + a] + c];
  double e1[3], e2[3];
  for (int c = 0; c < 3; ++c) {
    e1[c] = __dsub_rn(v[1][c], v[0][c]);
    e2[c] = __dsub_rn(v[2][c], v[0][c]);
  }
  double cr[3];
  cr[0] = __dsub_rn(__dmul_rn(e1[1], e2[2]), __dmul_rn(e1[2], e2[1]));
  cr[1] = __dsub_rn(__dmul_rn(e1[2], e2[0]), __dmul_rn(e1[0], e2[2]));
  cr[2] = __dsub_rn(__dmul_rn(e1[0], e2[1]), __dmul_rn(e1[1], e2[0]));
  const double jac = __dsqrt_rn(__dadd_rn(
      __dadd_rn(__dmul_rn(cr[0], cr[0]), __dmul_rn(cr[1], cr[1])), __dmul_rn(cr[2], cr[2])));
  S.nx[e] = __ddiv_rn(cr[0], jac);
  S.ny[e] = __ddiv_rn(cr[1], jac);
  S.nz[e] = __ddiv_rn(cr[2], jac);
  for (int q = 0; q < nq; ++q) {
    const double xi = rp[2 * q], eta = rp[2 * q + 1];
    const long long o = e * nq + q;
    double p[3];
    for (int c = 0; c < 3; ++c) p[c] = __dadd_rn(__dadd_rn(v[0][c], __dmul_rn(xi, e1[c])),
                                                 __dmul_rn(eta, e2[c]));
    S.qx[o] = p[0];
    S.qy[o] = p[1];
    S.qz[o] = p[2];
    // einsum("ml,lq->mq", phi[dofmap], table) * (jac * w)
    double sr = 0.0, si = 0.0;
    for (int l = 0; l < ld; ++l) {
      const long long d = dofmap[e * ld + l];
      const double t = table[l * nq + q];
      sr = __dadd_rn(sr, __dmul_rn(phr[d], t));
      if (phi) si = __dadd_rn(si, __dmul_rn(phi[d], t));
    }
    const double jw = __dmul_rn(jac, rw[q]);
    S.dre[o] = __dmul_rn(sr, jw);
    S.dim[o] = __dmul_rn(si, jw);
  }
}

template <bool HELM>
__global__ void __launch_bounds__(kFarPts * kFarLanes) k_far(const double *pts, long long n,
                                                             FarSoA S, long long m, int nq,
                                                             long long chunk, double k,
                                                             double *part /* (chunks, n, 3) */) {
  __shared__ double sx[kFarStage], sy[kFarStage], sz[kFarStage], snx[kFarStage],
      sny[kFarStage], snz[kFarStage], sdr[kFarStage], sdi[kFarStage];
  __shared__ double red[3][kFarLanes][kFarPts];
  const int pl = threadIdx.x % kFarPts, lane = threadIdx.x / kFarPts;
  const long long p = blockIdx.x * (long long)kFarPts + pl;
  const long long c = blockIdx.y;
  const long long q0 = c * chunk * nq, q1 = min(m, (c + 1) * chunk) * nq;
  double x0 = 0.0, x1 = 0.0, x2 = 0.0;
  if (p < n) {
    x0 = pts[3 * p];
    x1 = pts[3 * p + 1];
    x2 = pts[3 * p + 2];
  }
  double are = 0.0, aim = 0.0, rmin = INFINITY;
  for (long long base = q0; base < q1; base += kFarStage) {
    const int cnt = (int)min((long long)kFarStage, q1 - base);
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const long long o = base + i, e = o / nq;
      sx[i] = S.qx[o];
      sy[i] = S.qy[o];
      sz[i] = S.qz[o];
      snx[i] = S.nx[e];
      sny[i] = S.ny[e];
      snz[i] = S.nz[e];
      sdr[i] = S.dre[o];
      sdi[i] = S.dim[o];
    }
    __syncthreads();
    for (int i = lane; i < cnt; i += kFarLanes) {
      const double d0 = x0 - sx[i], d1 = x1 - sy[i], d2 = x2 - sz[i];
      const double r2 = d0 * d0 + d1 * d1 + d2 * d2;
      const double r = sqrt(r2);
      rmin = fmin(rmin, r);
      const double dot = d0 * snx[i] + d1 * sny[i] + d2 * snz[i];
      const double amp = dot * (kInv4Pi / (r2 * r));
      if (HELM) {
        const double kr = k * r;
        double s, co;
        sincos(kr, &s, &co);
        const double kre = amp * (co + kr * s), kim = amp * (s - kr * co);
        are += kre * sdr[i] - kim * sdi[i];
        aim += kre * sdi[i] + kim * sdr[i];
      } else {
        are += amp * sdr[i];
        aim += amp * sdi[i];
      }
    }
  }
  red[0][lane][pl] = are;
  red[1][lane][pl] = aim;
  red[2][lane][pl] = rmin;
  __syncthreads();
  if (lane == 0 && p < n) {
    double sr = red[0][0][pl], si = red[1][0][pl], mn = red[2][0][pl];
    for (int l = 1; l < kFarLanes; ++l) {
      sr += red[0][l][pl];
      si += red[1][l][pl];
      mn = fmin(mn, red[2][l][pl]);
    }
    double *o = part + 3 * (c * n + p);
    o[0] = sr;
    o[1] = si;
    o[2] = mn;
  }
}

__global__ void k_far_sum(const double *part, long long n, int chunks, double *ore, double *oim,
                          double *rmin) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= n) return;
  double sr = 0.0, si = 0.0, mn = INFINITY;
  for (int c = 0; c < chunks; ++c) {
    const double *o = part + 3 * (c * n + p);
    sr += o[0];
    si += o[1];
    mn = fmin(mn, o[2]);
  }
  ore[p] = sr;
  oim[p] = si;
  rmin[p] = mn;
}

}  // namespace
}  // namespace hb

using namespace hb;

extern "C" int hbem_far_field(int32_t device, int64_t n_points, const double *points,
                              int64_t n_vertices, const double *vertices, int64_t m,
                              const int64_t *elements, int32_t nq, const double *rule_points,
                              const double *rule_weights, int32_t local_dim, const double *table,
                              const int64_t *dofmap, int64_t n_dofs, const double *phi_re,
                              const double *phi_im, double wavenumber, double *out_re,
                              double *out_im, double *r_min) {
  clear_error();
  if (!points || !vertices || !elements || !rule_points || !rule_weights || !table || !dofmap ||
      !phi_re || !out_re || !out_im)
    return set_error(HBEM_ERR_ARG, "null argument");
  if (n_points < 0 || m < 1 || nq < 1 || nq > kMaxQ || local_dim < 1 || local_dim > 3)
    return set_error(HBEM_ERR_ARG, "bad sizes (points %lld, elements %lld, rule %d, local %d)",
                     (long long)n_points, (long long)m, nq, local_dim);
  for (int64_t i = 0; i < 3 * m; ++i)
    if (elements[i] < 0 || elements[i] >= n_vertices)
      return set_error(HBEM_ERR_ARG, "element vertex index out of range");
  for (int64_t i = 0; i < m * local_dim; ++i)
    if (dofmap[i] < 0 || dofmap[i] >= n_dofs)
      return set_error(HBEM_ERR_ARG, "dofmap index out of range");
  if (n_points == 0) return HBEM_OK;
  HB_CUDA(cudaSetDevice(device));
  std::vector<void *> allocs;
  auto cleanup = [&]() {
    for (void *q : allocs) cudaFree(q);
  };
  auto dev = [&](void **p, size_t bytes, const void *src) -> cudaError_t {
    cudaError_t e = cudaMalloc(p, std::max<size_t>(bytes, 8));
    if (e != cudaSuccess) return e;
    allocs.push_back(*p);
    if (src) e = cudaMemcpy(*p, src, bytes, cudaMemcpyHostToDevice);
    return e;
  };
  const long long mq = m * (long long)nq;
  // element chunks: (point tiles x chunks) just below four full waves of
  // resident CTAs (a fraction of a wave left over would idle most SMs)
  const long long tiles = (n_points + kFarPts - 1) / kFarPts;
  int sms = 148, per_sm = 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (wavenumber != 0.0)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_far<true>, kFarPts * kFarLanes, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_far<false>, kFarPts * kFarLanes, 0);
  const long long slots = (long long)sms * std::max(per_sm, 1);
  long long chunks = std::max<long long>(1, std::min<long long>(4 * slots / tiles,
                                                                (m + 63) / 64));
  chunks = std::min<long long>(chunks, 65535);
  const long long chunk = (m + chunks - 1) / chunks;
  chunks = (m + chunk - 1) / chunk;
  void *d_vtx, *d_el, *d_rp, *d_rw, *d_tab, *d_dm, *d_pr, *d_pi = nullptr, *d_pts, *d_soa,
      *d_part, *d_out;
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = dev(&d_vtx, (size_t)n_vertices * 24, vertices);
  if (e == cudaSuccess) e = dev(&d_el, (size_t)m * 24, elements);
  if (e == cudaSuccess) e = dev(&d_rp, (size_t)nq * 16, rule_points);
  if (e == cudaSuccess) e = dev(&d_rw, (size_t)nq * 8, rule_weights);
  if (e == cudaSuccess) e = dev(&d_tab, (size_t)local_dim * nq * 8, table);
  if (e == cudaSuccess) e = dev(&d_dm, (size_t)m * local_dim * 8, dofmap);
  if (e == cudaSuccess) e = dev(&d_pr, (size_t)n_dofs * 8, phi_re);
  if (e == cudaSuccess && phi_im) e = dev(&d_pi, (size_t)n_dofs * 8, phi_im);
  if (e == cudaSuccess) e = dev(&d_pts, (size_t)n_points * 24, points);
  if (e == cudaSuccess) e = dev(&d_soa, (size_t)(6 * mq + 3 * m) * 8, nullptr);
  if (e == cudaSuccess) e = dev(&d_part, (size_t)chunks * n_points * 24, nullptr);
  if (e == cudaSuccess) e = dev(&d_out, (size_t)n_points * 24, nullptr);
  if (e != cudaSuccess) {
    cleanup();
    cudaGetLastError();
    return set_error(HBEM_ERR_CAPACITY, "far field: device allocation failed: %s",
                     cudaGetErrorString(e));
  }
  double *soa = static_cast<double *>(d_soa);
  FarSoA S{soa, soa + mq, soa + 2 * mq, soa + 3 * mq, soa + 3 * mq + m, soa + 3 * mq + 2 * m,
           soa + 3 * mq + 3 * m, soa + 4 * mq + 3 * m};
  k_far_dens<<<(unsigned)((m + 127) / 128), 128>>>(
      static_cast<const double *>(d_vtx), static_cast<const long long *>(d_el), m, nq,
      static_cast<const double *>(d_rp), static_cast<const double *>(d_rw), local_dim,
      static_cast<const double *>(d_tab), static_cast<const long long *>(d_dm),
      static_cast<const double *>(d_pr), static_cast<const double *>(d_pi), S);
  const dim3 grid((unsigned)tiles, (unsigned)chunks);
  double *part = static_cast<double *>(d_part);
  if (wavenumber != 0.0)
    k_far<true><<<grid, kFarPts * kFarLanes>>>(static_cast<const double *>(d_pts), n_points, S,
                                               m, nq, chunk, wavenumber, part);
  else
    k_far<false><<<grid, kFarPts * kFarLanes>>>(static_cast<const double *>(d_pts), n_points, S,
                                                m, nq, chunk, 0.0, part);
  double *o = static_cast<double *>(d_out);
  k_far_sum<<<(unsigned)((n_points + 127) / 128), 128>>>(part, n_points, (int)chunks, o,
                                                         o + n_points, o + 2 * n_points);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(out_re, o, (size_t)n_points * 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess)
    e = cudaMemcpy(out_im, o + n_points, (size_t)n_points * 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && r_min)
    e = cudaMemcpy(r_min, o + 2 * n_points, (size_t)n_points * 8, cudaMemcpyDeviceToHost);
  cleanup();
  HB_CUDA(e);
  return HBEM_OK;
}
