// Internal host-side state shared by the hbem_b200 translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>
#include <type_traits>
#include <utility>

#include "../../include/hbem_b200.h"
#include "hbem_device.cuh"

namespace hb {

int set_error(int code, const char *fmt, ...);
void clear_error();

#define HB_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess)                                                              \
      return ::hb::set_error(HBEM_ERR_CUDA, "CUDA error %s at %s:%d: %s",               \
                             cudaGetErrorName(_e), __FILE__, __LINE__,                  \
                             cudaGetErrorString(_e));                                   \
  } while (0)

#define HB_CHECK(call)            \
  do {                            \
    int _s = (call);              \
    if (_s != HBEM_OK) return _s; \
  } while (0)

template <int V> using IC = std::integral_constant<int, V>;

// Calls fn(IC<OP>, IC<HELM>, IC<NT>, IC<NS>) for the runtime combination.
// hyps is only instantiated for linear x linear spaces (kernels.py:212-214).
template <typename Fn>
int dispatch_op(int op, bool helm, int nt, int ns, Fn &&fn) {
  auto shapes = [&](auto OPc, auto Hc) -> int {
    constexpr int OPv = decltype(OPc)::value;
    if (nt == 3 && ns == 3) return fn(OPc, Hc, IC<3>{}, IC<3>{});
    if constexpr (OPv != HBEM_HYPS) {
      if (nt == 1 && ns == 1) return fn(OPc, Hc, IC<1>{}, IC<1>{});
      if (nt == 1 && ns == 3) return fn(OPc, Hc, IC<1>{}, IC<3>{});
      if (nt == 3 && ns == 1) return fn(OPc, Hc, IC<3>{}, IC<1>{});
    }
    return set_error(HBEM_ERR_KERNEL, "unsupported block shape (%d, %d) for operator %d", nt,
                     ns, op);
  };
  auto eq = [&](auto OPc) -> int {
    return helm ? shapes(OPc, IC<1>{}) : shapes(OPc, IC<0>{});
  };
  switch (op) {
    case HBEM_SLP: return eq(IC<HBEM_SLP>{});
    case HBEM_DLP: return eq(IC<HBEM_DLP>{});
    case HBEM_ADLP: return eq(IC<HBEM_ADLP>{});
    case HBEM_HYPS: return eq(IC<HBEM_HYPS>{});
  }
  return set_error(HBEM_ERR_KERNEL, "unknown operator %d", op);
}

}  // namespace hb

struct hbem_ctx {
  int device = 0;
  int equation = 0, op = 0, precision = 0;
  double wavenumber = 0.0;
  int test_family = 0, trial_family = 0;
  int nt = 1, ns = 1;
  bool helm = false;
  int64_t m = 0, nv = 0;
  // device buffers
  void *q = nullptr;        // m x QStride<T>
  void *nj = nullptr;       // m x 4 T
  void *curl = nullptr;     // m x 9 T (hyps)
  double *nj64 = nullptr;   // m x 4 double (aliases nj when T = double)
  double *curl64 = nullptr; // m x 9 double (hyps; aliases curl when T = double)
  double *vtx = nullptr;    // nv x 3
  int4 *elem = nullptr;     // m
  double *sp[3] = {nullptr, nullptr, nullptr};
  double *sw[3] = {nullptr, nullptr, nullptr};
  int sn[3] = {0, 0, 0};
  hb::RuleTab<double> rd;
  hb::RuleTab<float> rf;

  int real_bytes() const { return precision == HBEM_DOUBLE ? 8 : 4; }
  template <typename T> hb::Geo<T> geo() const {
    return hb::Geo<T>{static_cast<const T *>(q), static_cast<const T *>(nj),
                      static_cast<const T *>(curl), m};
  }
  template <typename T> const hb::RuleTab<T> &rule() const;
  hb::Geo64 geo64() const {
    hb::Geo64 g;
    g.vtx = vtx;
    g.elem = elem;
    g.nj = nj64;
    g.curl = curl64;
    g.m = m;
    for (int i = 0; i < 3; ++i) { g.sp[i] = sp[i]; g.sw[i] = sw[i]; g.sn[i] = sn[i]; }
    g.k = wavenumber;
    g.k2 = wavenumber * wavenumber;
    return g;
  }
};

template <> inline const hb::RuleTab<double> &hbem_ctx::rule<double>() const { return rd; }
template <> inline const hb::RuleTab<float> &hbem_ctx::rule<float>() const { return rf; }

namespace hb {
// Internal device-side entry points used by the H-matrix assembler.
// Integrate arbitrary pairs (device pointers), any adjacency, into
// (p, nt, ns) planes of the working precision.  flags: device scratch of
// >= 4 unsigned long long, sing_list: device scratch of p ints.
int integrate_pairs_device(hbem_ctx *ctx, const int64_t *d_pairs, int64_t p, void *d_re,
                           void *d_im, int mode, int *d_sing_list, unsigned long long *d_flags,
                           cudaStream_t stream);
}  // namespace hb
