// Device H-matrix assembly: near-field dense leaves + lock-step batched ACA
// over every admissible leaf (assemble_hmatrix, hmatrix.py:759-811).
//
// This translation unit holds the host orchestration (setup = partition
// upload and index structures, execute = one full assembly), the generic
// dense-entry kernels (linear spaces, ACA fallback blocks) and payload
// packing.  The ACA wave kernels live in aca_impl.cuh, the P0 near-field
// kernels in near_impl.cuh (instantiated per precision in kern_f64.cu /
// kern_f32.cu).
//
// Per-block decisions follow aca() (hmatrix.py:271-382) exactly:
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
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <initializer_list>
#include <tuple>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#include <cub/cub.cuh>

#include "hmat_common.cuh"

namespace hb {

// K4: dense entries (near-field leaves and ACA fallback blocks).
// tiles: (slot, first entry); slot -> (r0, c0, h, w, offset)
// P0 touching entries are queued for the warp-per-pair singular kernel.
// ---------------------------------------------------------------------------


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
    for (int l = 0; l < k; ++l) {  // record [u | r | p], v = r / p
      const V *t = pool + S.terms[(long long)b * S.tmax + l];
      acc = N::fma_acc(acc, t[i], N::div(t[h + c], t[h + w]));
    }
    o[idx] = acc;
  }
}

// pack the factors of low-rank blocks into the U / V arenas, one CTA per
// block (v = r / p as r * (1 / p): one division per term)
template <typename Tr, bool Cc, typename V = typename Num<Tr, Cc>::V>
__global__ void k_pack_factors(const int *slots, int n, AcaDev S, const long long *uoff,
                               const long long *voff, long long ubase, long long vbase, V *u,
                               V *v) {
  using N = Num<Tr, Cc>;
  const int q = blockIdx.x;
  if (q >= n) return;
  const int b = slots[q];
  const int h = S.h[b], w = S.w[b], k = S.rank[b];
  const V *pool = static_cast<const V *>(S.pool);
  for (int l = 0; l < k; ++l) {
    const V *t = pool + S.terms[(long long)b * S.tmax + l];
    for (int r = threadIdx.x; r < h; r += blockDim.x)
      u[uoff[q] - ubase + (long long)l * h + r] = t[r];
    const V inv = N::div(N::mk(Tr(1), Tr(0)), t[h + w]);
    for (int c = threadIdx.x; c < w; c += blockDim.x)
      v[voff[q] - vbase + (long long)l * w + c] = N::fma_acc(N::zero(), t[h + c], inv);
  }
}

// streamed emission straight into the caller's page-locked host arenas: SM
// stores over PCIe (posted writes; a few CTAs saturate the link), a warp per
// block, grid-stride; no device staging arena and no copy engine. Same
// values as k_pack_factors bit for bit.
template <typename Tr, bool Cc, typename V = typename Num<Tr, Cc>::V>
__global__ void __launch_bounds__(256) k_pack_host(const int *slots, int n, AcaDev S,
                                                   const long long *uoff, const long long *voff,
                                                   V *u, V *v) {
  using N = Num<Tr, Cc>;
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * (blockDim.x >> 5);
  const V *pool = static_cast<const V *>(S.pool);
  for (int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < n; q += nw) {
    const int b = slots[q];
    const int h = S.h[b], w = S.w[b], k = S.rank[b];
    V *ub = u + uoff[q], *vb = v + voff[q];
    const long long *terms = S.terms + (long long)b * S.tmax;
    for (int l0 = 0; l0 < k; l0 += 32) {
      // term offsets fetched lane-parallel, values loaded ahead of the
      // (posted) PCIe stores: several independent loads in flight per lane
      const long long my = l0 + lane < k ? terms[l0 + lane] : 0;
      const int nl = min(32, k - l0);
      for (int j = 0; j < nl; ++j) {
        const V *t = pool + __shfl_sync(0xffffffffu, my, j);
        const long long l = l0 + j;
        const V p = t[h + w];
        V ur[4], vr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = lane + 32 * i, c = lane + 32 * i;
          if (r < h) ur[i] = t[r];
          if (c < w) vr[i] = t[h + c];
        }
        const V inv = N::div(N::mk(Tr(1), Tr(0)), p);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = lane + 32 * i, c = lane + 32 * i;
          if (r < h) ub[l * h + r] = ur[i];
          if (c < w) vb[l * w + c] = N::fma_acc(N::zero(), vr[i], inv);
        }
        for (int r = lane + 128; r < h; r += 32) ub[l * h + r] = t[r];
        for (int c = lane + 128; c < w; c += 32) vb[l * w + c] = N::fma_acc(N::zero(), t[h + c], inv);
      }
    }
  }
}

// per-wave emission of converged low-rank blocks (lowrank_leaf rule,
// hmatrix.py:721-729): flags in block order, not yet emitted
__global__ void k_emit_flags(AcaDev S, int na, unsigned char *emitted, unsigned char *flag) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= na) return;
  const long long h = S.h[b], w = S.w[b], k = S.rank[b];
  const bool f = !emitted[b] && S.status[b] == ST_CONVERGED && k * (h + w) < h * w;
  flag[b] = f ? 1 : 0;
  if (f) emitted[b] = 1;
}

__global__ void k_emit_need(AcaDev S, const int *list, const int *cnt, int na, longlong2 *need) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= na) return;
  longlong2 d = make_longlong2(0, 0);
  if (p < *cnt) {
    const int b = list[p];
    const long long k = S.rank[b];
    d = make_longlong2((long long)S.h[b] * k, (long long)S.w[b] * k);
  }
  need[p] = d;
}

__global__ void k_emit_offsets(const int *list, int n, const longlong2 *scan,
                               const longlong2 *need, long long ubase, long long vbase,
                               long long *blk_uoff, long long *blk_voff, long long *q_uoff,
                               long long *q_voff) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int b = list[p];
  const long long uo = ubase + scan[p].x - need[p].x, vo = vbase + scan[p].y - need[p].y;
  blk_uoff[b] = uo;
  blk_voff[b] = vo;
  q_uoff[p] = uo;
  q_voff[p] = vo;
}

// small device -> host reads (phase totals, counters) while payloads stream:
// a one-warp kernel stores into the mapped page-locked mailbox, because a
// cudaMemcpyAsync D2H would queue on the copy engine behind the multi-GB
// payload copies and stall the wave loop on them
struct MailCopy {
  const unsigned *src[3];
  unsigned *dst[3];
  int words[3];
};

__global__ void k_mail(MailCopy m) {
  for (int r = 0; r < 3; ++r)
    for (int i = threadIdx.x; i < m.words[r]; i += blockDim.x) m.dst[r][i] = m.src[r][i];
}

// classification of every admissible block after the waves (lowrank_leaf /
// dense fallback, hmatrix.py:721-735), on the device: per-leaf metadata
// written in place (kind, rank, flags | off_u, off_v, off_dense), dense sizes
// for the offset scan, low-rank / dense flags for the two block lists
struct LeafMeta {
  int *kind, *rank, *flags;           // L each
  long long *off_u, *off_v, *off_d;   // L each
  double *resid;                      // L: ACA residual indicator (LowRankBlock.residual)
};

struct ClsStat {
  unsigned long long converged, exhausted;
  int overflow_q, pad;
};

__global__ void k_classify(AcaDev S, int na, const int *adm_leaf, const long long *blk_uoff,
                           const long long *blk_voff, LeafMeta M, longlong2 *dsz,
                           unsigned char *flag_lr, unsigned char *flag_dn, ClsStat *cs) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  bool conv = false, exh = false;
  if (q < na) {
    const int s = S.status[q];
    const long long h = S.h[q], w = S.w[q], k = S.rank[q];
    conv = s == ST_CONVERGED;
    exh = S.exhausted[q] != 0;
    if (s == ST_OVERFLOW) atomicMin(&cs->overflow_q, q);
    const bool lr = conv && k * (h + w) < h * w;
    const int lf = adm_leaf[q];
    M.kind[lf] = lr ? 1 : 0;
    M.rank[lf] = (int)k;
    M.flags[lf] = (conv ? 1 : 0) | (exh ? 2 : 0);
    M.off_u[lf] = lr ? blk_uoff[q] : -1;
    M.off_v[lf] = lr ? blk_voff[q] : -1;
    // last update relative to the Frobenius norm (hmatrix.py:377-382); inf
    // until a term was accepted, 0 for a block without terms
    M.resid[lf] = k > 0 ? S.resid[q] : 0.0;
    if (lr) M.off_d[lf] = -1;  // dense offsets after the scan
    dsz[q] = make_longlong2(lr ? 0 : h * w, 0);
    flag_lr[q] = lr ? 1 : 0;
    flag_dn[q] = lr ? 0 : 1;
  }
  const unsigned nc = __popc(__ballot_sync(0xffffffffu, conv));
  const unsigned ne = __popc(__ballot_sync(0xffffffffu, exh));
  if ((threadIdx.x & 31) == 0) {
    if (nc) atomicAdd(&cs->converged, (unsigned long long)nc);
    if (ne) atomicAdd(&cs->exhausted, (unsigned long long)ne);
  }
}

// dense admissible blocks (block order): off_dense after the near field and
// the host record {block | converged << 31, offset}
__global__ void k_classify_dense(const int *list, const int *cnt, AcaDev S,
                                 const longlong2 *scan, const longlong2 *dsz, const int *adm_leaf,
                                 long long nf_entries, LeafMeta M, longlong2 *info) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= *cnt) return;
  const int q = list[p];
  const long long off = scan[q].x - dsz[q].x;
  M.off_d[adm_leaf[q]] = nf_entries + off;
  const long long conv = S.status[q] == ST_CONVERGED ? 1 : 0;
  info[p] = make_longlong2((long long)q | (conv << 31), off);
}

__global__ void k_gather_ll(const int *list, int n, const long long *src, long long *dst) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) dst[p] = src[list[p]];
}

struct SumLL2 {
  __device__ __forceinline__ longlong2 operator()(const longlong2 &a, const longlong2 &b) const {
    return make_longlong2(a.x + b.x, a.y + b.y);
  }
};

}  // namespace hb

using namespace hb;

// ---------------------------------------------------------------------------
// host side: setup (partition upload, index structures) and execute (one
// complete assembly: record gather, near-field leaves, ACA waves, payloads)
// ---------------------------------------------------------------------------
// Growable device pool on the CUDA virtual memory API: a large virtual range
// is reserved once and physical memory is mapped in 2 GiB steps as the ACA
// waves need it, so the factor pool occupies what the assembly actually
// stores (a few % over the payload) instead of a worst-case estimate.
// driver-API entry points resolved through the runtime (no link-time
// dependency on libcuda, so the library still loads on GPU-less hosts)
struct VmmApi {
  PFN_cuMemGetAllocationGranularity granularity = nullptr;
  PFN_cuMemAddressReserve reserve = nullptr;
  PFN_cuMemAddressFree address_free = nullptr;
  PFN_cuMemCreate create = nullptr;
  PFN_cuMemRelease release = nullptr;
  PFN_cuMemMap map = nullptr;
  PFN_cuMemUnmap unmap = nullptr;
  PFN_cuMemSetAccess set_access = nullptr;
  bool load() {
    if (create) return true;
    auto get = [](const char *name, void **fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn;
    };
    return get("cuMemGetAllocationGranularity", (void **)&granularity) &&
           get("cuMemAddressReserve", (void **)&reserve) &&
           get("cuMemAddressFree", (void **)&address_free) &&
           get("cuMemCreate", (void **)&create) && get("cuMemRelease", (void **)&release) &&
           get("cuMemMap", (void **)&map) && get("cuMemUnmap", (void **)&unmap) &&
           get("cuMemSetAccess", (void **)&set_access);
  }
};
static VmmApi g_vmm;


struct VPool {
  CUdeviceptr base = 0;
  size_t reserved = 0, mapped = 0, step = 0;
  double grow_s = 0.0;  // host time spent mapping (trace)
  std::vector<CUmemGenericAllocationHandle> handles;
  std::vector<size_t> sizes;
  CUmemAllocationProp prop{};
  int dev = 0;
  int init(int device, size_t reserve_bytes) {
    dev = device;
    if (!g_vmm.load()) return set_error(HBEM_ERR_CUDA, "CUDA virtual memory API unavailable");
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = device;
    size_t gran = 0;
    if (g_vmm.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) !=
        CUDA_SUCCESS)
      return set_error(HBEM_ERR_CUDA, "cuMemGetAllocationGranularity failed");
    step = std::max<size_t>(gran, (size_t)2 << 30);
    step = (step + gran - 1) / gran * gran;
    reserved = (reserve_bytes + step - 1) / step * step;
    if (g_vmm.reserve(&base, reserved, 0, 0, 0) != CUDA_SUCCESS)
      return set_error(HBEM_ERR_CAPACITY, "cannot reserve %zu bytes of device address space",
                       reserved);
    return HBEM_OK;
  }
  // map until at least `bytes` are backed
  int grow(size_t bytes) {
    if (mapped >= bytes) return HBEM_OK;
    const auto t0 = std::chrono::steady_clock::now();
    struct Acc {
      double &s;
      std::chrono::steady_clock::time_point t;
      ~Acc() { s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count(); }
    } acc_{grow_s, t0};
    while (mapped < bytes) {
      if (mapped + step > reserved)
        return set_error(HBEM_ERR_CAPACITY, "ACA factor pool exhausted (%zu bytes reserved)",
                         reserved);
      CUmemGenericAllocationHandle hnd;
      if (g_vmm.create(&hnd, step, &prop, 0) != CUDA_SUCCESS)
        return set_error(HBEM_ERR_CAPACITY,
                         "device memory exhausted growing the ACA factor pool to %zu bytes",
                         mapped + step);
      if (g_vmm.map(base + mapped, step, 0, hnd, 0) != CUDA_SUCCESS) {
        g_vmm.release(hnd);
        return set_error(HBEM_ERR_CUDA, "cuMemMap failed");
      }
      CUmemAccessDesc acc{};
      acc.location = prop.location;
      acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
      if (g_vmm.set_access(base + mapped, step, &acc, 1) != CUDA_SUCCESS)
        return set_error(HBEM_ERR_CUDA, "cuMemSetAccess failed");
      handles.push_back(hnd);
      sizes.push_back(step);
      mapped += step;
    }
    return HBEM_OK;
  }
  ~VPool() {
    if (!base) return;
    size_t off = 0;
    for (size_t i = 0; i < handles.size(); ++i) {
      g_vmm.unmap(base + off, sizes[i]);
      g_vmm.release(handles[i]);
      off += sizes[i];
    }
    g_vmm.address_free(base, reserved);
  }
};

struct hbem_hmat {
  hbem_ctx *ctx = nullptr;
  int device = 0;
  int64_t n_leaves = 0;
  bool complex_ = false;
  size_t vbytes = 8;
  int nt = 1, ns = 1;
  bool p0 = false;  // both spaces P0: register-resident record kernels
  // per leaf results (device; near-field entries written once at setup,
  // admissible ones by k_classify every execute)
  LeafMeta meta{};
  // partition views (device)
  const int *rperm = nullptr, *cperm = nullptr;
  const int *tptr = nullptr, *tel = nullptr, *sptr = nullptr, *sel = nullptr;
  const signed char *tloc = nullptr, *sloc = nullptr;
  // tree-ordered element records (P0)
  void *trec = nullptr, *srec = nullptr;
  int n_rows = 0, n_cols = 0;
  bool same_tree = false;
  // admissible blocks
  int na = 0;
  std::vector<int> adm_leaf, ah, aw, ar0, ac0;
  int *row_order = nullptr, *col_order = nullptr;
  int *listA = nullptr, *listC = nullptr, *d_cnt = nullptr, *sel_tmp = nullptr;
  void *cub_tmp = nullptr;
  size_t cub_bytes = 0;
  double *partA = nullptr, *partC = nullptr;
  size_t partA_cap = 0, partC_cap = 0;  // doubles
  long long items_cap = 0;
  bool use_erows = false;       // linear spaces: element-level ACA rows
  long long eitems_cap = 0;
  void *rsc = nullptr;          // element-row values of the current phase
  size_t rsc_cap = 0;           // bytes
  AcaDev S{};
  VPool vpool;  // ACA factor pool
  Geo64 *g64p = nullptr;  // device copy of the context's float64 geometry view
  // pinned mailbox for the per-phase host reads
  struct Mail { Need tot; int n; int pad; int cls_cnt[2]; ClsStat cls; long long adm_dense; } *mail = nullptr;
  char *mail_dev = nullptr;  // device view of the mailbox
  // D2H of up to three small device ranges into mailbox fields (k_mail)
  int read_mail(cudaStream_t st, std::initializer_list<std::tuple<void *, const void *, size_t>> r) {
    if (!streaming()) {
      // copy engine idle: plain D2H (a kernel would wait for an SM slot
      // behind the low-priority near-field CTAs, ~ms per phase)
      for (const auto &[dst, src, bytes] : r)
        HB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
      HB_CUDA(cudaStreamSynchronize(st));
      return HBEM_OK;
    }
    MailCopy m{};
    int i = 0;
    for (const auto &[dst, src, bytes] : r) {
      m.dst[i] = reinterpret_cast<unsigned *>(mail_dev + (static_cast<char *>(dst) -
                                                          reinterpret_cast<char *>(mail)));
      m.src[i] = static_cast<const unsigned *>(src);
      m.words[i] = (int)(bytes / 4);
      ++i;
    }
    k_mail<<<1, 32, 0, st>>>(m);
    HB_CUDA(cudaGetLastError());
    HB_CUDA(cudaStreamSynchronize(st));
    return HBEM_OK;
  }
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
  // block lists of the last execute (device, block order)
  int *d_adm_leaf = nullptr, *lr_list = nullptr, *dn_list = nullptr, *cls_cnt = nullptr;
  unsigned char *cls_flag = nullptr;
  ClsStat *cls_stat = nullptr;
  longlong2 *dn_info = nullptr;
  int n_lowrank = 0;
  // matvec: admissible blocks stored densely (host lists, uploaded lazily)
  std::vector<int> ad_r0, ad_c0, ad_h, ad_w;
  std::vector<long long> ad_off, ad_rowbase;
  long long nf_rows = 0;
  const long long *nf_rowbase = nullptr;
  long long sing_pairs_table = 0;  // Sauter-Schwab pairs of this handle's table
  bool mv_dirty = true;
  void *mv_buf = nullptr;  // x, y, xt, yt
  int *mv_ad = nullptr;
  long long *mv_ad_l = nullptr;
  int2 *mv_items = nullptr;       // low-rank dots items, then rows items
  long long *mv_sbase = nullptr;  // per low-rank list position
  void *mv_s = nullptr;
  long long mv_nd = 0, mv_nr = 0, mv_ns = 0;
  // deterministic matvec: partial slots, chunk dots, cover lists (device)
  void *mv_part = nullptr, *mv_dpart = nullptr;
  long long *mv_ifirst = nullptr, *mv_ibase = nullptr, *mv_rbase = nullptr;
  int *mv_cstart = nullptr;
  long long *mv_cptr = nullptr, *mv_cover = nullptr;
  int mv_ncl = 0;
  long long mv_ad_rows = 0;
  // host copies for the matvec's cover lists
  std::vector<int> nf_r0, nf_c0, nf_h;
  std::vector<int> rleaf_start;  // row clusters of the tree's leaves (sorted starts + n_rows)
  // streamed payloads: per-wave packing of converged low-rank blocks into
  // device U / V arenas (growable), optional D2H into caller host arenas
  VPool uarena, varena;
  unsigned char *emitted = nullptr, *emit_flag = nullptr;
  int *emit_list = nullptr, *emit_cnt = nullptr;
  longlong2 *emit_need = nullptr, *emit_scan = nullptr;
  long long *blk_uoff = nullptr, *blk_voff = nullptr, *q_uoff = nullptr, *q_voff = nullptr;
  void *emit_tmp = nullptr;
  size_t emit_tmp_bytes = 0;
  long long u_top = 0, v_top = 0;
  bool packed = false;  // U / V arenas hold the current factors
  bool streaming() const { return out_u || out_v || out_dense; }
  void *out_u = nullptr, *out_v = nullptr, *out_dense = nullptr;
  void *zc_u = nullptr, *zc_v = nullptr;  // device views of out_u / out_v (zero-copy)
  long long out_u_cap = 0, out_v_cap = 0, out_dense_cap = 0;
  cudaStream_t cp = nullptr;    // factor packing + D2H, middle priority
  cudaStream_t cpd = nullptr;   // dense-arena D2H (waits for the near field)
  cudaEvent_t emit_ev = nullptr;
  cudaEvent_t tab_done = nullptr;  // singular table complete (side stream)
  cudaStream_t side = nullptr;  // near-field leaves, lowest priority
  cudaStream_t hi = nullptr;    // ACA waves, highest priority
  cudaEvent_t side_done = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t iev[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // integration launches
  bool int_pending[2] = {false, false};
  std::vector<void *> dev_allocs;
  std::vector<void *> exec_allocs;  // per-execute scratch
  hbem_hmat_stats stats{};
  double setup_s = 0.0;
  ~hbem_hmat() {
    cudaSetDevice(device);
    for (void *p : dev_allocs) cudaFree(p);
    for (void *p : exec_allocs) cudaFree(p);
    cudaFree(dense_nf);
    cudaFree(dense_adm);
    cudaFree(partA);
    cudaFree(partC);
    cudaFree(rsc);
    cudaFree(mv_buf);
    cudaFree(mv_ad);
    cudaFree(mv_ad_l);
    cudaFree(mv_items);
    cudaFree(mv_sbase);
    cudaFree(mv_s);
    cudaFree(mv_part); cudaFree(mv_dpart);
    cudaFree(mv_ifirst); cudaFree(mv_ibase); cudaFree(mv_rbase);
    cudaFree(mv_cstart); cudaFree(mv_cptr); cudaFree(mv_cover);
    if (mail) cudaFreeHost(mail);
    if (side) cudaStreamDestroy(side);
    if (hi) cudaStreamDestroy(hi);
    if (cp) cudaStreamDestroy(cp);
    if (cpd) cudaStreamDestroy(cpd);
    if (emit_ev) cudaEventDestroy(emit_ev);
    if (tab_done) cudaEventDestroy(tab_done);
    if (side_done) cudaEventDestroy(side_done);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    for (auto &pr : iev)
      for (auto e : pr)
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

// per-execute scratch: released at the start of the next execute / destroy
template <typename X> int dalloc_tmp(hbem_hmat *H, X **p, size_t n) {
  void *q = nullptr;
  cudaError_t e = cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(X));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(HBEM_ERR_CAPACITY, "device allocation of %zu bytes failed: %s",
                     n * sizeof(X), cudaGetErrorString(e));
  }
  H->exec_allocs.push_back(q);
  *p = static_cast<X *>(q);
  return HBEM_OK;
}
template <typename X> int upload_tmp(hbem_hmat *H, X **p, const std::vector<X> &v) {
  HB_CHECK(dalloc_tmp(H, p, v.size()));
  if (!v.empty()) HB_CUDA(cudaMemcpy(*p, v.data(), v.size() * sizeof(X), cudaMemcpyHostToDevice));
  return HBEM_OK;
}

template <typename X> int upload(hbem_hmat *H, X **p, const std::vector<X> &v) {
  HB_CHECK(dalloc(H, p, v.size()));
  if (!v.empty()) HB_CUDA(cudaMemcpy(*p, v.data(), v.size() * sizeof(X), cudaMemcpyHostToDevice));
  return HBEM_OK;
}

// grow-only device scratch; the old buffer is retired until the next execute
// (cudaFree would synchronise the device, stalling the payload copies)
int ensure(std::vector<void *> &retire, double **p, size_t *cap, size_t need) {
  if (need <= *cap) return HBEM_OK;
  if (*p) retire.push_back(*p);
  *p = nullptr;
  *cap = 0;
  const size_t n = std::max(need + need / 4, (size_t)1 << 16);
  cudaError_t e = cudaMalloc(p, n * sizeof(double));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(HBEM_ERR_CAPACITY, "device allocation of %zu partial-record bytes failed: %s",
                     n * sizeof(double), cudaGetErrorString(e));
  }
  *cap = n;
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
  P.G64p = H->g64p;
  P.nb_ptr = H->D.nb_ptr;
  P.nb_idx = H->D.nb_idx;
  P.stab = H->D.stab;
  P.elem = H->ctx->elem;
  P.rperm = H->rperm;
  P.cperm = H->cperm;
  P.tptr = H->tptr; P.tel = H->tel; P.tloc = H->tloc;
  P.sptr = H->sptr; P.sel = H->sel; P.sloc = H->sloc;
  P.trec = static_cast<const T *>(H->trec);
  P.srec = static_cast<const T *>(H->srec);
  return P;
}

// one-time: partition / DOF maps / ACA state / pools on the device
// HBEM_TRACE=1: per-stage wall times of setup on stderr
struct Trace {
  bool on = std::getenv("HBEM_TRACE") != nullptr;
  clk::time_point t = clk::now();
  void mark(const char *what) {
    if (!on) return;
    cudaDeviceSynchronize();
    const auto n = clk::now();
    std::fprintf(stderr, "[hbem setup] %-28s %8.3f s\n", what, secs(t, n));
    t = n;
  }
};

int setup(hbem_hmat *H, const hbem_hmat_desc *d) {
  Trace tr;
  hbem_ctx *ctx = H->ctx;
  const int64_t m = ctx->m;
  const int nt = ctx->nt, ns = ctx->ns;
  H->nt = nt;
  H->ns = ns;
  H->p0 = nt == 1 && ns == 1;
  H->n_rows = (int)d->n_rows;
  H->n_cols = (int)d->n_cols;
  {
    std::vector<int> rp(d->n_rows), cp(d->n_cols);
    for (int64_t i = 0; i < d->n_rows; ++i) rp[i] = (int)d->row_perm[i];
    for (int64_t i = 0; i < d->n_cols; ++i) cp[i] = (int)d->col_perm[i];
    int *a, *b;
    HB_CHECK(upload(H, &a, rp));
    H->same_tree = rp == cp;
    if (H->same_tree) {
      b = a;
    } else {
      HB_CHECK(upload(H, &b, cp));
    }
    H->rperm = a;
    H->cperm = b;
  }
  if (H->p0) {
    const size_t rb = (size_t)ctx->real_bytes();
    const size_t L = ctx->precision == HBEM_DOUBLE ? RecLen<double>::value : RecLen<float>::value;
    char *t = nullptr, *s = nullptr;
    HB_CHECK(dalloc(H, &t, (size_t)H->n_rows * L * rb));
    if (H->same_tree) {
      s = t;
    } else {
      HB_CHECK(dalloc(H, &s, (size_t)H->n_cols * L * rb));
    }
    H->trec = t;
    H->srec = s;
  }
  Incidence tinc, sinc;  // host copies (linear spaces): element unions per cluster
  if (nt == 3) {
    Incidence I = incidence(d->test_dofmap, m, 3, d->n_rows);
    tinc = I;
    int *p, *e;
    signed char *l;
    HB_CHECK(upload(H, &p, I.ptr));
    HB_CHECK(upload(H, &e, I.el));
    HB_CHECK(upload(H, &l, I.loc));
    H->tptr = p; H->tel = e; H->tloc = l;
  }
  if (ns == 3) {
    Incidence I = incidence(d->trial_dofmap, m, 3, d->n_cols);
    sinc = I;
    int *p, *e;
    signed char *l;
    HB_CHECK(upload(H, &p, I.ptr));
    HB_CHECK(upload(H, &e, I.el));
    HB_CHECK(upload(H, &l, I.loc));
    H->sptr = p; H->sel = e; H->sloc = l;
  }
  const int64_t L = d->n_leaves;
  H->n_leaves = L;
  std::vector<long long> off_dense0(L, -1);  // near-field leaves: fixed offsets
  for (int64_t q = 0; q < L; ++q)
    (d->leaves[3 * q + 2] ? H->adm_leaf : H->den_leaf).push_back((int)q);
  auto rng = [&](const int64_t *nodes, int64_t n) {
    return std::pair<int, int>((int)nodes[5 * n], (int)(nodes[5 * n + 1] - nodes[5 * n]));
  };
  tr.mark("perms + records + incidence");
  // ---- admissible blocks --------------------------------------------------------
  const int na = (int)H->adm_leaf.size();
  H->na = na;
  H->ah.resize(na); H->aw.resize(na); H->ar0.resize(na); H->ac0.resize(na);
  std::vector<int> rnode(na), cnode(na);
  std::vector<long long> rmo(na), cmo(na);
  long long rmw = 0, cmw = 0, sum_hw = 0, max_items = 0;
  for (int q = 0; q < na; ++q) {
    const int64_t lf = H->adm_leaf[q];
    rnode[q] = (int)d->leaves[3 * lf];
    cnode[q] = (int)d->leaves[3 * lf + 1];
    auto [r0, h] = rng(d->row_nodes, rnode[q]);
    auto [c0, w] = rng(d->col_nodes, cnode[q]);
    H->ar0[q] = r0; H->ah[q] = h; H->ac0[q] = c0; H->aw[q] = w;
    rmo[q] = rmw; rmw += (h + 31) / 32;
    cmo[q] = cmw; cmw += (w + 31) / 32;
    sum_hw += h + w;
    max_items += std::max(tiles_of(h), tiles_of(w));
  }
  H->items_cap = std::max<long long>(max_items, 1);
  // ---- linear spaces: sorted element union per cluster node (row and column
  // tree), the varying side of the element-level ACA rows (k_p1_erow)
  H->use_erows = !H->p0 && ctx->op != HBEM_HYPS;
  if (H->use_erows) {
    auto unions = [&](const int64_t *nodes, int64_t n_nodes, const int64_t *perm,
                      const Incidence &inc, bool single, long long **dptr, int **del,
                      long long &tiles) -> int {
      std::vector<long long> ptr(n_nodes + 1, 0);
      std::vector<std::vector<int>> lists(n_nodes);
      // bottom-up where children follow their parent, direct otherwise
      for (int64_t q = n_nodes - 1; q >= 0; --q) {
        const int64_t l = nodes[5 * q + 3], r = nodes[5 * q + 4];
        std::vector<int> &E = lists[q];
        if (l > q && r > q && l < n_nodes && r < n_nodes) {
          E.resize(lists[l].size() + lists[r].size());
          auto it = std::set_union(lists[l].begin(), lists[l].end(), lists[r].begin(),
                                   lists[r].end(), E.begin());
          E.resize(it - E.begin());
        } else {
          for (int64_t tp = nodes[5 * q]; tp < nodes[5 * q + 1]; ++tp) {
            const int64_t dof = perm[tp];
            if (single) {
              E.push_back((int)dof);
            } else {
              for (int k = inc.ptr[dof]; k < inc.ptr[dof + 1]; ++k) E.push_back(inc.el[k]);
            }
          }
          std::sort(E.begin(), E.end());
          E.erase(std::unique(E.begin(), E.end()), E.end());
        }
      }
      for (int64_t q = 0; q < n_nodes; ++q) {
        ptr[q + 1] = ptr[q] + (long long)lists[q].size();
        tiles += ((long long)lists[q].size() + 31) / 32;
      }
      std::vector<int> flat(ptr[n_nodes]);
      for (int64_t q = 0; q < n_nodes; ++q)
        std::copy(lists[q].begin(), lists[q].end(), flat.begin() + ptr[q]);
      HB_CHECK(upload(H, dptr, ptr));
      HB_CHECK(upload(H, del, flat));
      return HBEM_OK;
    };
    long long et = 0;
    long long *rp = nullptr, *cpp = nullptr;
    int *re = nullptr, *ce = nullptr;
    HB_CHECK(unions(d->row_nodes, d->n_row_nodes, d->row_perm, tinc, nt == 1, &rp, &re, et));
    if (H->same_tree && nt == ns) {
      cpp = rp;
      ce = re;
      et *= 2;
    } else {
      HB_CHECK(unions(d->col_nodes, d->n_col_nodes, d->col_perm, sinc, ns == 1, &cpp, &ce, et));
    }
    H->S.recl_ptr = rp;
    H->S.recl = re;
    H->S.cecl_ptr = cpp;
    H->S.cecl = ce;
    H->eitems_cap = std::max<long long>(et, 1);
  }
  AcaDev &S = H->S;
  if (d->rank_capacity > (1 << 16))
    return set_error(HBEM_ERR_CONFIG, "rank_capacity %lld exceeds %d",
                     (long long)d->rank_capacity, 1 << 16);
  S.tmax = d->rank_capacity > 0 ? (int)d->rank_capacity : 64;
  S.kmax_cfg = d->k_max > 0 ? (int)std::min<int64_t>(d->k_max, 1 << 30) : (1 << 30);
  S.eps = d->epsilon;
  {
    int *p;
    HB_CHECK(upload(H, &p, H->ah)); S.h = p;
    HB_CHECK(upload(H, &p, H->aw)); S.w = p;
    HB_CHECK(upload(H, &p, H->ar0)); S.r0 = p;
    HB_CHECK(upload(H, &p, H->ac0)); S.c0 = p;
    HB_CHECK(upload(H, &p, rnode)); S.rnode = p;
    HB_CHECK(upload(H, &p, cnode)); S.cnode = p;
    long long *pl;
    HB_CHECK(upload(H, &pl, rmo)); S.rmask_off = pl;
    HB_CHECK(upload(H, &pl, cmo)); S.cmask_off = pl;
    {
      std::vector<BlockInfo> bi((size_t)na);
      for (int q = 0; q < na; ++q)
        bi[(size_t)q] = BlockInfo{H->ah[q], H->aw[q], H->ar0[q], H->ac0[q], rnode[q], cnode[q],
                                  rmo[q], cmo[q]};
      BlockInfo *pb;
      HB_CHECK(upload(H, &pb, bi));
      S.binfo = pb;
    }
    // static phase orders: row jobs grouped by column cluster, column jobs
    // by row cluster, ties by block index (counting sort: deterministic lists)
    auto by_key = [&](const std::vector<int> &key, int64_t n_keys) {
      std::vector<int> cnt(n_keys + 1, 0), order(na);
      for (int q = 0; q < na; ++q) cnt[key[q] + 1]++;
      for (int64_t k = 0; k < n_keys; ++k) cnt[k + 1] += cnt[k];
      for (int q = 0; q < na; ++q) order[cnt[key[q]]++] = q;
      return order;
    };
    HB_CHECK(upload(H, &H->row_order, by_key(cnode, d->n_col_nodes)));
    HB_CHECK(upload(H, &H->col_order, by_key(rnode, d->n_row_nodes)));
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
  HB_CHECK(dalloc(H, &S.rowpart, na));
  HB_CHECK(dalloc(H, &S.rsum, (size_t)na * kFinRegs * 2));
  HB_CHECK(dalloc(H, &S.terms, (size_t)na * S.tmax));
  HB_CHECK(dalloc(H, (char **)&S.tpiv, (size_t)na * S.tmax * H->vbytes));
  HB_CHECK(dalloc(H, &S.rmask, rmw));
  HB_CHECK(dalloc(H, &S.cmask, cmw));
  HB_CHECK(dalloc(H, &S.flagA, na));
  HB_CHECK(dalloc(H, &S.flagC, na));
  HB_CHECK(dalloc(H, &H->sel_tmp, (na + 3) / 4));
  HB_CHECK(dalloc(H, &H->listA, na));
  HB_CHECK(dalloc(H, &H->listC, na));
  HB_CHECK(dalloc(H, &H->d_cnt, 1));
  HB_CHECK(dalloc(H, &S.need, na));
  HB_CHECK(dalloc(H, &S.pkey, na));
  HB_CHECK(dalloc(H, &S.scan, na));
  HB_CHECK(dalloc(H, &S.jobs, na));
  HB_CHECK(dalloc(H, &S.jt, (size_t)na * kFinRegs));
  HB_CHECK(dalloc(H, (char **)&S.jc, (size_t)na * kFinRegs * H->vbytes));
  HB_CHECK(dalloc(H, &S.items, H->items_cap));
  HB_CHECK(dalloc(H, &S.iglen, H->items_cap));
  if (H->p0) HB_CHECK(dalloc(H, (char **)&S.stage, (size_t)na * kStageRecMax));
  if (H->use_erows) HB_CHECK(dalloc(H, &S.eitems, H->eitems_cap));
  HB_CHECK(dalloc(H, &S.stat, 16));  // [0..1] counters, [4..] HB_PROF phase cycles
  H->cub_bytes = aca_cub_bytes(na);
  HB_CHECK(dalloc(H, (char **)&H->cub_tmp, H->cub_bytes));
  HB_CUDA(cudaMallocHost(&H->mail, sizeof(hbem_hmat::Mail)));
  HB_CUDA(cudaHostGetDevicePointer((void **)&H->mail_dev, H->mail, 0));
  tr.mark("admissible blocks");
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
    off_dense0[lf] = tot;
    tot += (long long)h * w;
  }
  H->nf_r0 = dr0;
  H->nf_c0 = dc0;
  H->nf_h = dh;
  {
    // row clusters of the row tree's leaves (they partition [0, n_rows))
    std::vector<int> st;
    for (int64_t q = 0; q < d->n_row_nodes; ++q)
      if (d->row_nodes[5 * q + 3] < 0) st.push_back((int)d->row_nodes[5 * q]);
    std::sort(st.begin(), st.end());
    st.push_back(H->n_rows);
    H->rleaf_start = st;
  }
  H->nf_entries = tot;
  {
    std::vector<long long> rb(nd);
    long long acc = 0;
    for (int q = 0; q < nd; ++q) { rb[q] = acc; acc += dh[q]; }
    H->nf_rows = acc;
    long long *p;
    HB_CHECK(upload(H, &p, rb));
    H->nf_rowbase = p;
  }
  {
    DenseDev &D = H->D;
    int *p;
    long long *pl;
    HB_CHECK(upload(H, &p, dr0)); D.r0 = p;
    HB_CHECK(upload(H, &p, dc0)); D.c0 = p;
    HB_CHECK(upload(H, &p, dh)); D.h = p;
    HB_CHECK(upload(H, &p, dw)); D.w = p;
    HB_CHECK(upload(H, &pl, doff)); D.off = pl;
    HB_CHECK(dalloc(H, &D.sing_count, 1));
    HB_CHECK(dalloc(H, &D.stat, 2));
    if ((H->p0 && nd > 0) || !H->p0) {
      // touching element pairs integrated once per execute into a table the
      // near-field kernel reads (single layer: each unordered pair once)
      SingTable tab;
      tr.mark("near-field arrays");
      // symmetric operators on equal spaces: S(f, e) = S(e, f)^T bit for bit
      // (canonical orientation, kernels.py:340-344), one integration per pair
      const bool sym = (ctx->op == HBEM_SLP || ctx->op == HBEM_HYPS) && nt == ns &&
                       ctx->test_family == ctx->trial_family;
      HB_CHECK(build_sing_table(ctx->elem, (int)m, (int)ctx->nv, sym, tab, H->dev_allocs, 0));
      if (H->p0) {
        // only the touching pairs of this handle's near-field leaves (the
        // admissible leaves' rare touching pairs are integrated in place by
        // k_aca_p0): a multi-GPU split shards the singular work too
        std::vector<int> cinv((size_t)m, -1);
        for (int64_t i = 0; i < d->n_cols; ++i) cinv[(size_t)d->col_perm[i]] = (int)i;
        int *dci;
        HB_CHECK(upload(H, &dci, cinv));
        HB_CHECK(restrict_sing_pairs(tab, H->rperm, dci, H->nf_rowbase, nd, H->nf_rows, D.r0,
                                     D.c0, D.w, H->dev_allocs, 0));
      }
      if (H->p0 && sym) HB_CHECK(sort_sing_pairs(tab, ctx->elem, H->dev_allocs, 0));
      D.skind[0] = 0;
      for (int c = 1; c < 4; ++c) D.skind[c] = D.skind[c - 1] + tab.kind_n[c];
      H->sing_pairs_table = tab.n_pairs;
      D.nb_ptr = tab.nb_ptr;
      D.nb_idx = tab.nb_idx;
      D.spairs = tab.pairs;
      D.n_spairs = tab.n_pairs;
      char *st_vals = nullptr;
      HB_CHECK(dalloc(H, &st_vals, (size_t)tab.nnz * nt * ns * H->vbytes));
      D.stab = st_vals;
      tr.mark("singular table topology");
    }
    if (H->p0) {
      // warp items (leaf, 32-column tile); touching pairs read from the table
      std::vector<int2> items;
      for (int s = 0; s < nd; ++s)
        for (int t = 0; t < tiles_of(dw[s]); ++t) items.push_back(make_int2(s, t));
      int2 *pi;
      HB_CHECK(upload(H, &pi, items));
      D.items = pi;
      D.n_items = (long long)items.size();
    } else {
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
      HB_CHECK(upload(H, &p, tslot)); D.tile_slot = p;
      HB_CHECK(upload(H, &p, tstart)); D.tile_start = p;
    }
  }
  {
    // per-leaf metadata on the device: near-field leaves are dense, rank 0
    LeafMeta &M = H->meta;
    HB_CHECK(dalloc(H, &M.kind, (size_t)std::max<int64_t>(3 * L, 1)));
    M.rank = M.kind + L;
    M.flags = M.kind + 2 * L;
    HB_CHECK(dalloc(H, &M.off_u, (size_t)std::max<int64_t>(3 * L, 1)));
    M.off_v = M.off_u + L;
    M.off_d = M.off_u + 2 * L;
    HB_CHECK(dalloc(H, &M.resid, (size_t)std::max<int64_t>(L, 1)));
    HB_CUDA(cudaMemset(M.resid, 0, (size_t)std::max<int64_t>(L, 1) * 8));
    HB_CUDA(cudaMemset(M.kind, 0, (size_t)3 * L * 4));
    HB_CUDA(cudaMemset(M.off_u, 0xff, (size_t)2 * L * 8));
    HB_CUDA(cudaMemcpy(M.off_d, off_dense0.data(), (size_t)L * 8, cudaMemcpyHostToDevice));
    HB_CHECK(upload(H, &H->d_adm_leaf, H->adm_leaf));
    HB_CHECK(dalloc(H, &H->lr_list, std::max(na, 1)));
    HB_CHECK(dalloc(H, &H->dn_list, std::max(na, 1)));
    HB_CHECK(dalloc(H, &H->cls_cnt, 2));
    HB_CHECK(dalloc(H, &H->cls_flag, (size_t)2 * std::max(na, 1)));
    HB_CHECK(dalloc(H, &H->cls_stat, 1));
    HB_CHECK(dalloc(H, &H->dn_info, std::max(na, 1)));
  }
  const size_t vb = H->vbytes;
  HB_CUDA(cudaMalloc(&H->dense_nf, std::max<size_t>((size_t)tot * vb, vb)));
  H->D.out = H->dense_nf;
  tr.mark("near-field leaves");
  // ---- factor pool: virtual range of the free memory, mapped on demand
  size_t free_b = 0, total_b = 0;
  {
    Geo64 g = ctx->geo64();
    HB_CHECK(dalloc(H, &H->g64p, 1));
    HB_CUDA(cudaMemcpy(H->g64p, &g, sizeof(Geo64), cudaMemcpyHostToDevice));
  }
  HB_CUDA(cudaFree(nullptr));
  HB_CUDA(cudaMemGetInfo(&free_b, &total_b));
  HB_CHECK(H->vpool.init(H->device, std::max<size_t>(free_b, (size_t)4 << 30)));
  (void)sum_hw;
  tr.mark("factor pool");
  S.pool = reinterpret_cast<void *>(H->vpool.base);
  S.pool_cap = (long long)(H->vpool.reserved / vb);
  {
    // the ACA waves (latency-bound finalize phases, host reads between
    // phases) run on a high-priority stream; the compute-bound near-field
    // leaves on a low-priority stream fill the gaps
    int least = 0, greatest = 0;
    HB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    HB_CUDA(cudaStreamCreateWithPriority(&H->side, cudaStreamNonBlocking, least));
    HB_CUDA(cudaStreamCreateWithPriority(&H->hi, cudaStreamNonBlocking, greatest));
    // payload packing between the two: ahead of the near field so the PCIe
    // copies start while the ACA waves still run
    HB_CUDA(cudaStreamCreateWithPriority(&H->cp, cudaStreamNonBlocking,
                                         greatest < least ? greatest + 1 : least));
    HB_CUDA(cudaStreamCreateWithPriority(&H->cpd, cudaStreamNonBlocking, least));
    HB_CUDA(cudaEventCreateWithFlags(&H->emit_ev, cudaEventDisableTiming));
    HB_CUDA(cudaEventCreateWithFlags(&H->tab_done, cudaEventDisableTiming));
  }
  // streamed payload arenas (virtual ranges, mapped as blocks converge)
  HB_CHECK(H->uarena.init(H->device, std::max<size_t>(free_b / 2, (size_t)4 << 30)));
  HB_CHECK(H->varena.init(H->device, std::max<size_t>(free_b / 2, (size_t)4 << 30)));
  HB_CHECK(dalloc(H, &H->emitted, std::max(na, 1)));
  HB_CHECK(dalloc(H, &H->emit_flag, std::max(na, 1)));
  HB_CHECK(dalloc(H, &H->emit_list, std::max(na, 1)));
  HB_CHECK(dalloc(H, &H->emit_cnt, 1));
  HB_CHECK(dalloc(H, &H->emit_need, std::max(na, 1)));
  HB_CHECK(dalloc(H, &H->emit_scan, std::max(na, 1)));
  HB_CHECK(dalloc(H, &H->blk_uoff, std::max(na, 1)));
  HB_CHECK(dalloc(H, &H->blk_voff, std::max(na, 1)));
  HB_CHECK(dalloc(H, &H->q_uoff, std::max(na, 1)));
  HB_CHECK(dalloc(H, &H->q_voff, std::max(na, 1)));
  {
    size_t b1 = 0, b2 = 0;
    cub::DeviceSelect::Flagged(nullptr, b1, cub::CountingInputIterator<int>(0),
                               (const unsigned char *)nullptr, (int *)nullptr, (int *)nullptr,
                               std::max(na, 1));
    cub::DeviceScan::InclusiveScan(nullptr, b2, (const longlong2 *)nullptr, (longlong2 *)nullptr,
                                   SumLL2(), std::max(na, 1));
    H->emit_tmp_bytes = std::max(b1, b2);
    HB_CHECK(dalloc(H, (char **)&H->emit_tmp, H->emit_tmp_bytes));
  }
  H->out_u = d->out_u;
  H->out_v = d->out_v;
  H->out_dense = d->out_dense;
  H->out_u_cap = d->out_u_cap;
  H->out_v_cap = d->out_v_cap;
  H->out_dense_cap = d->out_dense_cap;
  {
    // page-locked U / V arenas are device-addressable: with HBEM_ZEROCOPY=1
    // the emission kernel writes them directly over PCIe (no device staging
    // arena, 56 GB less HBM at C5); the default stages the packed factors in
    // HBM and moves them with the copy engine, which sustains the PCIe rate
    // without taking SM slots from the ACA waves
    const char *zc_env = std::getenv("HBEM_ZEROCOPY");
    if (H->out_u && H->out_v && zc_env && zc_env[0] == '1') {
      void *pu = nullptr, *pv = nullptr;
      if (cudaHostGetDevicePointer(&pu, H->out_u, 0) == cudaSuccess &&
          cudaHostGetDevicePointer(&pv, H->out_v, 0) == cudaSuccess) {
        H->zc_u = pu;
        H->zc_v = pv;
      }
      cudaGetLastError();
    }
  }
  HB_CUDA(cudaEventCreateWithFlags(&H->side_done, cudaEventDisableTiming));
  for (auto &e : H->ev) HB_CUDA(cudaEventCreate(&e));
  for (auto &pr : H->iev)
    for (auto &e : pr) HB_CUDA(cudaEventCreate(&e));
  return HBEM_OK;
}

// one phase of one wave: select + scan, one host read, jobs/items/integrate/finalize
template <typename T, bool C>
int run_phase(hbem_hmat *H, const Prob<T> &P, int col, long long &pool_top, int wave, int *n_out,
              cudaStream_t st) {
  hbem_ctx *ctx = H->ctx;
  AcaDev &S = H->S;
  PhaseArgs A{};
  A.na = H->na;
  A.col_phase = col;
  A.order = col ? H->col_order : H->row_order;
  A.cub_tmp = H->cub_tmp;
  A.cub_bytes = H->cub_bytes;
  A.sel_tmp = H->sel_tmp;
  A.nt = H->nt;
  A.ns = H->ns;
  S.list = col ? H->listC : H->listA;
  S.nlist = H->d_cnt;
  HB_CHECK((aca_select<T, C>(P, S, A, st)));
  // grand total of the needs: k_need_blocks leaves it behind the block totals
  const Need *need_tot =
      reinterpret_cast<const Need *>(H->cub_tmp) + (H->na + kNeedThreads - 1) / kNeedThreads;
  HB_CHECK(H->read_mail(st, {{&H->mail->tot, need_tot, sizeof(Need)},
                             {&H->mail->n, H->d_cnt, sizeof(int)}}));
  const Need tot = H->mail->tot;
  const int n = H->mail->n;
  *n_out = n;
  if (n == 0) return HBEM_OK;
  if (!col) {
    // kPoolSlack: the integration kernel's bulk copies of 32-entry factor
    // tiles may read up to one 16-byte granule past the last record
    if (pool_top + tot.pool + kPoolSlack > S.pool_cap)
      return set_error(HBEM_ERR_CAPACITY,
                       "ACA factor pool of %lld values exhausted at wave %d (need %lld more)",
                       (long long)S.pool_cap, wave,
                       (long long)(pool_top + tot.pool + kPoolSlack - S.pool_cap));
    HB_CHECK(H->vpool.grow((size_t)(pool_top + tot.pool + kPoolSlack) * H->vbytes));
    S.pool_base = pool_top;
    pool_top += tot.pool;
  }
  if (tot.items > H->items_cap)
    return set_error(HBEM_ERR_CAPACITY, "ACA item table overflow (%lld > %lld)",
                     (long long)tot.items, (long long)H->items_cap);
  if (col) {
    HB_CHECK(ensure(H->exec_allocs, &H->partC, &H->partC_cap, (size_t)tot.part));
    S.part = H->partC;
    S.rpart = H->partA;
  } else {
    HB_CHECK(ensure(H->exec_allocs, &H->partA, &H->partA_cap, (size_t)tot.part));
    S.part = H->partA;
  }
  A.int_beg = H->iev[col][0];
  A.int_end = H->iev[col][1];
  H->int_pending[col] = tot.items > 0;
  S.rsc = nullptr;
  if (H->use_erows) {
    if (tot.eitems > H->eitems_cap)
      return set_error(HBEM_ERR_CAPACITY, "element item table overflow (%lld > %lld)",
                       (long long)tot.eitems, (long long)H->eitems_cap);
    const size_t need = (size_t)std::max<long long>(tot.rsc, 1) * H->vbytes;
    if (need > H->rsc_cap) {
      if (H->rsc) H->exec_allocs.push_back(H->rsc);
      H->rsc = nullptr;
      const size_t cap = need + need / 4;
      cudaError_t e = cudaMalloc(&H->rsc, cap);
      if (e != cudaSuccess) {
        cudaGetLastError();
        H->rsc_cap = 0;
        return set_error(HBEM_ERR_CAPACITY, "element-row scratch of %zu bytes: %s", cap,
                         cudaGetErrorString(e));
      }
      H->rsc_cap = cap;
    }
    S.rsc = H->rsc;
  }
  return aca_phase<T, C>(P, S, A, ctx->op, ctx->helm, H->nt, H->ns, n, tot.items, tot.eitems, st);
}

// pack the low-rank blocks converged since the last call into the device
// U / V arenas (cp stream, low priority) and stream them into the caller's
// host arenas when given; one host read per call
template <typename T, bool C> int emit_converged(hbem_hmat *H, cudaStream_t st, bool pack = true) {
  using V = typename Num<T, C>::V;
  const int na = H->na;
  if (na <= 0) return HBEM_OK;
  AcaDev &S = H->S;
  k_emit_flags<<<(na + 255) / 256, 256, 0, st>>>(S, na, H->emitted, H->emit_flag);
  size_t tb = H->emit_tmp_bytes;
  HB_CUDA(cub::DeviceSelect::Flagged(H->emit_tmp, tb, cub::CountingInputIterator<int>(0),
                                     H->emit_flag, H->emit_list, H->emit_cnt, na, st));
  k_emit_need<<<(na + 255) / 256, 256, 0, st>>>(S, H->emit_list, H->emit_cnt, na, H->emit_need);
  tb = H->emit_tmp_bytes;
  HB_CUDA(cub::DeviceScan::InclusiveScan(H->emit_tmp, tb, H->emit_need, H->emit_scan, SumLL2(),
                                         na, st));
  HB_CHECK(H->read_mail(st, {{&H->mail->tot, H->emit_scan + (na - 1), sizeof(longlong2)},
                             {&H->mail->n, H->emit_cnt, sizeof(int)}}));
  const int n = H->mail->n;
  const longlong2 tot = *reinterpret_cast<const longlong2 *>(&H->mail->tot);
  if (n == 0) return HBEM_OK;
  const size_t vb = sizeof(V);
  const bool zc = pack && H->zc_u && H->zc_v;
  if (pack && !zc) {
    HB_CHECK(H->uarena.grow((size_t)(H->u_top + tot.x) * vb));
    HB_CHECK(H->varena.grow((size_t)(H->v_top + tot.y) * vb));
  }
  if (H->out_u && H->u_top + tot.x > H->out_u_cap)
    return set_error(HBEM_ERR_CAPACITY, "host U arena of %lld values too small",
                     (long long)H->out_u_cap);
  if (H->out_v && H->v_top + tot.y > H->out_v_cap)
    return set_error(HBEM_ERR_CAPACITY, "host V arena of %lld values too small",
                     (long long)H->out_v_cap);
  k_emit_offsets<<<(n + 255) / 256, 256, 0, st>>>(H->emit_list, n, H->emit_scan, H->emit_need,
                                                  H->u_top, H->v_top, H->blk_uoff, H->blk_voff,
                                                  H->q_uoff, H->q_voff);
  if (!pack) {
    H->u_top += tot.x;
    H->v_top += tot.y;
    return HBEM_OK;
  }
  HB_CUDA(cudaEventRecord(H->emit_ev, st));
  HB_CUDA(cudaStreamWaitEvent(H->cp, H->emit_ev, 0));
  // the emission list is rebuilt next wave: the pack reads a private copy
  int *lst = nullptr;
  long long *uo = nullptr, *vo = nullptr;
  HB_CHECK(dalloc_tmp(H, &lst, (size_t)n));
  HB_CHECK(dalloc_tmp(H, &uo, (size_t)n));
  HB_CHECK(dalloc_tmp(H, &vo, (size_t)n));
  HB_CUDA(cudaMemcpyAsync(lst, H->emit_list, (size_t)n * 4, cudaMemcpyDeviceToDevice, H->cp));
  HB_CUDA(cudaMemcpyAsync(uo, H->q_uoff, (size_t)n * 8, cudaMemcpyDeviceToDevice, H->cp));
  HB_CUDA(cudaMemcpyAsync(vo, H->q_voff, (size_t)n * 8, cudaMemcpyDeviceToDevice, H->cp));
  if (zc) {
    k_pack_host<T, C><<<std::min((n + 7) / 8, 64), 256, 0, H->cp>>>(
        lst, n, S, uo, vo, static_cast<V *>(H->zc_u), static_cast<V *>(H->zc_v));
    HB_CUDA(cudaGetLastError());
    H->u_top += tot.x;
    H->v_top += tot.y;
    return HBEM_OK;
  }
  V *ua = reinterpret_cast<V *>(H->uarena.base), *va = reinterpret_cast<V *>(H->varena.base);
  k_pack_factors<T, C><<<n, 128, 0, H->cp>>>(lst, n, S, uo, vo, 0, 0, ua, va);
  HB_CUDA(cudaGetLastError());
  if (H->out_u)
    HB_CUDA(cudaMemcpyAsync(static_cast<V *>(H->out_u) + H->u_top, ua + H->u_top,
                            (size_t)tot.x * vb, cudaMemcpyDeviceToHost, H->cp));
  if (H->out_v)
    HB_CUDA(cudaMemcpyAsync(static_cast<V *>(H->out_v) + H->v_top, va + H->v_top,
                            (size_t)tot.y * vb, cudaMemcpyDeviceToHost, H->cp));
  H->u_top += tot.x;
  H->v_top += tot.y;
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
  for (void *p : H->exec_allocs) cudaFree(p);
  H->exec_allocs.clear();
  H->u_top = H->v_top = 0;
  if (na > 0) {
    HB_CUDA(cudaMemsetAsync(H->emitted, 0, na, st));
    HB_CUDA(cudaMemsetAsync(H->blk_uoff, 0xff, (size_t)na * 8, st));
    HB_CUDA(cudaMemsetAsync(H->blk_voff, 0xff, (size_t)na * 8, st));
  }
  // ---- tree-ordered element records (P0) -------------------------------------------
  if (H->p0) {
    HB_CHECK(build_recs<T>(P.g, ctx->elem, H->rperm, H->n_rows, static_cast<T *>(H->trec), st));
    ++launches;
    if (!H->same_tree) {
      HB_CHECK(build_recs<T>(P.g, ctx->elem, H->cperm, H->n_cols, static_cast<T *>(H->srec), st));
      ++launches;
    }
  }
  // ---- near-field leaves on the side stream (overlaps the ACA waves) ---------
  cudaEvent_t start_ev;
  HB_CUDA(cudaEventCreateWithFlags(&start_ev, cudaEventDisableTiming));
  HB_CUDA(cudaEventRecord(start_ev, st));
  HB_CUDA(cudaStreamWaitEvent(H->side, start_ev, 0));
  cudaEventDestroy(start_ev);
  HB_CUDA(cudaEventRecord(H->ev[2], H->side));
  const bool skip_nf = std::getenv("HBEM_SKIP_NEARFIELD") != nullptr;  // timing experiments only
  if (H->D.n_spairs > 0 && !skip_nf) {
    HB_CHECK((sing_table_launch<T, C>(P, H->D, ctx->op, ctx->helm, nt, ns, H->side)));
    ++launches;
  }
  HB_CUDA(cudaEventRecord(H->tab_done, H->side));
  if (!H->p0) HB_CUDA(cudaStreamWaitEvent(st, H->tab_done, 0));  // k_aca_gen reads the table
  if (H->nd > 0 && !skip_nf) {
    HB_CUDA(cudaMemsetAsync(H->D.sing_count, 0, 8, H->side));
    HB_CUDA(cudaMemsetAsync(H->D.stat, 0, 16, H->side));
    if (H->p0) {
      HB_CHECK((near_p0_launch<T, C>(P, H->D, ctx->op, ctx->helm, H->side)));
      launches += 1;
    } else {
      int rc = dispatch_op(ctx->op, ctx->helm, nt, ns, [&](auto OPc, auto Hc, auto NTc,
                                                           auto NSc) -> int {
        constexpr int OP = decltype(OPc)::value;
        constexpr bool HH = decltype(Hc)::value != 0;
        constexpr int NT = decltype(NTc)::value, NS = decltype(NSc)::value;
        if constexpr (HH == C) {
          k_dense<T, C, OP, HH, NT, NS><<<H->n_tiles, kThreads, 0, H->side>>>(P, H->D);
          HB_CUDA(cudaGetLastError());
          return HBEM_OK;
        } else {
          return set_error(HBEM_ERR_KERNEL, "value type does not match the equation");
        }
      });
      if (rc != HBEM_OK) return rc;
      ++launches;
    }
  }
  HB_CUDA(cudaEventRecord(H->side_done, H->side));
  HB_CUDA(cudaEventRecord(H->ev[3], H->side));
  if (H->out_dense && H->nf_entries > 0) {
    if (H->nf_entries > H->out_dense_cap)
      return set_error(HBEM_ERR_CAPACITY, "host dense arena of %lld values too small",
                       (long long)H->out_dense_cap);
    HB_CUDA(cudaStreamWaitEvent(H->cpd, H->side_done, 0));
    HB_CUDA(cudaMemcpyAsync(H->out_dense, H->dense_nf, (size_t)H->nf_entries * sizeof(V),
                            cudaMemcpyDeviceToHost, H->cpd));
  }
  // ---- ACA waves ------------------------------------------------------------------
  HB_CUDA(cudaMemsetAsync(S.stat, 0, 128, st));
  int waves = 0;
  long long pool_top = 0;
  // HBEM_TRACE: per-wave timeline (host clock, copy-stream completion)
  const bool wtrace = std::getenv("HBEM_TRACE") != nullptr;
  cudaEvent_t wt0 = nullptr;
  std::vector<cudaEvent_t> wcp;
  std::vector<double> whost;
  std::vector<long long> wbytes;
  if (wtrace) {
    HB_CUDA(cudaEventCreate(&wt0));
    HB_CUDA(cudaEventRecord(wt0, st));
  }
  if (na > 0) {
    HB_CHECK((aca_init<T, C>(P, S, na, st)));
    ++launches;
    for (;;) {
      HB_CUDA(cudaEventRecord(H->ev[0], st));
      int nA = 0, nC = 0;
      HB_CHECK((run_phase<T, C>(H, P, 0, pool_top, waves, &nA, st)));
      if (nA == 0) break;
      HB_CHECK((run_phase<T, C>(H, P, 1, pool_top, waves, &nC, st)));
      const long long top0 = H->u_top + H->v_top;
      if (H->streaming()) HB_CHECK((emit_converged<T, C>(H, st)));
      if (wtrace) {
        cudaEvent_t e;
        HB_CUDA(cudaEventCreate(&e));
        HB_CUDA(cudaEventRecord(e, H->streaming() ? H->cp : st));
        wcp.push_back(e);
        whost.push_back(secs(t0, clk::now()));
        wbytes.push_back((H->u_top + H->v_top - top0) * (long long)sizeof(V));
      }
      launches += (nC > 0 ? 10 : 7) + (H->streaming() ? 4 : 0);
      HB_CUDA(cudaEventRecord(H->ev[1], st));
      HB_CUDA(cudaEventSynchronize(H->ev[1]));
      float ms = 0.f;
      HB_CUDA(cudaEventElapsedTime(&ms, H->ev[0], H->ev[1]));
      ST.aca_kernel_ms += ms;
      for (int ph = 0; ph < 2; ++ph)
        if (H->int_pending[ph]) {
          float im = 0.f;
          HB_CUDA(cudaEventElapsedTime(&im, H->iev[ph][0], H->iev[ph][1]));
          ST.int_kernel_ms += im;
          ST.int_launches += 1;
          H->int_pending[ph] = false;
        }
      ST.row_jobs += nA;
      ST.col_jobs += nC;
      ++waves;
    }
  }
  if (!H->streaming() && na > 0) {
    // offsets of every low-rank block (block order); packing deferred to
    // hbem_hmat_copy_arenas (the device-resident H-matrix is the pool)
    HB_CHECK((emit_converged<T, C>(H, st, /*pack=*/false)));
  }
  // zero-copy emission leaves the device U / V arenas unpacked
  H->packed = H->streaming() && !(H->zc_u && H->zc_v);
  const auto t_aca = clk::now();
  // ---- classify admissible blocks (lowrank_leaf, hmatrix.py:721-735) -------------
  // on the device: per-leaf metadata in place, block-ordered low-rank and
  // dense lists, dense offsets by a scan; the host reads the counters and the
  // (short) dense list only
  std::vector<int> expand_slots, fb_r0, fb_c0, fb_h, fb_w;
  std::vector<long long> expand_off, fb_off;
  std::vector<int> fb_q;
  long long adm_dense = 0;
  H->n_lowrank = 0;
  if (na > 0) {
    const unsigned g = (unsigned)((na + 255) / 256);
    HB_CUDA(cudaMemsetAsync(H->cls_stat, 0, 16, st));
    HB_CUDA(cudaMemsetAsync(&H->cls_stat->overflow_q, 0x7f, 4, st));
    unsigned char *flr = H->cls_flag, *fdn = H->cls_flag + na;
    k_classify<<<g, 256, 0, st>>>(S, na, H->d_adm_leaf, H->blk_uoff, H->blk_voff, H->meta,
                                  H->emit_need, flr, fdn, H->cls_stat);
    size_t tb = H->emit_tmp_bytes;
    HB_CUDA(cub::DeviceScan::InclusiveScan(H->emit_tmp, tb, H->emit_need, H->emit_scan, SumLL2(),
                                           na, st));
    tb = H->emit_tmp_bytes;
    HB_CUDA(cub::DeviceSelect::Flagged(H->emit_tmp, tb, cub::CountingInputIterator<int>(0), flr,
                                       H->lr_list, H->cls_cnt, na, st));
    tb = H->emit_tmp_bytes;
    HB_CUDA(cub::DeviceSelect::Flagged(H->emit_tmp, tb, cub::CountingInputIterator<int>(0), fdn,
                                       H->dn_list, H->cls_cnt + 1, na, st));
    k_classify_dense<<<g, 256, 0, st>>>(H->dn_list, H->cls_cnt + 1, S, H->emit_scan,
                                        H->emit_need, H->d_adm_leaf, H->nf_entries, H->meta,
                                        H->dn_info);
    HB_CUDA(cudaGetLastError());
    launches += 6;
    auto *ml = H->mail;
    HB_CHECK(H->read_mail(st, {{ml->cls_cnt, H->cls_cnt, 8},
                               {&ml->cls, H->cls_stat, sizeof(ClsStat)},
                               {&ml->adm_dense, &H->emit_scan[na - 1].x, 8}}));
    if (ml->cls.overflow_q < na) {
      const int q = ml->cls.overflow_q;
      return set_error(HBEM_ERR_CAPACITY,
                       "ACA rank capacity %d exceeded for block rows [%d, %d) x cols [%d, %d); "
                       "raise rank_capacity",
                       S.tmax, H->ar0[q], H->ar0[q] + H->ah[q], H->ac0[q], H->ac0[q] + H->aw[q]);
    }
    H->n_lowrank = ml->cls_cnt[0];
    const int n_dn = ml->cls_cnt[1];
    adm_dense = ml->adm_dense;
    ST.aca_converged = (int64_t)ml->cls.converged;
    ST.aca_exhausted = (int64_t)ml->cls.exhausted;
    ST.lowrank_leaves = H->n_lowrank;
    std::vector<longlong2> info(n_dn);
    if (n_dn > 0)
      HB_CUDA(cudaMemcpy(info.data(), H->dn_info, (size_t)n_dn * sizeof(longlong2),
                         cudaMemcpyDeviceToHost));
    for (const longlong2 &r : info) {
      const int q = (int)(r.x & 0x7fffffffll);
      if (r.x >> 31) {  // converged, no compression: expanded from the factors
        expand_slots.push_back(q);
        expand_off.push_back(r.y);
      } else {          // ST_FALLBACK: rank cap without convergence -> exact rows
        ST.aca_fallback_dense++;
        fb_q.push_back(q);
        fb_r0.push_back(H->ar0[q]); fb_c0.push_back(H->ac0[q]);
        fb_h.push_back(H->ah[q]); fb_w.push_back(H->aw[q]);
        fb_off.push_back(r.y);
      }
    }
  }
  H->u_entries = H->u_top;
  H->v_entries = H->v_top;
  const auto t_cls = clk::now();
  ST.dense_leaves = H->nd + (int64_t)expand_slots.size() + (int64_t)fb_r0.size();
  H->ad_r0.clear(); H->ad_c0.clear(); H->ad_h.clear(); H->ad_w.clear();
  H->ad_off.clear(); H->ad_rowbase.clear();
  {
    long long rows = 0;
    auto add = [&](int q, long long off) {
      H->ad_r0.push_back(H->ar0[q]); H->ad_c0.push_back(H->ac0[q]);
      H->ad_h.push_back(H->ah[q]); H->ad_w.push_back(H->aw[q]);
      H->ad_off.push_back(off); H->ad_rowbase.push_back(rows);
      rows += H->ah[q];
    };
    for (size_t z = 0; z < expand_slots.size(); ++z) add(expand_slots[z], expand_off[z]);
    for (size_t z = 0; z < fb_q.size(); ++z) add(fb_q[z], fb_off[z]);
  }
  H->mv_dirty = true;
  H->dense_entries = H->nf_entries + adm_dense;
  const size_t vb = sizeof(V);
  if ((size_t)adm_dense * vb > H->dense_adm_cap) {
    if (H->dense_adm) H->exec_allocs.push_back(H->dense_adm);  // no device sync here
    H->dense_adm = nullptr;
    H->dense_adm_cap = (size_t)adm_dense * vb;
    HB_CUDA(cudaMalloc(&H->dense_adm, std::max(H->dense_adm_cap, vb)));
  }
  if (!expand_slots.empty()) {
    int *slots;
    long long *offs;
    HB_CHECK(upload_tmp(H, &slots, expand_slots));
    HB_CHECK(upload_tmp(H, &offs, expand_off));
    k_expand<T, C><<<(unsigned)expand_slots.size(), 128, 0, st>>>(
        slots, (int)expand_slots.size(), S, offs, H->dense_adm);
    HB_CUDA(cudaGetLastError());
    ++launches;
  }
  unsigned long long fb_sing = 0;
  if (!fb_r0.empty()) {
    // exact rows of non-converged blocks: the generic dense kernels on a
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
    HB_CHECK(upload_tmp(H, &p, tslot)); F.tile_slot = p;
    HB_CHECK(upload_tmp(H, &p, tstart)); F.tile_start = p;
    HB_CHECK(upload_tmp(H, &p, fb_r0)); F.r0 = p;
    HB_CHECK(upload_tmp(H, &p, fb_c0)); F.c0 = p;
    HB_CHECK(upload_tmp(H, &p, fb_h)); F.h = p;
    HB_CHECK(upload_tmp(H, &p, fb_w)); F.w = p;
    HB_CHECK(upload_tmp(H, &pl, fb_off)); F.off = pl;
    F.out = H->dense_adm;
    HB_CHECK(dalloc_tmp(H, &F.sing_count, 1));
    HB_CHECK(dalloc_tmp(H, &F.stat, 2));
    HB_CUDA(cudaMemsetAsync(F.sing_count, 0, 8, st));
    HB_CUDA(cudaMemsetAsync(F.stat, 0, 16, st));
    if (nt == 1 && ns == 1) {
      HB_CHECK(dalloc_tmp(H, &F.sing_slot, ent));
      HB_CHECK(dalloc_tmp(H, &F.sing_pos, ent));
    }
    const unsigned ntl = (unsigned)tslot.size();
    HB_CUDA(cudaStreamWaitEvent(st, H->tab_done, 0));  // exact rows may read the table
    int rc = dispatch_op(ctx->op, ctx->helm, nt, ns, [&](auto OPc, auto Hc, auto NTc,
                                                         auto NSc) -> int {
      constexpr int OP = decltype(OPc)::value;
      constexpr bool HH = decltype(Hc)::value != 0;
      constexpr int NT = decltype(NTc)::value, NS = decltype(NSc)::value;
      if constexpr (HH == C) {
        k_dense<T, C, OP, HH, NT, NS><<<ntl, kThreads, 0, st>>>(P, F);
        HB_CUDA(cudaGetLastError());
        if constexpr (NT == 1 && NS == 1) {
          k_dense_singular<T, C, OP, HH><<<148 * 16, kThreads, 0, st>>>(P, F);
          HB_CUDA(cudaGetLastError());
        }
        return HBEM_OK;
      } else {
        return set_error(HBEM_ERR_KERNEL, "value type does not match the equation");
      }
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
  if (H->out_dense && adm_dense > 0) {
    if (H->nf_entries + adm_dense > H->out_dense_cap)
      return set_error(HBEM_ERR_CAPACITY, "host dense arena of %lld values too small",
                       (long long)H->out_dense_cap);
    HB_CUDA(cudaEventRecord(H->emit_ev, st));
    HB_CUDA(cudaStreamWaitEvent(H->cpd, H->emit_ev, 0));
    HB_CUDA(cudaMemcpyAsync(static_cast<V *>(H->out_dense) + H->nf_entries, H->dense_adm,
                            (size_t)adm_dense * sizeof(V), cudaMemcpyDeviceToHost, H->cpd));
  }
  HB_CUDA(cudaStreamSynchronize(H->cp));
  HB_CUDA(cudaStreamSynchronize(H->cpd));
  const auto t_pre_wait = clk::now();
  HB_CUDA(cudaStreamWaitEvent(st, H->side_done, 0));
  unsigned long long nf_sing = 0, nf_stat[2] = {0, 0}, aca_stat[2] = {0, 0};
  HB_CUDA(cudaMemcpyAsync(&nf_sing, H->D.sing_count, 8, cudaMemcpyDeviceToHost, st));
  HB_CUDA(cudaMemcpyAsync(nf_stat, H->D.stat, 16, cudaMemcpyDeviceToHost, st));
  HB_CUDA(cudaMemcpyAsync(aca_stat, S.stat, 16, cudaMemcpyDeviceToHost, st));
  HB_CUDA(cudaStreamSynchronize(st));
  if (std::getenv("HBEM_PROF")) {  // phase cycles of a -DHB_PROF=1 kernel build
    unsigned long long pc[16];
    HB_CUDA(cudaMemcpy(pc, S.stat, sizeof(pc), cudaMemcpyDeviceToHost));
    if (pc[10] > 0)
    std::fprintf(stderr, "[hbem prof] warps %llu jobs %llu | cycles/job: life %.0f prologue %.0f "
                 "stage %.0f fload %.0f quad %.0f sing %.0f epi: resid %.0f argmax %.0f sums %.0f\n",
                 pc[11], pc[10], (double)pc[4] / pc[10], (double)pc[5] / pc[10],
                 (double)pc[6] / pc[10], (double)pc[12] / pc[10], (double)pc[7] / pc[10],
                 (double)pc[8] / pc[10], (double)pc[9] / pc[10], (double)pc[13] / pc[10],
                 (double)pc[14] / pc[10]);
  }
  const auto t_end = clk::now();
  if (wtrace) {
    for (size_t i = 0; i < wcp.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, wt0, wcp[i]);
      std::fprintf(stderr, "[hbem wave %2zu] host %.4f s  copies done %.4f s  %.2f GB\n", i,
                   whost[i], ms / 1e3, wbytes[i] / 1e9);
      cudaEventDestroy(wcp[i]);
    }
    cudaEventDestroy(wt0);
  }
  if (std::getenv("HBEM_TRACE"))
    std::fprintf(stderr, "[hbem execute] waves %.4f classify %.4f expand/fallback %.4f "
                 "near-field wait + stats %.4f s; mapping pool %.3f u %.3f v %.3f s "
                 "(%.1f / %.1f / %.1f GB)\n", secs(t0, t_aca), secs(t_aca, t_cls),
                 secs(t_cls, t_pre_wait), secs(t_pre_wait, t_end), H->vpool.grow_s,
                 H->uarena.grow_s, H->varena.grow_s, H->vpool.mapped / 1e9,
                 H->uarena.mapped / 1e9, H->varena.mapped / 1e9);
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
  ST.sing_table_pairs = H->sing_pairs_table;
  return HBEM_OK;
}

int execute(hbem_hmat *H, cudaStream_t caller) {
  hbem_ctx *ctx = H->ctx;
  cudaEvent_t e0, e1;
  HB_CUDA(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
  HB_CUDA(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
  HB_CUDA(cudaEventRecord(e0, caller));
  HB_CUDA(cudaStreamWaitEvent(H->hi, e0, 0));
  int rc;
  if (ctx->precision == HBEM_DOUBLE)
    rc = ctx->helm ? execute_t<double, true>(H, H->hi) : execute_t<double, false>(H, H->hi);
  else
    rc = ctx->helm ? execute_t<float, true>(H, H->hi) : execute_t<float, false>(H, H->hi);
  cudaEventRecord(e1, H->hi);
  cudaStreamWaitEvent(caller, e1, 0);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return rc;
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
  clear_error();
  HB_CUDA(cudaSetDevice(h->device));
  const size_t L = (size_t)h->n_leaves;
  const LeafMeta &M = h->meta;
  if (kind) HB_CUDA(cudaMemcpy(kind, M.kind, L * 4, cudaMemcpyDeviceToHost));
  if (rank) HB_CUDA(cudaMemcpy(rank, M.rank, L * 4, cudaMemcpyDeviceToHost));
  if (flags) HB_CUDA(cudaMemcpy(flags, M.flags, L * 4, cudaMemcpyDeviceToHost));
  if (off_u) HB_CUDA(cudaMemcpy(off_u, M.off_u, L * 8, cudaMemcpyDeviceToHost));
  if (off_v) HB_CUDA(cudaMemcpy(off_v, M.off_v, L * 8, cudaMemcpyDeviceToHost));
  if (off_dense) HB_CUDA(cudaMemcpy(off_dense, M.off_d, L * 8, cudaMemcpyDeviceToHost));
  return HBEM_OK;
}

int hbem_hmat_leaf_residual(const hbem_hmat *h, double *resid) {
  if (!h || !resid) return set_error(HBEM_ERR_ARG, "null argument");
  clear_error();
  HB_CUDA(cudaSetDevice(h->device));
  if (h->n_leaves > 0)
    HB_CUDA(cudaMemcpy(resid, h->meta.resid, (size_t)h->n_leaves * 8, cudaMemcpyDeviceToHost));
  return HBEM_OK;
}

// pack the converged low-rank factors of the last execute into the
// contiguous U / V arenas (k_pack_factors), once: copy_arenas and the device
// matvec read them
int ensure_packed(hbem_hmat *h, cudaStream_t st) {
  const size_t vb = h->vbytes;
  if (!h->packed && h->n_lowrank > 0) {
    const size_t n = (size_t)h->n_lowrank;
    const int *d_slots = h->lr_list;
    long long *d_uo = h->q_uoff, *d_vo = h->q_voff;  // free after the waves
    k_gather_ll<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_slots, (int)n, h->blk_uoff, d_uo);
    k_gather_ll<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_slots, (int)n, h->blk_voff, d_vo);
    HB_CHECK(h->uarena.grow((size_t)h->u_entries * vb));
    HB_CHECK(h->varena.grow((size_t)h->v_entries * vb));
    const int cnt = (int)n;
    void *ua = reinterpret_cast<void *>(h->uarena.base), *va = reinterpret_cast<void *>(h->varena.base);
    if (h->vbytes == 16)
      k_pack_factors<double, true><<<cnt, 128, 0, st>>>(d_slots, cnt, h->S, d_uo, d_vo, 0, 0,
                                                           (Cx<double> *)ua, (Cx<double> *)va);
    else if (h->vbytes == 8 && h->complex_)
      k_pack_factors<float, true><<<cnt, 128, 0, st>>>(d_slots, cnt, h->S, d_uo, d_vo, 0, 0,
                                                          (Cx<float> *)ua, (Cx<float> *)va);
    else if (h->vbytes == 8)
      k_pack_factors<double, false><<<cnt, 128, 0, st>>>(d_slots, cnt, h->S, d_uo, d_vo, 0, 0,
                                                            (double *)ua, (double *)va);
    else
      k_pack_factors<float, false><<<cnt, 128, 0, st>>>(d_slots, cnt, h->S, d_uo, d_vo, 0, 0,
                                                           (float *)ua, (float *)va);
    HB_CUDA(cudaGetLastError());
    HB_CUDA(cudaStreamSynchronize(st));
    h->packed = true;
  }
  return HBEM_OK;
}

int hbem_hmat_copy_arenas(const hbem_hmat *hc, void *u, void *v, void *dense) {
  clear_error();
  hbem_hmat *h = const_cast<hbem_hmat *>(hc);
  if (!h) return set_error(HBEM_ERR_ARG, "null hmat");
  HB_CUDA(cudaSetDevice(h->device));
  const size_t vb = h->vbytes;
  // three streams: dense arenas straight to the host, and the factor records
  // gathered into two alternating staging buffers so packing chunk i + 1
  // overlaps the PCIe copy of chunk i
  cudaStream_t sd = nullptr, sp[2] = {nullptr, nullptr};
  HB_CUDA(cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking));
  HB_CUDA(cudaStreamCreateWithFlags(&sp[0], cudaStreamNonBlocking));
  HB_CUDA(cudaStreamCreateWithFlags(&sp[1], cudaStreamNonBlocking));
  std::vector<void *> tmp;
  auto done = [&]() {
    cudaStreamSynchronize(sd);
    cudaStreamSynchronize(sp[0]);
    cudaStreamSynchronize(sp[1]);
    for (void *q : tmp) cudaFree(q);
    cudaStreamDestroy(sd);
    cudaStreamDestroy(sp[0]);
    cudaStreamDestroy(sp[1]);
  };
  auto fail = [&](cudaError_t e) {
    done();
    return set_error(HBEM_ERR_CUDA, "CUDA error %s in copy_arenas: %s", cudaGetErrorName(e),
                     cudaGetErrorString(e));
  };
  cudaError_t e = cudaSuccess;
  if (dense) {
    if (h->nf_entries > 0)
      e = cudaMemcpyAsync(dense, h->dense_nf, (size_t)h->nf_entries * vb, cudaMemcpyDeviceToHost,
                          sd);
    const long long adm = h->dense_entries - h->nf_entries;
    if (e == cudaSuccess && adm > 0)
      e = cudaMemcpyAsync((char *)dense + (size_t)h->nf_entries * vb, h->dense_adm,
                          (size_t)adm * vb, cudaMemcpyDeviceToHost, sd);
    if (e != cudaSuccess) return fail(e);
  }
  // low-rank factors: packed per wave when streaming, else packed here
  {
    const int rc = ensure_packed(h, sp[0]);
    if (rc != HBEM_OK) {
      done();
      return rc;
    }
  }
  if (e == cudaSuccess && u && h->u_entries > 0)
    e = cudaMemcpyAsync(u, reinterpret_cast<const void *>(h->uarena.base),
                        (size_t)h->u_entries * vb, cudaMemcpyDeviceToHost, sp[0]);
  if (e == cudaSuccess && v && h->v_entries > 0)
    e = cudaMemcpyAsync(v, reinterpret_cast<const void *>(h->varena.base),
                        (size_t)h->v_entries * vb, cudaMemcpyDeviceToHost, sp[1]);
  if (e != cudaSuccess) return fail(e);
  done();
  HB_CUDA(cudaGetLastError());
  return HBEM_OK;
}

// build the matvec's work items, slot layout and cover lists once per
// assembly (host lists from the last execute, uploaded)
static int matvec_prepare(hbem_hmat *h) {
  if (!h->mv_dirty) return HBEM_OK;
  const size_t vb = h->vbytes;
  cudaFree(h->mv_ad); cudaFree(h->mv_ad_l);
  h->mv_ad = nullptr; h->mv_ad_l = nullptr;
  const size_t na = h->ad_r0.size();
  HB_CUDA(cudaMalloc(&h->mv_ad, std::max<size_t>(na, 1) * 4 * 4));
  HB_CUDA(cudaMalloc(&h->mv_ad_l, std::max<size_t>(na, 1) * 8 * 2));
  if (na) {
    HB_CUDA(cudaMemcpy(h->mv_ad, h->ad_r0.data(), na * 4, cudaMemcpyHostToDevice));
    HB_CUDA(cudaMemcpy(h->mv_ad + na, h->ad_c0.data(), na * 4, cudaMemcpyHostToDevice));
    HB_CUDA(cudaMemcpy(h->mv_ad + 2 * na, h->ad_h.data(), na * 4, cudaMemcpyHostToDevice));
    HB_CUDA(cudaMemcpy(h->mv_ad + 3 * na, h->ad_w.data(), na * 4, cudaMemcpyHostToDevice));
    HB_CUDA(cudaMemcpy(h->mv_ad_l, h->ad_off.data(), na * 8, cudaMemcpyHostToDevice));
    HB_CUDA(cudaMemcpy(h->mv_ad_l + na, h->ad_rowbase.data(), na * 8, cudaMemcpyHostToDevice));
  }
  long long ad_rows = 0;
  for (int hh : h->ad_h) ad_rows += hh;
  h->mv_ad_rows = ad_rows;
  // low-rank work items: (list position, chunk start) over columns (dots)
  // and rows, kMvChunk each; per-position offsets of the k dots
  cudaFree(h->mv_items); cudaFree(h->mv_sbase); cudaFree(h->mv_s);
  cudaFree(h->mv_part); cudaFree(h->mv_dpart);
  cudaFree(h->mv_ifirst); cudaFree(h->mv_ibase); cudaFree(h->mv_rbase);
  cudaFree(h->mv_cstart); cudaFree(h->mv_cptr); cudaFree(h->mv_cover);
  h->mv_items = nullptr; h->mv_sbase = nullptr; h->mv_s = nullptr;
  h->mv_part = h->mv_dpart = nullptr;
  h->mv_ifirst = h->mv_ibase = h->mv_rbase = nullptr;
  h->mv_cstart = nullptr; h->mv_cptr = h->mv_cover = nullptr;
  const int nl = h->n_lowrank;
  std::vector<int> lst(nl), rk(h->na > 0 ? h->na : 1);
  if (nl > 0) {
    HB_CUDA(cudaMemcpy(lst.data(), h->lr_list, (size_t)nl * 4, cudaMemcpyDeviceToHost));
    HB_CUDA(cudaMemcpy(rk.data(), h->S.rank, (size_t)h->na * 4, cudaMemcpyDeviceToHost));
  }
  const long long lr0 = h->nf_rows + ad_rows;  // first low-rank partial slot
  std::vector<int2> items;
  std::vector<long long> sbase(std::max(nl, 1)), ifirst(nl + 1), ibase, rbase(std::max(nl, 1));
  long long ns = 0, nsd = 0, rows = lr0;
  for (int p = 0; p < nl; ++p) {
    const int b = lst[p];
    sbase[p] = ns;
    ns += rk[b];
    rbase[p] = rows;
    rows += h->ah[b];
    ifirst[p] = (long long)items.size();
    for (int c = 0; c < h->aw[b]; c += kMvChunk) {
      items.push_back(make_int2(p, c));
      ibase.push_back(nsd);
      nsd += rk[b];
    }
  }
  ifirst[nl] = (long long)items.size();
  const long long nd_items = (long long)items.size();
  for (int p = 0; p < nl; ++p)
    for (int r = 0; r < h->ah[lst[p]]; r += kMvChunk) items.push_back(make_int2(p, r));
  h->mv_nd = nd_items;
  h->mv_nr = (long long)items.size() - nd_items;
  h->mv_ns = ns;
  const long long nslots = rows;
  // cover lists: every leaf component (near-field leaf, admissible block
  // stored densely, low-rank block) in the reference's (row start, column
  // start) order, appended to each tree row cluster inside its row range
  struct Comp { int r0, c0, h; long long cover; };
  std::vector<Comp> comps;
  comps.reserve((size_t)h->nd + na + nl);
  {
    long long acc = 0;  // near-field leaf rows: exclusive prefix of the heights (nf_rowbase)
    for (int q = 0; q < h->nd; ++q) {
      comps.push_back({h->nf_r0[q], h->nf_c0[q], h->nf_h[q], acc - h->nf_r0[q]});
      acc += h->nf_h[q];
    }
  }
  for (size_t z = 0; z < na; ++z)
    comps.push_back({h->ad_r0[z], h->ad_c0[z], h->ad_h[z],
                     h->nf_rows + h->ad_rowbase[z] - h->ad_r0[z]});
  for (int p = 0; p < nl; ++p) {
    const int b = lst[p];
    comps.push_back({h->ar0[b], h->ac0[b], h->ah[b], rbase[p] - h->ar0[b]});
  }
  std::sort(comps.begin(), comps.end(), [](const Comp &a, const Comp &b) {
    return a.r0 != b.r0 ? a.r0 < b.r0 : a.c0 < b.c0;
  });
  const std::vector<int> &cs = h->rleaf_start;
  const int ncl = (int)cs.size() - 1;
  std::vector<long long> cnt(ncl + 1, 0);
  auto cl_of = [&](int r) {  // row cluster containing row r
    return (int)(std::upper_bound(cs.begin(), cs.end(), r) - cs.begin()) - 1;
  };
  for (const Comp &c : comps)
    for (int g = cl_of(c.r0); g < ncl && cs[g] < c.r0 + c.h; ++g) ++cnt[g];
  std::vector<long long> cptr(ncl + 1, 0);
  for (int g = 0; g < ncl; ++g) cptr[g + 1] = cptr[g] + cnt[g];
  std::vector<long long> cover((size_t)std::max<long long>(cptr[ncl], 1));
  std::vector<long long> fill(cptr.begin(), cptr.end() - 1);
  for (const Comp &c : comps)
    for (int g = cl_of(c.r0); g < ncl && cs[g] < c.r0 + c.h; ++g) cover[fill[g]++] = c.cover;
  h->mv_ncl = ncl;
  HB_CUDA(cudaMalloc(&h->mv_items, std::max<size_t>(items.size(), 1) * sizeof(int2)));
  HB_CUDA(cudaMalloc(&h->mv_sbase, sbase.size() * 8));
  HB_CUDA(cudaMalloc(&h->mv_s, (size_t)std::max<long long>(ns, 1) * vb));
  HB_CUDA(cudaMalloc(&h->mv_dpart, (size_t)std::max<long long>(nsd, 1) * vb));
  HB_CUDA(cudaMalloc(&h->mv_part, (size_t)std::max<long long>(nslots, 1) * vb));
  HB_CUDA(cudaMalloc(&h->mv_ifirst, ifirst.size() * 8));
  HB_CUDA(cudaMalloc(&h->mv_ibase, std::max<size_t>(ibase.size(), 1) * 8));
  HB_CUDA(cudaMalloc(&h->mv_rbase, rbase.size() * 8));
  HB_CUDA(cudaMalloc(&h->mv_cstart, cs.size() * 4));
  HB_CUDA(cudaMalloc(&h->mv_cptr, cptr.size() * 8));
  HB_CUDA(cudaMalloc(&h->mv_cover, cover.size() * 8));
  if (!items.empty())
    HB_CUDA(cudaMemcpy(h->mv_items, items.data(), items.size() * sizeof(int2),
                       cudaMemcpyHostToDevice));
  HB_CUDA(cudaMemcpy(h->mv_sbase, sbase.data(), sbase.size() * 8, cudaMemcpyHostToDevice));
  HB_CUDA(cudaMemcpy(h->mv_ifirst, ifirst.data(), ifirst.size() * 8, cudaMemcpyHostToDevice));
  if (!ibase.empty())
    HB_CUDA(cudaMemcpy(h->mv_ibase, ibase.data(), ibase.size() * 8, cudaMemcpyHostToDevice));
  HB_CUDA(cudaMemcpy(h->mv_rbase, rbase.data(), rbase.size() * 8, cudaMemcpyHostToDevice));
  HB_CUDA(cudaMemcpy(h->mv_cstart, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice));
  HB_CUDA(cudaMemcpy(h->mv_cptr, cptr.data(), cptr.size() * 8, cudaMemcpyHostToDevice));
  HB_CUDA(cudaMemcpy(h->mv_cover, cover.data(), cover.size() * 8, cudaMemcpyHostToDevice));
  h->mv_dirty = false;
  return HBEM_OK;
}

// y = H x with x, y device pointers in the original DOF order, on stream st
static int matvec_device(hbem_hmat *h, const void *dx, void *dy, cudaStream_t st) {
  const size_t vb = h->vbytes;
  const int nr = h->n_rows, nc = h->n_cols;
  if (!h->mv_buf) HB_CUDA(cudaMalloc(&h->mv_buf, (size_t)2 * (nr + nc) * vb));
  char *buf = static_cast<char *>(h->mv_buf);
  void *dxt = buf + (size_t)nc * vb, *dyt = buf + (size_t)(2 * nc + nr) * vb;
  HB_CHECK(matvec_prepare(h));
  MatvecArgs M{};
  M.n_rows = nr;
  M.n_cols = nc;
  M.rperm = h->rperm;
  M.cperm = h->cperm;
  M.x = dx; M.y = dy; M.xt = dxt; M.yt = dyt;
  M.dense[0] = MatvecArgs::Dense{h->nd, h->D.r0, h->D.c0, h->D.h, h->D.w, h->D.off,
                                 h->nf_rowbase, h->nf_rows, h->dense_nf, 0};
  const int na = (int)h->ad_r0.size();
  M.dense[1] = MatvecArgs::Dense{na, h->mv_ad, h->mv_ad + na, h->mv_ad + 2 * na,
                                 h->mv_ad + 3 * na, h->mv_ad_l, h->mv_ad_l + na, h->mv_ad_rows,
                                 h->dense_adm, h->nf_rows};
  M.n_lowrank = h->n_lowrank;
  M.lowrank = h->lr_list;
  HB_CHECK(ensure_packed(h, st));
  M.ua = reinterpret_cast<const void *>(h->uarena.base);
  M.va = reinterpret_cast<const void *>(h->varena.base);
  M.uoff = h->blk_uoff;
  M.voff = h->blk_voff;
  M.n_ditems = h->mv_nd;
  M.n_ritems = h->mv_nr;
  M.ditems = h->mv_items;
  M.ritems = h->mv_items + h->mv_nd;
  M.sbase = h->mv_sbase;
  M.ifirst = h->mv_ifirst;
  M.ibase = h->mv_ibase;
  M.rbase = h->mv_rbase;
  M.s = h->mv_s;
  M.dpart = h->mv_dpart;
  M.n_s = h->mv_ns;
  M.part = h->mv_part;
  M.n_clusters = h->mv_ncl;
  M.cstart = h->mv_cstart;
  M.cptr = h->mv_cptr;
  M.cover = h->mv_cover;
  const hbem_ctx *ctx = h->ctx;
  if (ctx->precision == HBEM_DOUBLE)
    return ctx->helm ? matvec_launch<double, true>(M, h->S, st)
                     : matvec_launch<double, false>(M, h->S, st);
  return ctx->helm ? matvec_launch<float, true>(M, h->S, st)
                   : matvec_launch<float, false>(M, h->S, st);
}

int hbem_hmat_matvec(const hbem_hmat *hc, const void *x, void *y) {
  clear_error();
  hbem_hmat *h = const_cast<hbem_hmat *>(hc);
  if (!h || !x || !y) return set_error(HBEM_ERR_ARG, "null argument");
  HB_CUDA(cudaSetDevice(h->device));
  const size_t vb = h->vbytes;
  const int nr = h->n_rows, nc = h->n_cols;
  if (!h->mv_buf) HB_CUDA(cudaMalloc(&h->mv_buf, (size_t)2 * (nr + nc) * vb));
  char *buf = static_cast<char *>(h->mv_buf);
  void *dx = buf, *dy = buf + (size_t)2 * nc * vb;
  HB_CUDA(cudaMemcpy(dx, x, (size_t)nc * vb, cudaMemcpyHostToDevice));
  HB_CHECK(matvec_device(h, dx, dy, 0));
  HB_CUDA(cudaMemcpy(y, dy, (size_t)nr * vb, cudaMemcpyDeviceToHost));
  return HBEM_OK;
}

int hbem_hmat_matvec_device(const hbem_hmat *hc, const void *d_x, void *d_y, void *stream) {
  clear_error();
  hbem_hmat *h = const_cast<hbem_hmat *>(hc);
  if (!h || !d_x || !d_y) return set_error(HBEM_ERR_ARG, "null argument");
  HB_CUDA(cudaSetDevice(h->device));
  return matvec_device(h, d_x, d_y, (cudaStream_t)stream);
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
