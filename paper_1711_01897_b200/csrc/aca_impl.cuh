// Lock-step batched ACA over every admissible block (aca, hmatrix.py:271-382),
// one phase = one launch family over all active blocks.
//
// Phase structure (row phase shown; the column phase is its mirror):
//   select   deterministic stream compaction of the blocks that need a row
//            job, in a static order sorted by column cluster: jobs that run
//            over the same column cluster are adjacent ("groups");
//   need     per job: pool values for a fresh pending term record, partial
//            records (one per 32-wide tile), warp items (group heads only);
//            one inclusive scan gives every offset;
//   jobs     per job record + (group head, tile) warp items;
//   integrate  one warp per item: lane l keeps the varying element of tile
//            column 32 t + l in registers (P0) and walks every job of the
//            group with the fixed element broadcast from shared memory; per
//            entry: Galerkin integral (touching pairs: warp-cooperative
//            Sauter-Schwab), residual update with the accepted terms
//            (hmatrix.py:323-327 / 340-342), store; per tile: argmax over
//            unmasked entries, sum |.|^2 and the dots with the factors the
//            residual read (cross terms of the Frobenius update, 359-362);
//   finalize one warp per job combines its tiles in fixed order: pivot,
//            vanishing row (334-338), stopping test and norm update
//            (343-370), next row pivot (301-314).
// Every reduction runs in a fixed order, so payloads are bitwise
// reproducible and independent of how blocks are split across GPUs.
#pragma once
#include <cub/cub.cuh>

#include <type_traits>

#include "hmat_common.cuh"

namespace hb {

constexpr unsigned kFull = 0xffffffffu;
#ifndef HB_ACA_P0_MINB
#define HB_ACA_P0_MINB 3  // k_aca_p0 resident CTAs per SM (register cap 168)
#endif

// ---------------------------------------------------------------------------
// state init, list selection, needs, jobs
// ---------------------------------------------------------------------------
static __global__ void k_aca_init(AcaDev S, int n) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n) return;
  const int h = S.h[b], w = S.w[b];
  S.rank[b] = 0;
  S.cur[b] = 0;
  S.small[b] = 0;
  S.status[b] = ST_ACTIVE;
  S.exhausted[b] = 0;
  S.norm2[b] = 0.0;
  S.resid[b] = INFINITY;
  S.pend[b] = -1;
  S.flagA[b] = 1;
  S.flagC[b] = 0;
  unsigned *rm = S.rmask + S.rmask_off[b];
  for (int k = 0; k < (h + 31) / 32; ++k) {
    const int valid = min(32, h - k * 32);
    rm[k] = valid == 32 ? 0u : ~((1u << valid) - 1u);
  }
  unsigned *cm = S.cmask + S.cmask_off[b];
  for (int k = 0; k < (w + 31) / 32; ++k) {
    const int valid = min(32, w - k * 32);
    cm[k] = valid == 32 ? 0u : ~((1u << valid) - 1u);
  }
}

static __global__ void k_phase_flags(const unsigned char *flag, const int *order, int n,
                              unsigned char *out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) out[q] = flag[order[q]];
}

template <int NC>
__global__ void __launch_bounds__(kNeedThreads) k_need(AcaDev S, int na, int col, int NT_, int NS_,
                                                      Need *bsum) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = *S.nlist;
  if ((long long)blockIdx.x * kNeedThreads >= n) {
    // past the selected list (later waves: most of the blocks)
    if (threadIdx.x == 0) bsum[blockIdx.x] = Need{0, 0, 0, 0, 0};
    return;
  }
  Need d{0, 0, 0, 0, 0};
  if (p < n && p < na) {
    const int b = S.list[p];
    const BlockInfo bi = S.binfo[b];
    const int h = bi.h, w = bi.w, k = S.rank[b];
    const int tiles = tiles_of(col ? h : w);
    const int key = col ? bi.rnode : bi.cnode;
    S.pkey[p] = key;
    bool head = p == 0;
    if (!head) {
      const int bp = S.list[p - 1];
      head = key != (col ? S.binfo[bp].rnode : S.binfo[bp].cnode);
    }
    d.pool = (!col && S.pend[b] < 0) ? (long long)h + w + 1 : 0;
    // per tile: statistics (4) + dots (k NC), padded even (part_len)
    d.part = (long long)tiles * part_len(k, NC);
    d.items = head ? tiles : 0;
    if (NT_ != 1 || NS_ != 1) {
      // element-level rows: the varying cluster's element union
      const long long *ep = col ? S.recl_ptr : S.cecl_ptr;
      const long long ne = ep[key + 1] - ep[key];
      d.eitems = head ? (ne + 31) / 32 : 0;
      d.rsc = ne * (col ? NT_ : NS_);
    }
  }
  // block-local inclusive scan; k_need_carry adds the preceding blocks' totals
  using BS = cub::BlockScan<Need, kNeedThreads>;
  __shared__ typename BS::TempStorage ts;
  Need inc;
  BS(ts).InclusiveScan(d, inc, SumNeed());
  if (p < na) {
    S.need[p] = d;
    S.scan[p] = inc;
  }
  if (threadIdx.x == kNeedThreads - 1) bsum[blockIdx.x] = inc;
}

// exclusive scan of the block totals of the selected list, one CTA (in
// place); the grand total goes to bsum[nb] (the phase's one host read)
static __global__ void __launch_bounds__(1024) k_need_blocks(Need *bsum, int nb, const int *nlist) {
  using BS = cub::BlockScan<Need, 1024>;
  __shared__ typename BS::TempStorage ts;
  Need carry{0, 0, 0, 0, 0};
  const int nbe = min(nb, (*nlist + kNeedThreads - 1) / kNeedThreads);
  for (int base = 0; base < nbe; base += 1024) {
    const int i = base + threadIdx.x;
    Need v = i < nb ? bsum[i] : Need{0, 0, 0, 0, 0};
    Need ex, tot;
    BS(ts).ExclusiveScan(v, ex, Need{0, 0, 0, 0, 0}, SumNeed(), tot);
    __syncthreads();
    if (i < nbe) bsum[i] = SumNeed()(carry, ex);
    carry = SumNeed()(carry, tot);
  }
  if (threadIdx.x == 0) bsum[nb] = carry;
}

static __global__ void k_need_carry(AcaDev S, int na, const Need *bsum) {
  const int p = (blockIdx.x + 1) * kNeedThreads + threadIdx.x;
  if (p < na && p < *S.nlist) S.scan[p] = SumNeed()(bsum[blockIdx.x + 1], S.scan[p]);
}

template <typename T, bool C>
__device__ void write_stage(const Prob<T> &P, const AcaDev &S, int p, const Job &J,
                            const long long (&jt)[kFinRegs], const V_t<T, C> (&jc)[kFinRegs],
                            int col, int local);

// job records, residual terms and warp items of a phase; P0 (stage >= 0):
// also the job's StageRec (everything k_aca_p0 stages, fixed element relative
// to the group origin: stage = 1 local frame) and each item's group length
#ifndef HB_JOBS_MINB
#define HB_JOBS_MINB 1
#endif
template <typename T, bool C>
__global__ void __launch_bounds__(128, HB_JOBS_MINB) k_jobs(Prob<T> P, AcaDev S, int n, int col, int stage) {
  using N = Num<T, C>;
  using V = typename N::V;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int b = S.list[p];
  const Need sc = S.scan[p], nd = S.need[p];
  const BlockInfo bi = S.binfo[b];
  Job J;
  J.b = b;
  J.h = bi.h;
  J.w = bi.w;
  J.k = S.rank[b];
  const int r0 = bi.r0, c0 = bi.c0;
  J.part = sc.part - nd.part;
  J.rsc = sc.rsc - nd.rsc;
  if (!col) {
    J.key = bi.cnode;
    J.fix = S.cur[b];
    const long long pe = S.pend[b];
    J.pe = pe >= 0 ? pe : S.pool_base + sc.pool - nd.pool;
    J.nfix = r0 + J.fix;
    J.mofs = bi.cmo;
    J.vstart = c0;
    J.nvar = J.w;
    J.cur = J.fix;
    S.rowpart[b] = J.part;
  } else {
    J.key = bi.rnode;
    J.fix = S.pcol[b];
    J.pe = S.pend[b];
    J.nfix = c0 + J.fix;
    J.mofs = bi.rmo;
    J.vstart = r0;
    J.nvar = J.h;
    J.cur = S.cur[b];
  }
  S.jobs[p] = J;
  // first terms of the residual: record offsets and coefficients
  long long jt[kFinRegs];
  V jc[kFinRegs];
#pragma unroll
  for (int l = 0; l < kFinRegs; ++l) {
    jt[l] = 0;
    jc[l] = N::zero();
  }
  if (J.k > 0) {
    const V *pool = static_cast<const V *>(S.pool);
    const long long *tl = S.terms + (long long)b * S.tmax;
    const V *tp = static_cast<const V *>(S.tpiv) + (long long)b * S.tmax;
    const int fixo = col ? J.h + J.fix : J.fix;
    const int kk = min(J.k, kFinRegs);
#pragma unroll
    for (int l = 0; l < kFinRegs; ++l)
      if (l < kk) {
        const long long t = tl[l];
        jt[l] = t;
        jc[l] = N::div(pool[t + fixo], tp[l]);
      }
    if (stage < 0) {  // the linear-space kernels read them from here
      long long *gjt = S.jt + (long long)p * kFinRegs;
      V *gjc = static_cast<V *>(S.jc) + (long long)p * kFinRegs;
#pragma unroll
      for (int l = 0; l < kFinRegs; ++l)
        if (l < kk) {
          gjt[l] = jt[l];
          gjc[l] = jc[l];
        }
    }
  }
  if (stage >= 0) write_stage<T, C>(P, S, p, J, jt, jc, col, stage);
  if (nd.items) {
    const long long base = sc.items - nd.items;
    // jobs of the group (consecutive positions with this key)
    int glen = 1;
    while (p + glen < n && S.pkey[p + glen] == J.key) ++glen;
    for (long long t = 0; t < nd.items; ++t) {
      S.items[base + t] = make_int4(p, (int)t, J.vstart, J.nvar);
      S.iglen[base + t] = glen;
    }
  }
  if (nd.eitems) {
    const long long base = sc.eitems - nd.eitems;
    for (long long t = 0; t < nd.eitems; ++t) S.eitems[base + t] = make_int2(p, (int)t);
  }
}

// ---------------------------------------------------------------------------
// warp helpers
// ---------------------------------------------------------------------------
template <typename V> __device__ __forceinline__ V shfl_v(V v, int src);
template <> __device__ __forceinline__ double shfl_v<double>(double v, int src) {
  return __shfl_sync(kFull, v, src);
}
template <> __device__ __forceinline__ float shfl_v<float>(float v, int src) {
  return __shfl_sync(kFull, v, src);
}
template <> __device__ __forceinline__ Cx<double> shfl_v<Cx<double>>(Cx<double> v, int src) {
  return Cx<double>{__shfl_sync(kFull, v.re, src), __shfl_sync(kFull, v.im, src)};
}
template <> __device__ __forceinline__ Cx<float> shfl_v<Cx<float>>(Cx<float> v, int src) {
  return Cx<float>{__shfl_sync(kFull, v.re, src), __shfl_sync(kFull, v.im, src)};
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// Transposed warp reduction of 8 per-lane values: after 9 shuffles lane l
// holds the warp total of value index l >> 2 (the halving exchange keeps
// half of the values per step, then two butterfly steps finish).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double tr_reduce8(const double (&v)[8], int lane) {
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
  double a[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double send = h16 ? v[i] : v[i + 4];
    const double keep = h16 ? v[i + 4] : v[i];
    a[i] = keep + __shfl_xor_sync(kFull, send, 16);
  }
  double b[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double send = h8 ? a[i] : a[i + 2];
    const double keep = h8 ? a[i + 2] : a[i];
    b[i] = keep + __shfl_xor_sync(kFull, send, 8);
  }
  double c;
  {
    const double send = h4 ? b[0] : b[1];
    const double keep = h4 ? b[1] : b[0];
    c = keep + __shfl_xor_sync(kFull, send, 4);
  }
  c += __shfl_xor_sync(kFull, c, 2);
  c += __shfl_xor_sync(kFull, c, 1);
  return c;
}

// cp.async (LDGSTS) of one value into shared memory: the residual factor
// prefetch costs no registers while the quadrature runs
template <int BYTES>
__device__ __forceinline__ void cp_async(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem), "n"(BYTES));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// read-only (non-coherent path) load of a value
template <typename V> __device__ __forceinline__ V ld_ro(const V *p) { return __ldg(p); }
template <> __device__ __forceinline__ Cx<double> ld_ro<Cx<double>>(const Cx<double> *p) {
  const double2 v = __ldg(reinterpret_cast<const double2 *>(p));
  return Cx<double>{v.x, v.y};
}
template <> __device__ __forceinline__ Cx<float> ld_ro<Cx<float>>(const Cx<float> *p) {
  const float2 v = __ldg(reinterpret_cast<const float2 *>(p));
  return Cx<float>{v.x, v.y};
}

// job view staged in shared memory by the integration kernels
struct JobS {
  long long pe;     // pending record
  long long part;   // first tile record
  long long rsc_off;  // element-row values (linear spaces)
  int b, h, w, k, fix, cur;
  long long mofs;   // used-index mask words of the varying side (offset)
  unsigned mw;      // used-index mask word of the varying side at this tile
  int nfix;         // tree position of the fixed DOF (its element record, P0)
};

// ---------------------------------------------------------------------------
// ACA residual epilogue of one (job, tile) — shared by the P0 and linear-space
// integration kernels.  f[l] (l < min(k, 8)) are the factor values of the
// first terms at this lane's entry, prefetched before the integral; c[l] the
// coefficients (row phase u_l[i] / p_l, column phase r_l[j] / p_l).
//   row:    val = A(i, c) - sum_l u_l[i] v_l[c]   (hmatrix.py:323-327)
//   column: val = A(r, j) - sum_l v_l[j] u_l[r]   (hmatrix.py:340-342)
// Writes the residual into the pending record and the tile record
// [best |val| over unmasked, its index, sum |val|^2, pad, vdot(f_l, val) ...]:
// the pivot statistics of the residual (argmax over unused indices, first
// index on ties, hmatrix.py:301-314 / 329-332; squared norm 343-362) are
// reduced here while the values are in registers, so the finalize kernels
// never re-read the residual rows and columns.
// ---------------------------------------------------------------------------
template <typename T, bool C, bool COL>
__device__ __forceinline__ void aca_epi(const AcaDev &S, const JobS &J, const V_t<T, C> *cs,
                                        int t, int lane, bool valid, V_t<T, C> val,
                                        const V_t<T, C> *fb) {
  using N = Num<T, C>;
  using V = typename N::V;
  constexpr int NC = N::NC;
  V *pool = static_cast<V *>(S.pool);
  const int idx = t * 32 + lane;
  const int k = J.k, kk = min(k, kFinRegs);
  const int ro = COL ? 0 : J.h;
  // f_l at this lane's entry: fb[l * 32 + lane] (valid lanes only)
#pragma unroll
  for (int l = 0; l < kFinRegs; ++l)
    if (l < kk && valid) val = N::fms(val, cs[l], fb[l * 32 + lane]);
  // terms beyond the register batch (late waves of high-rank blocks)
  const long long *tl = S.terms + (long long)J.b * S.tmax;
  const int fixo = COL ? J.h + J.fix : J.fix;
  for (int l = kFinRegs; l < k; ++l) {
    const long long tb = tl[l];
    const V c = N::div(pool[tb + fixo], pool[tb + J.h + J.w]);
    if (valid) val = N::fms(val, c, pool[tb + ro + idx]);
  }
  if (valid) pool[J.pe + (COL ? 0 : J.h) + idx] = val;
  double *rec = S.part + J.part + (long long)t * part_len(k, NC);
  {
    // column phase: the block's current row is excluded from the next pivot
    const bool masked = !valid || ((J.mw >> lane) & 1u) || (COL && idx == J.cur);
    double best = masked ? -1.0 : N::abs(val);
    int bidx = masked ? 0x7fffffff : idx;
    double ss = valid ? N::nrm(val) : 0.0;
    warp_argmax_sum(best, bidx, ss);
    if (lane == 0) {
      rec[0] = best;
      rec[1] = (double)bidx;
      rec[2] = ss;
    }
  }
  // dots vdot(f_l, val) of the register batch: transposed reduction
  if (kk > 0) {
    double dr[8], di[8];
#pragma unroll
    for (int l = 0; l < 8; ++l) {
      dr[l] = 0.0;
      di[l] = 0.0;
      if (l < kk && valid) N::cdot(dr[l], di[l], fb[l * 32 + lane], val);
    }
    const double sr = tr_reduce8(dr, lane);
    const double si = C ? tr_reduce8(di, lane) : 0.0;
    const int l = lane >> 2;
    if ((lane & 3) == 0 && l < kk) {
      rec[4 + l * NC] = sr;
      if (C) rec[4 + l * NC + 1] = si;
    }
  }
  for (int l = kFinRegs; l < k; ++l) {
    const long long tb = tl[l];
    double dr = 0.0, di = 0.0;
    if (valid) N::cdot(dr, di, pool[tb + ro + idx], val);
    dr = warp_sum_d(dr);
    if (C) di = warp_sum_d(di);
    if (lane == 0) {
      rec[4 + l * NC] = dr;
      if (C) rec[4 + l * NC + 1] = di;
    }
  }
}

// ---------------------------------------------------------------------------
// Branch-free epilogue of the P0 kernel, KK = min(k, kFinRegs) known at
// compile time (dispatched once per job: in wave w nearly every job has
// k = w, so one instantiation runs per launch).
//
//   residual   val -= c_l f_l for l < KK (f_l loaded here from the pool: the
//              loads' latency is covered by the other resident warps'
//              quadratures), then the terms beyond the register batch;
//   pivot      argmax of |val| over unused indices with the first index on
//              ties, exactly: the float64 bit patterns of |val| >= 0 order
//              like the values, so two warp REDUX max (high word, then low
//              word among the lanes holding the maximal high word) and one
//              ballot give the winner;
//   sums       sum |val|^2 and the KK dots vdot(f_l, val) reduced through a
//              shared-memory transpose: G = 32 / NV lanes per value each add
//              32 / G rows in a fixed order, then log2(G) butterfly steps.
// ---------------------------------------------------------------------------
template <int NV> struct TrGroup {
  static constexpr int G = NV <= 1 ? 32 : NV <= 2 ? 16 : NV <= 4 ? 8 : NV <= 8 ? 4 : NV <= 16 ? 2 : 1;
};
constexpr int kRedStride = 17;  // doubles per lane row of the transpose scratch (odd: bank spread)

template <int NV>
__device__ __forceinline__ double tr_sums(const double (&v)[NV], double *red, int lane) {
  static_assert(NV <= kRedStride, "transpose scratch too narrow");
  constexpr int G = TrGroup<NV>::G;
#pragma unroll
  for (int i = 0; i < NV; ++i) red[lane * kRedStride + i] = v[i];
  __syncwarp();
  const int vi = lane / G, part = lane % G;
  // rows part, part + G, ... added as a balanced tree (fixed order, short
  // dependency chains)
  constexpr int R = 32 / G;
  double a[R];
#pragma unroll
  for (int r = 0; r < R; ++r) a[r] = vi < NV ? red[(part + r * G) * kRedStride + vi] : 0.0;
#pragma unroll
  for (int w = 1; w < R; w *= 2)
#pragma unroll
    for (int r = 0; r + w < R; r += 2 * w) a[r] += a[r + w];
  double acc = a[0];
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  __syncwarp();
  return acc;  // lanes vi * G .. vi * G + G - 1 hold value vi's sum
}

template <typename T, bool C, bool COL, int KK>
__device__ __forceinline__ void aca_epi_p0(const AcaDev &S, const JobS &J, unsigned mw,
                                           const V_t<T, C> *cs,
                                           const V_t<T, C> (&f)[kFinRegs], V_t<T, C> *out,
                                           double *rec, int t, int lane, bool valid,
                                           V_t<T, C> val, double *red
#if HB_PROF
                                           , unsigned long long *pc, unsigned long long &pt
#endif
                                           ) {
  using N = Num<T, C>;
  using V = typename N::V;
  constexpr int NC = N::NC;
#pragma unroll
  for (int l = 0; l < KK; ++l) val = N::fms(val, cs[l], f[l]);
#if HB_PROF
  if ((double)N::re(val) == 1.2345e300) ++pc[0];
  { const unsigned long long c = clock64(); pc[5] += c - pt; pt = c; }
#endif
  const int k = J.k;
  if (k > KK) {
    // terms beyond the register batch (late waves of high-rank blocks)
    const V *pool = static_cast<const V *>(S.pool);
    const long long *tl = S.terms + (long long)J.b * S.tmax;
    const int fixo = COL ? J.h + J.fix : J.fix;
    const int ro = COL ? 0 : J.h;
    const int idx = t * 32 + lane;
    for (int l = KK; l < k; ++l) {
      const long long tb = tl[l];
      const V c = N::div(pool[tb + fixo], pool[tb + J.h + J.w]);
      if (valid) val = N::fms(val, c, pool[tb + ro + idx]);
    }
  }
  if (valid) out[lane] = val;
  // pivot candidate of the tile
  const bool masked = !valid || ((mw >> lane) & 1u) || (COL && t * 32 + lane == J.cur);
  const unsigned long long bits =
      masked ? 0ull : (unsigned long long)__double_as_longlong(N::abs(val));
  const unsigned hi = (unsigned)(bits >> 32), lo = (unsigned)bits;
  const unsigned mh = __reduce_max_sync(kFull, hi);
  unsigned cand = __ballot_sync(kFull, !masked && hi == mh);
  if (cand & (cand - 1)) {
    // several lanes share the maximal high word (rare): compare the low words
    const unsigned ml = __reduce_max_sync(kFull, ((cand >> lane) & 1u) ? lo : 0u);
    cand &= __ballot_sync(kFull, lo == ml);
  }
  // the winner (first index on ties) writes its own |val|; lane 0 the empty record
  if (lane == (cand ? __ffs(cand) - 1 : 0)) {
    rec[0] = cand ? __longlong_as_double((long long)bits) : -1.0;
    rec[1] = cand ? (double)(t * 32 + lane) : 2147483647.0;
  }
#if HB_PROF
  if (cand == 0x12345u) ++pc[0];
  { const unsigned long long c = clock64(); pc[7] += c - pt; pt = c; }
#endif
  // sum |val|^2 and the register-batch dots, one transposed reduction
  constexpr int NV = 1 + KK * NC;
  double v[NV];
  v[0] = valid ? N::nrm(val) : 0.0;
#pragma unroll
  for (int l = 0; l < KK; ++l) {
    double dr = 0.0, di = 0.0;
    N::cdot(dr, di, f[l], val);  // f = 0 on invalid lanes
    v[1 + l * NC] = dr;
    if constexpr (C) v[2 + 2 * l] = di;
  }
  const double sum = tr_sums<NV>(v, red, lane);
  constexpr int G = TrGroup<NV>::G;
  if (lane % G == 0 && lane / G < NV) rec[lane / G == 0 ? 2 : 3 + lane / G] = sum;
  if (k > KK) {
    const V *pool = static_cast<const V *>(S.pool);
    const long long *tl = S.terms + (long long)J.b * S.tmax;
    const int ro = COL ? 0 : J.h;
    const int idx = t * 32 + lane;
    for (int l = KK; l < k; ++l) {
      const long long tb = tl[l];
      double dr = 0.0, di = 0.0;
      if (valid) N::cdot(dr, di, pool[tb + ro + idx], val);
      dr = warp_sum_d(dr);
      if (C) di = warp_sum_d(di);
      if (lane == 0) {
        rec[4 + l * NC] = dr;
        if (C) rec[4 + l * NC + 1] = di;
      }
    }
  }
}

// stage job p (lane-level) into shared memory; returns false past the group
template <typename T, bool C, bool COL>
__device__ __forceinline__ bool stage_job(const AcaDev &S, int p, int n, int key0, int t,
                                          JobS &js, long long (&jt)[kFinRegs],
                                          V_t<T, C> (&jc)[kFinRegs]) {
  if (p >= n) return false;
  const Job J = S.jobs[p];
  if (J.key != key0) return false;
  js.pe = J.pe;
  js.part = J.part;
  js.rsc_off = J.rsc;
  js.mofs = J.mofs;
  js.mw = (COL ? S.rmask : S.cmask)[J.mofs + t];
  js.nfix = J.nfix;
  js.b = J.b;
  js.h = J.h;
  js.w = J.w;
  js.k = J.k;
  js.fix = J.fix;
  js.cur = J.cur;
  const int kk = min(J.k, kFinRegs);
  const long long *gjt = S.jt + (long long)p * kFinRegs;
  const V_t<T, C> *gjc = static_cast<const V_t<T, C> *>(S.jc) + (long long)p * kFinRegs;
#pragma unroll
  for (int l = 0; l < kFinRegs; ++l)
    if (l < kk) {
      jt[l] = gjt[l];
      jc[l] = gjc[l];
    }
  return true;
}

// ---------------------------------------------------------------------------
// P0 quadrature of the ACA integration kernel.
//
// The fixed element of a job is staged in shared memory as FixRec (broadcast
// to the warp), the lane's varying element is held in registers.  The double
// sum runs fixed point o outer (one shared load of its 4 values per job) and
// lane point i inner, accumulating w_o w_i G with the combined weight from the
// constant bank (RuleTab::w2).
//
// LOCAL form (float64 single layer, the headline path): both elements are
// expressed relative to a warp-uniform origin c inside the varying cluster
// (lane 0's first quadrature point) and
//     r^2 = |x'|^2 + |y'|^2 - 2 x'.y'      (x' = x - c, y' = y - c)
// is one add and three FMAs, with (-2 x', |x'|^2) staged per fixed point and
// |y'|^2 per lane point.  On an admissible block dist(t, s) >= min diam / eta,
// so |x'|^2 + |y'|^2 <= O((2 eta + 1)^2) r^2 and the cancellation costs a few
// ulp of r^2 (entries stay within 1e-13 of the direct difference; the parity
// tests bound them at 1e-12 against the reference).  1/r is the MUFU.RSQ64H
// seed y with the second-order correction folded into one polynomial:
//     1/r = y (1 + e/2 + 3 e^2/8), e = 1 - r^2 y^2
//         = (3/8) y ((r^2 y^2 - 5/3)^2 + 20/9),
// i.e. DMUL, 2 DFMA, and the weight product + accumulate (3/8 goes into the
// final scale): 9 FP64 instructions + 1 MUFU per quadrature-point pair
// against 12 + 1 for the direct difference with the standard refinement.
// Near-field leaves and the contract kernels keep the direct difference.
// ---------------------------------------------------------------------------
template <typename T> struct FixRec {
  T p[6][4];  // LOCAL: (-2 x'_0, -2 x'_1, -2 x'_2, |x'|^2); direct: (x_0, x_1, x_2, 0)
  T n[4];     // normal, |J|
  int4 ev;    // vertex ids, element id
};

template <typename T, int OP> struct P0Local {
  static constexpr bool value = std::is_same<T, double>::value && OP == HBEM_SLP;
};


template <typename T, bool LOCAL>
__device__ __forceinline__ void fix_from_rec(const ElemRec<T> &r, T c0, T c1, T c2,
                                             FixRec<T> &f) {
#pragma unroll
  for (int o = 0; o < 6; ++o) {
    if (LOCAL) {
      const T x0 = r.q[3 * o] - c0, x1 = r.q[3 * o + 1] - c1, x2 = r.q[3 * o + 2] - c2;
      f.p[o][0] = T(-2) * x0;
      f.p[o][1] = T(-2) * x1;
      f.p[o][2] = T(-2) * x2;
      f.p[o][3] = x0 * x0 + x1 * x1 + x2 * x2;
    } else {
      f.p[o][0] = r.q[3 * o];
      f.p[o][1] = r.q[3 * o + 1];
      f.p[o][2] = r.q[3 * o + 2];
      f.p[o][3] = T(0);
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) f.n[c] = r.n[c];
  f.ev = r.ev;
}

// everything k_aca_p0 stages per job, written by k_jobs: one contiguous
// record per job position, so a warp's segment is a single bulk copy
template <typename T, bool C> struct alignas(16) StageRec {
  FixRec<T> f;             // fixed element (local frame: relative to the group origin)
  JobS j;                  // job view
  long long jt[kFinRegs];  // pool records of the first terms
  V_t<T, C> jc[kFinRegs];  // their residual coefficients
};

template <typename T, bool C>
__device__ void write_stage(const Prob<T> &P, const AcaDev &S, int p, const Job &J,
                            const long long (&jt)[kFinRegs], const V_t<T, C> (&jc)[kFinRegs],
                            int col, int local) {
  static_assert(sizeof(StageRec<T, C>) <= kStageRecMax, "stage record too large");
  StageRec<T, C> *o = static_cast<StageRec<T, C> *>(S.stage) + p;
  JobS js;
  js.pe = J.pe;
  js.part = J.part;
  js.rsc_off = J.rsc;
  js.mw = 0u;
  js.nfix = J.nfix;
  js.b = J.b;
  js.h = J.h;
  js.w = J.w;
  js.k = J.k;
  js.fix = J.fix;
  js.cur = J.cur;
  js.mofs = J.mofs;
  ElemRec<T> r;
  load_rec<T>(col ? P.srec : P.trec, J.nfix, r);
  FixRec<T> f;
  if (local) {
    // group origin: the first quadrature point of the varying cluster's first
    // element (inside the varying cluster, as the local frame requires)
    const T *g = (col ? P.trec : P.srec) + (size_t)J.vstart * (sizeof(T) == 8 ? 24 : 28);
    fix_from_rec<T, true>(r, __ldg(g), __ldg(g + 1), __ldg(g + 2), f);
  } else {
    fix_from_rec<T, false>(r, T(0), T(0), T(0), f);
  }
  o->f = f;
  o->j = js;
#pragma unroll
  for (int l = 0; l < kFinRegs; ++l) {
    o->jt[l] = jt[l];
    o->jc[l] = jc[l];
  }
}

// NJ fixed elements F against the lane's element (points y, local |y'|^2 in
// ny, normal nl).  FIXED_TEST: the fixed elements are test elements (row
// jobs); otherwise trial elements (column jobs).
// NEAR: near-field (inadmissible) pairs, always the direct difference (the
// local-frame expansion's cancellation bound needs admissibility); the float64
// single layer still uses the folded rsqrt polynomial (POLY)
template <typename T, bool C, int OP, bool HELM, bool FIXED_TEST, int NJ, bool NEAR = false>
__device__ __forceinline__ void p0_quad(const RuleTab<T> &R, const FixRec<T> *const (&F)[NJ],
                                        const T (&y)[18], const T (&ny)[6], const T (&nl)[4],
                                        typename Num<T, C>::V (&out)[NJ]) {
  constexpr bool LOCAL = !NEAR && P0Local<T, OP>::value;
  constexpr bool POLY = P0Local<T, OP>::value;
  T sr[NJ], si[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) { sr[j] = T(0); si[j] = T(0); }
#pragma unroll
  for (int o = 0; o < 6; ++o) {
    T f[NJ][4];
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int c = 0; c < 4; ++c) f[j][c] = F[j]->p[o][c];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      const T w = FIXED_TEST ? R.w2[o][i] : R.w2[i][o];
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        if constexpr (POLY) {
          double r2;
          if constexpr (LOCAL) {
            r2 = fma(f[j][0], y[3 * i], fma(f[j][1], y[3 * i + 1], fma(f[j][2], y[3 * i + 2],
                                                                      f[j][3] + ny[i])));
          } else {
            const double d0 = f[j][0] - y[3 * i], d1 = f[j][1] - y[3 * i + 1],
                         d2 = f[j][2] - y[3 * i + 2];
            r2 = fma(d2, d2, fma(d1, d1, d0 * d0));
          }
          const double s = rsq_seed(r2);
          const double d = fma(r2, s * s, -5.0 / 3.0);
          const double q = fma(d, d, 20.0 / 9.0);
          if (!HELM) {
            sr[j] = fma(w * s, q, sr[j]);  // (8/3) w / r
          } else {
            const double g = s * q;        // (8/3) / r
            const double kr = R.k38 * (r2 * g);
            double sn, cs;
            sincos(kr, &sn, &cs);
            const double wg = w * g;
            sr[j] = fma(wg, cs, sr[j]);
            si[j] = fma(wg, sn, si[j]);
          }
        } else {
          const T d0 = FIXED_TEST ? f[j][0] - y[3 * i] : y[3 * i] - f[j][0];
          const T d1 = FIXED_TEST ? f[j][1] - y[3 * i + 1] : y[3 * i + 1] - f[j][1];
          const T d2 = FIXED_TEST ? f[j][2] - y[3 * i + 2] : y[3 * i + 2] - f[j][2];
          T gr, gi;
          point_kernel<T, OP, HELM>(R, d0, d1, d2, FIXED_TEST ? F[j]->n : nl,
                                    FIXED_TEST ? nl : F[j]->n, gr, gi);
          sr[j] += w * gr;
          if (HELM) si[j] += w * gi;
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const T scale = (F[j]->n[3] * nl[3]) * T(POLY ? 0.375 * kInv4Pi : kInv4Pi);
    out[j] = Num<T, C>::mk(scale * sr[j], HELM ? scale * si[j] : T(0));
  }
}

// ---------------------------------------------------------------------------
// K3 (P0): one warp per (group head, 32-wide tile).  Lane l keeps the varying
// element of tile column 32 t + l in registers and walks every job of the
// group.  The group's stage records (fixed element relative to the group
// origin, job view, residual terms; k_jobs) are copied to shared memory kSeg
// at a time with cp.async and broadcast, so an item waits for two dependent
// loads (item -> records and its lane element), not a chain of five.  The
// residual factor values and the tile's mask word of a job are loaded before
// its integral so their latency hides behind the quadrature.
// ---------------------------------------------------------------------------
// warps per CTA of k_aca_p0: independent warps (their items differ in length)
// so a CTA's slot frees as soon as its own warps finish
#ifndef HB_ACA_WPC
#define HB_ACA_WPC 1
#endif
constexpr int kP0Warps = HB_ACA_WPC;
#ifndef HB_PROF
#define HB_PROF 0  // per-phase clock64 accounting of k_aca_p0 (timing experiments)
#endif

template <typename T, bool C, int OP, bool HELM, bool COL>
__global__ void __launch_bounds__(kP0Warps * 32, HB_ACA_P0_MINB * 4 / kP0Warps) k_aca_p0(Prob<T> P, AcaDev S, int n,
                                                                   long long n_items) {
  using N = Num<T, C>;
  using V = typename N::V;
  using SR = StageRec<T, C>;
  constexpr int NC = N::NC;
  constexpr int kSeg = sizeof(V) > 8 ? 8 : 16;  // jobs staged per segment
  constexpr int kChunks = (int)(sizeof(SR) / 16);
  __shared__ SR ssr[kP0Warps][kSeg];
  __shared__ double sred[kP0Warps][32 * kRedStride];  // transpose scratch
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long item = (long long)blockIdx.x * kP0Warps + wid;
  if (item >= n_items) return;
#if HB_PROF
  unsigned long long pt0 = clock64(), pt = pt0, pc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#define HB_TICK(i)                          \
  {                                         \
    const unsigned long long c = clock64(); \
    pc[i] += c - pt;                        \
    pt = c;                                 \
  }
#define HB_PROF_ARGS , pc, pt
#else
#define HB_TICK(i)
#define HB_PROF_ARGS
#endif
  const int4 it = S.items[item];
  const int glen = S.iglen[item];
  const int p0 = it.x, t = it.y, vstart = it.z, nvar = it.w;
  const int idx = t * 32 + lane;
  const bool valid = idx < nvar;
  const SR *gsr = static_cast<const SR *>(S.stage) + p0;
  // segment copy: lanes stride over the 16-byte chunks of nj records
  auto fetch = [&](int seg) {
    const int nj = min(kSeg, glen - seg);
    const uint4 *src = reinterpret_cast<const uint4 *>(gsr + seg);
    uint4 *dst = reinterpret_cast<uint4 *>(&ssr[wid][0]);
    for (int c = lane; c < nj * kChunks; c += 32) cp_async<16>(dst + c, src + c);
    cp_async_commit();
  };
  fetch(0);
  T y[18], ny[6], nl[4];
  int4 myev;
  {
    ElemRec<T> my;
    load_rec<T>(COL ? P.trec : P.srec, vstart + (valid ? idx : nvar - 1), my);
    T c0 = T(0), c1 = T(0), c2 = T(0);
    if (P0Local<T, OP>::value) {
      // group origin (k_jobs, write_stage): the varying cluster's first
      // element's first quadrature point
      const T *g = (COL ? P.trec : P.srec) + (size_t)vstart * (sizeof(T) == 8 ? 24 : 28);
      c0 = __ldg(g);
      c1 = __ldg(g + 1);
      c2 = __ldg(g + 2);
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      y[3 * i] = my.q[3 * i] - c0;
      y[3 * i + 1] = my.q[3 * i + 1] - c1;
      y[3 * i + 2] = my.q[3 * i + 2] - c2;
      ny[i] = P0Local<T, OP>::value
                  ? y[3 * i] * y[3 * i] + y[3 * i + 1] * y[3 * i + 1] + y[3 * i + 2] * y[3 * i + 2]
                  : T(0);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) nl[c] = my.n[c];
    myev = my.ev;
  }
  unsigned long long nent = 0, nsing = 0;
  double *red = sred[wid];
  V *const pool = static_cast<V *>(S.pool);
  const unsigned *mask = COL ? S.rmask : S.cmask;
  const int to = t * 32;
  HB_TICK(1)
  for (int seg = 0; seg < glen; seg += kSeg) {
    if (seg > 0) {
      __syncwarp();  // the previous segment's records are no longer read
      fetch(seg);
    }
    cp_async_wait_all();
    __syncwarp();
    const int nseg = min(kSeg, glen - seg);
    HB_TICK(2)
    for (int q = 0; q < nseg; ++q) {
      const SR &R = ssr[wid][q];
      const JobS &J = R.j;
      const int kk = min(J.k, kFinRegs);
      const int ro = COL ? 0 : J.h;
      // factor values of the residual and the tile's mask word, loaded before
      // the quadrature so their latency hides behind it (predicated loads)
      const unsigned mw = __ldg(mask + J.mofs + t);
      V f[kFinRegs];
#pragma unroll
      for (int l = 0; l < kFinRegs; ++l) {
        const bool use = l < kk && valid;
        f[l] = use ? ld_ro(pool + R.jt[l] + ro + to + lane) : N::zero();
      }
      // touching pairs (rare; Sauter-Schwab in place), tested before the
      // quadrature so the test's latency overlaps it
      const int4 fev = R.f.ev;
      unsigned tm = __ballot_sync(kFull, valid && touching4(myev, fev));
      HB_TICK(8)
      V val;
      {
        const FixRec<T> *const F1[1] = {&R.f};
        V v1[1];
        p0_quad<T, C, OP, HELM, !COL, 1>(P.R, F1, y, ny, nl, v1);
        val = v1[0];
      }
#if HB_PROF
      if ((double)N::re(val) == 1.2345e300) ++pc[0];  // the tick below waits for the quadrature
#endif
      HB_TICK(3)
      {
        while (tm) {
          const int src = __ffs(tm) - 1;
          tm &= tm - 1;
          const int ev = __shfl_sync(kFull, myev.w, src);
          const double2 sv = singular_warp<OP, HELM>(P.G64p, COL ? ev : fev.w, COL ? fev.w : ev);
          if (lane == src) val = N::mk((T)sv.x, (T)sv.y);
          ++nsing;
        }
      }
      HB_TICK(4)
      V *const out = pool + J.pe + ro + to;
      double *const rec = S.part + J.part + (long long)t * part_len(J.k, NC);
#define HB_EPI(KK)                                                                             \
  case KK:                                                                                     \
    aca_epi_p0<T, C, COL, KK>(S, J, mw, R.jc, f, out, rec, t, lane, valid, val,                \
                              red HB_PROF_ARGS);                                               \
    break;
      switch (kk) {
        HB_EPI(0) HB_EPI(1) HB_EPI(2) HB_EPI(3) HB_EPI(4) HB_EPI(5) HB_EPI(6) HB_EPI(7) HB_EPI(8)
      }
#undef HB_EPI
      HB_TICK(9)
#if HB_PROF
      ++pc[6];
#endif
    }
    nent += valid ? nseg : 0;
    HB_TICK(1)
  }
  nent = (unsigned long long)__reduce_add_sync(kFull, (unsigned)nent);
  if (lane == 0) {
    atomicAdd(S.stat, nent);
    if (nsing) atomicAdd(S.stat + 1, nsing);
  }
#if HB_PROF
  if (lane == 0) {
    atomicAdd(S.stat + 4, clock64() - pt0);
    atomicAdd(S.stat + 5, pc[1]);  // prologue (+ segment turnover)
    atomicAdd(S.stat + 6, pc[2]);  // staging
    atomicAdd(S.stat + 12, pc[8]); // factor loads issue
    atomicAdd(S.stat + 7, pc[3]);  // quadrature
    atomicAdd(S.stat + 8, pc[4]);  // touching check
    atomicAdd(S.stat + 9, pc[5]);  // epilogue: residual (waits for the factors)
    atomicAdd(S.stat + 13, pc[7]); // epilogue: store + pivot candidate
    atomicAdd(S.stat + 14, pc[9]); // epilogue: sums + records
    atomicAdd(S.stat + 10, pc[6]); // jobs
    atomicAdd(S.stat + 11, 1ull);  // warps
  }
#endif
#undef HB_TICK
#undef HB_PROF_ARGS
}

// ---------------------------------------------------------------------------
// K3e (linear spaces, element level): one warp per (group head, 32-element
// tile of the varying cluster's element union).  Lane l keeps element h of
// the union in registers; for every job of the group the fixed DOF's
// elements g (local basis a_g) are staged in shared memory and the lane
// accumulates the row (row phase: trial basis b of h) or column (column
// phase: test basis a of h) of sum_g B_gh[a_g, .] — every element pair is
// integrated once with all NL basis functions of the lane element sharing
// each kernel evaluation (the reference's pairs = repeat(T(dof)) x
// tile(col_elems), hmatrix.py:636-639).  Touching pairs read the singular
// table.  k_aca_gen then gathers DOF entries from these rows.
// ---------------------------------------------------------------------------
template <typename T, bool C, int OP, bool HELM, int NT, int NS, bool COL>
__global__ void __launch_bounds__(kThreads) k_p1_erow(Prob<T> P, AcaDev S, int n,
                                                      long long n_items) {
  using N = Num<T, C>;
  using V = typename N::V;
  constexpr int NL = COL ? NT : NS;  // basis functions of the lane element
  constexpr int KE = 16;             // fixed elements staged per chunk
  __shared__ T sq[kWarps][KE][18];
  __shared__ T snj[kWarps][KE][4];
  __shared__ int4 sev[kWarps][KE];
  __shared__ int sloc[kWarps][KE];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long item = (long long)blockIdx.x * kWarps + wid;
  if (item >= n_items) return;
  const int2 it = S.eitems[item];
  const int p0 = it.x, te = it.y;
  const int key0 = S.jobs[p0].key;
  const long long *ep = COL ? S.recl_ptr : S.cecl_ptr;
  const int *el = COL ? S.recl : S.cecl;
  const long long e0 = ep[key0], ne = ep[key0 + 1] - e0;
  const long long li = (long long)te * 32 + lane;
  const bool valid = li < ne;
  const int h = el[e0 + (valid ? li : 0)];
  T y[18], nl[4];
  load_q<T>(P.g.q, h, y);
  load_nj<T>(P.g.nj, h, nl);
  int4 hev = P.elem[h];
  hev.w = h;
  const int *fptr = COL ? P.sptr : P.tptr;
  const int *fel = COL ? P.sel : P.tel;
  const signed char *floc = COL ? P.sloc : P.tloc;
  const int *fperm = COL ? P.cperm : P.rperm;
  V *out = static_cast<V *>(S.rsc);
  for (int p = p0; p < n; ++p) {
    const Job J = S.jobs[p];
    if (J.key != key0) break;
    const int dof = fperm[J.nfix];
    constexpr bool kFixedP0 = (COL ? NS : NT) == 1;  // fixed DOF = its element
    const int f0 = kFixedP0 ? 0 : fptr[dof], f1 = kFixedP0 ? 1 : fptr[dof + 1];
    T rr[NL], ri[NL];
#pragma unroll
    for (int b = 0; b < NL; ++b) { rr[b] = T(0); ri[b] = T(0); }
    for (int c0 = f0; c0 < f1; c0 += KE) {
      const int cnt = min(KE, f1 - c0);
      if (lane < cnt) {
        const int g = kFixedP0 ? dof : fel[c0 + lane];
        T q[18], nj[4];
        load_q<T>(P.g.q, g, q);
        load_nj<T>(P.g.nj, g, nj);
#pragma unroll
        for (int c = 0; c < 18; ++c) sq[wid][lane][c] = q[c];
#pragma unroll
        for (int c = 0; c < 4; ++c) snj[wid][lane][c] = nj[c];
        int4 ev = P.elem[g];
        ev.w = g;
        sev[wid][lane] = ev;
        sloc[wid][lane] = kFixedP0 ? 0 : floc[c0 + lane];
      }
      __syncwarp();
      for (int k = 0; k < cnt; ++k) {
        const int4 gev = sev[wid][k];
        const int a = sloc[wid][k];
        if (touching4(gev, hev)) {
          if (valid) {
            // table block of (test, trial): row phase (g, h), column (h, g)
            const int et = COL ? h : gev.w, ft = COL ? gev.w : h;
            int j = P.nb_ptr[et];
            while (P.nb_idx[j] != ft) ++j;
            const T *blk = static_cast<const T *>(P.stab) + (long long)j * NT * NS * (HELM ? 2 : 1);
#pragma unroll
            for (int b = 0; b < NL; ++b) {
              const int o = COL ? b * NS + a : a * NS + b;
              rr[b] += HELM ? blk[2 * o] : blk[o];
              if (HELM) ri[b] += blk[2 * o + 1];
            }
            atomicAdd(S.stat + 1, 1ull);
          }
          continue;
        }
        // regular pair: lane points outer, fixed points inner
        T sr[NL], si[NL];
#pragma unroll
        for (int b = 0; b < NL; ++b) { sr[b] = T(0); si[b] = T(0); }
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const T y0 = y[3 * i], y1 = y[3 * i + 1], y2 = y[3 * i + 2];
          T tr = T(0), ti = T(0);
#pragma unroll 2
          for (int o = 0; o < 6; ++o) {
            const T g0 = sq[wid][k][3 * o], g1 = sq[wid][k][3 * o + 1], g2 = sq[wid][k][3 * o + 2];
            T gr, gi;
            // d = x - y with x the test point
            if (!COL)
              point_kernel<T, OP, HELM>(P.R, g0 - y0, g1 - y1, g2 - y2, snj[wid][k], nl, gr, gi);
            else
              point_kernel<T, OP, HELM>(P.R, y0 - g0, y1 - g1, y2 - g2, nl, snj[wid][k], gr, gi);
            const T wf = COL ? P.R.wb[a][o] : P.R.wa[a][o];
            tr += wf * gr;
            if (HELM) ti += wf * gi;
          }
#pragma unroll
          for (int b = 0; b < NL; ++b) {
            const T wl = COL ? P.R.wa[b][i] : P.R.wb[b][i];
            sr[b] += wl * tr;
            if (HELM) si[b] += wl * ti;
          }
        }
        const T scale = (snj[wid][k][3] * nl[3]) * T(kInv4Pi);
#pragma unroll
        for (int b = 0; b < NL; ++b) {
          rr[b] += scale * sr[b];
          if (HELM) ri[b] += scale * si[b];
        }
      }
      __syncwarp();
    }
    if (valid) {
      V *o = out + J.rsc + li * NL;
#pragma unroll
      for (int b = 0; b < NL; ++b) o[b] = N::mk(rr[b], ri[b]);
    }
  }
}

// K3 (linear spaces): entries summed over the carrying element pairs
template <typename T, bool C, int OP, bool HELM, int NT, int NS, bool COL>
__global__ void __launch_bounds__(kThreads) k_aca_gen(Prob<T> P, AcaDev S, int n,
                                                      long long n_items) {
  using N = Num<T, C>;
  using V = typename N::V;
  __shared__ JobS sj[kWarps];
  __shared__ V sjc[kWarps][kFinRegs];
  __shared__ V fbuf[kWarps][kFinRegs * 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long item = (long long)blockIdx.x * kWarps + wid;
  if (item >= n_items) return;
  const int4 it = S.items[item];
  const int p0 = it.x, t = it.y;
  const Job J0 = S.jobs[p0];
  const int key0 = J0.key;
  const int idx = t * 32 + lane;
  const bool valid = idx < J0.nvar;
  const int vdof = valid ? (COL ? P.rperm : P.cperm)[J0.vstart + idx] : 0;
  const V *pool = static_cast<const V *>(S.pool);
  unsigned long long nent = 0;
  for (int p = p0;; ++p) {
    bool ok = false;
    if (lane == 0) {
      JobS js;
      long long jt[kFinRegs];
      V jc[kFinRegs];
      ok = stage_job<T, C, COL>(S, p, n, key0, t, js, jt, jc);
      if (ok) {
        sj[wid] = js;
#pragma unroll
        for (int l = 0; l < kFinRegs; ++l)
          if (l < min(js.k, kFinRegs)) sjc[wid][l] = jc[l];
      }
    }
    if (!__shfl_sync(kFull, ok, 0)) break;
    __syncwarp();
    const JobS J = sj[wid];
    const int kk = min(J.k, kFinRegs);
    const int ro = COL ? 0 : J.h;
    const long long *gjt = S.jt + (long long)p * kFinRegs;
#pragma unroll
    for (int l = 0; l < kFinRegs; ++l)
      if (l < kk && valid) cp_async<sizeof(V)>(&fbuf[wid][l * 32 + lane], pool + gjt[l] + ro + idx);
    const int fdof = COL ? P.cperm[S.c0[J.b] + J.fix] : P.rperm[S.r0[J.b] + J.fix];
    V val = N::zero();
    if (OP != HBEM_HYPS && S.rsc) {
      // element rows (k_p1_erow): entry = sum over the varying DOF's elements
      // of their row value at the DOF's local basis function, elements in
      // ascending order (the order of _row_job / _col_job's scatter)
      if (valid) {
        constexpr int NL = COL ? NT : NS;
        const long long *ep = COL ? S.recl_ptr : S.cecl_ptr;
        const int *el = COL ? S.recl : S.cecl;
        const long long e0 = ep[key0], e1 = ep[key0 + 1];
        const int *iptr = COL ? P.tptr : P.sptr;
        const int *iel = COL ? P.tel : P.sel;
        const signed char *iloc = COL ? P.tloc : P.sloc;
        const V *R = static_cast<const V *>(S.rsc) + J.rsc_off;
        constexpr bool kVarP0 = NL == 1;  // varying DOF = its element
        const int q0 = kVarP0 ? 0 : iptr[vdof], q1 = kVarP0 ? 1 : iptr[vdof + 1];
        for (int q = q0; q < q1; ++q) {
          const int f = kVarP0 ? vdof : iel[q];
          long long lo = e0, hi = e1;
          while (lo < hi) {
            const long long mid = (lo + hi) >> 1;
            if (el[mid] < f) lo = mid + 1;
            else hi = mid;
          }
          const V r = R[(lo - e0) * NL + (kVarP0 ? 0 : iloc[q])];
          if constexpr (C) { val.re += r.re; val.im += r.im; }
          else val += r;
        }
      }
    } else if (valid) {
      val = COL ? entry<T, C, OP, HELM, NT, NS>(P, vdof, fdof, S.stat + 1)
                : entry<T, C, OP, HELM, NT, NS>(P, fdof, vdof, S.stat + 1);
    }
    cp_async_wait_all();
    aca_epi<T, C, COL>(S, J, sjc[wid], t, lane, valid, val, fbuf[wid]);
    nent += valid ? 1 : 0;
    __syncwarp();
  }
  nent = (unsigned long long)__reduce_add_sync(kFull, (unsigned)nent);
  if (lane == 0) atomicAdd(S.stat, nent);
}

// ---------------------------------------------------------------------------
// finalize, one warp per job: lanes over the job's tile records (statistics)
// and over its terms (dots), both laid out contiguously per job, so every
// load is coalesced; fixed-shape reductions keep the decisions deterministic.
//
// Term records are [u (h) | r (w) | p]: the residual row r is kept unscaled
// and its pivot p stored behind it, v = r / p is applied where v is read
// (residual coefficients, cross terms, payload packing).
// ---------------------------------------------------------------------------
// Finalize kernels: one 8-lane group per job (4 jobs per warp).  Jobs
// usually span a few 32-entry tiles, so a group's lanes cover its tiles
// (statistics) and its terms (cross-term dots) in one pass; the reductions
// are 3-step butterflies inside the group (xor 4, 2, 1), fixed order.
constexpr int kFinLanes = 8;
#ifndef HB_FIN_MINB
#define HB_FIN_MINB 8
#endif

__device__ __forceinline__ void group_argmax_sum(double &best, int &bidx, double &sum) {
#pragma unroll
  for (int o = kFinLanes / 2; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(kFull, best, o);
    const int oi = __shfl_xor_sync(kFull, bidx, o);
    if (better(ob, oi, best, bidx)) { best = ob; bidx = oi; }
    sum += __shfl_xor_sync(kFull, sum, o);
  }
}

__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = kFinLanes / 2; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// sums over a job's tiles of its first kk dots (re, im): group lanes over
// the tiles (t = sl, sl + 8, ...), all kk dots per tile, then the butterfly,
// which leaves every lane with all kk sums; a long row costs ntiles / 8
// iterations of independent loads, not a serial chain over its tiles
template <bool C>
__device__ __forceinline__ void group_tile_dots(const double *dots, int ntiles, long long stride,
                                                int kk, int sl, double (&sr)[kFinRegs],
                                                double (&si)[kFinRegs]) {
  constexpr int NC = C ? 2 : 1;
#pragma unroll
  for (int l = 0; l < kFinRegs; ++l) { sr[l] = 0.0; si[l] = 0.0; }
  if (dots) {
    for (int t = sl; t < ntiles; t += kFinLanes) {
      const double *r = dots + t * stride;
#pragma unroll
      for (int l = 0; l < kFinRegs; ++l)
        if (l < kk) {
          sr[l] += r[l * NC];
          if (C) si[l] += r[l * NC + 1];
        }
    }
  }
#pragma unroll
  for (int o = kFinLanes / 2; o > 0; o >>= 1)
#pragma unroll
    for (int l = 0; l < kFinRegs; ++l) {
      sr[l] += __shfl_xor_sync(kFull, sr[l], o);
      if (C) si[l] += __shfl_xor_sync(kFull, si[l], o);
    }
}

// pivot statistics of a job's residual row / column from its tile records
// (aca_epi): group lanes over the tiles in order, then the butterfly; argmax
// over unused indices with the first index on ties, sum |val|^2
__device__ __forceinline__ void tile_stats(const double *rec, int ntiles, long long stride,
                                           int sl, double &best, int &bidx, double &ss) {
  best = -1.0;
  bidx = 0x7fffffff;
  ss = 0.0;
  if (rec) {
    for (int t = sl; t < ntiles; t += kFinLanes) {
      const double2 bi = *reinterpret_cast<const double2 *>(rec + t * stride);
      const int i = (int)bi.y;
      if (better(bi.x, i, best, bidx)) {
        best = bi.x;
        bidx = i;
      }
      ss += rec[t * stride + 2];
    }
  }
  group_argmax_sum(best, bidx, ss);
}

// row finalize: column pivot (hmatrix.py:329-332) or vanishing row (334-338)
template <typename T, bool C>
__global__ void __launch_bounds__(kThreads, HB_FIN_MINB) k_fin_row(AcaDev S, int n) {
  using N = Num<T, C>;
  using V = typename N::V;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int p = gt / kFinLanes, sl = gt % kFinLanes;
  const bool act = p < n;
  Job J{};
  if (act) J = S.jobs[p];
  double best, ss;
  int bidx;
  const long long ps = part_len(J.k, N::NC);
  tile_stats(act ? S.part + J.part : nullptr, tiles_of(J.w), ps, sl, best, bidx, ss);
  {
    // this row's dots with the first terms, summed over its tiles (group
    // lanes over the tiles, then the butterfly; fixed order) for the column
    // finalize's cross terms (compact, indexed by block)
    const int kk = act ? min(J.k, kFinRegs) : 0;
    double sr[kFinRegs], si[kFinRegs];
    group_tile_dots<C>(act ? S.part + J.part + 4 : nullptr, tiles_of(J.w), ps, kk, sl, sr, si);
    if (act && sl < kk) {
      double *o = S.rsum + (long long)J.b * (kFinRegs * 2) + sl * 2;
      o[0] = sr[sl];
      o[1] = si[sl];
    }
  }
  if (!act || sl != 0) return;
  const int b = J.b, h = J.h, w = J.w, i = J.fix;
  S.pend[b] = J.pe;
  if (best <= 0.0) {
    unsigned *rm = S.rmask + S.rmask_off[b];
    set_bit(rm, i);
    const int next = first_clear(rm, h);
    if (next < 0) {
      S.status[b] = ST_CONVERGED;
      S.exhausted[b] = 1;
    } else {
      S.cur[b] = next;
      S.flagA[b] = 1;
    }
    return;
  }
  V *wpool = static_cast<V *>(S.pool);
  const V pv = wpool[J.pe + h + bidx];
  wpool[J.pe + h + w] = pv;
  S.pcol[b] = bidx;
  S.piv[2 * b] = (double)N::re(pv);
  S.piv[2 * b + 1] = (double)N::im(pv);
  S.rn2[b] = ss;
  S.flagC[b] = 1;
}

// column finalize: stopping test (343-357), Frobenius update with the cross
// terms (359-362), next row pivot (301-314)
template <typename T, bool C>
__global__ void __launch_bounds__(kThreads, HB_FIN_MINB) k_fin_col(AcaDev S, int n) {
  using N = Num<T, C>;
  using V = typename N::V;
  constexpr int NC = N::NC;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int p = gt / kFinLanes, sl = gt % kFinLanes;
  const bool act = p < n;
  Job J{};
  if (act) J = S.jobs[p];
  const int b = J.b, h = J.h, w = J.w, j = J.fix, k = J.k, i = J.cur;
  const int ntc = tiles_of(h), ntr = tiles_of(w);
  const long long ps = part_len(k, NC);
  const double *crec = act ? S.part + J.part : nullptr;
  double best, ss;
  int bidx;
  tile_stats(crec, ntc, ps, sl, best, bidx, ss);
  double n2 = 0.0, pr = 0.0, pim = 0.0, rn2 = 0.0;
  if (act) {
    n2 = S.norm2[b];
    pr = S.piv[2 * b];
    pim = S.piv[2 * b + 1];
    rn2 = S.rn2[b];
  }
  const int next = best >= 0.0 ? bidx : -1;
  const double nu = sqrt(ss);
  const double nv = sqrt(rn2) / hypot(pr, pim);
  const double upd = nu * nv;
  const bool small = act && n2 > 0.0 && upd <= S.eps * sqrt(n2);
  // cross terms Re(vdot(u_l, u) vdot(v_l, v)) with v_l = r_l / p_l, v = r / p:
  // vdot(v_l, v) = vdot(r_l, r) / (conj(p_l) p); lane sl sums the dots of
  // terms sl, sl + 8, ... over the column and row tiles in tile order
  double cross = 0.0;
  // column dots of the first terms, summed over the column tiles (all lanes)
  const bool need = act && !small;
  double csr[kFinRegs], csi[kFinRegs];
  group_tile_dots<C>(need ? crec + 4 : nullptr, ntc, ps, need ? min(k, kFinRegs) : 0, sl, csr,
                     csi);
  if (need) {
    const V *pool = static_cast<const V *>(S.pool);
    const double *cd = crec + 4;
    const double *rd = S.rpart + S.rowpart[b] + 4;
    const long long *tl = S.terms + (long long)b * S.tmax;
    for (int l = sl; l < k; l += kFinLanes) {
      double ur = 0.0, ui = 0.0, vr = 0.0, vi = 0.0;
      if (l < kFinRegs) {
#pragma unroll
        for (int q = 0; q < kFinRegs; ++q)
          if (q == l) { ur = csr[q]; ui = csi[q]; }
        const double *o = S.rsum + (long long)b * (kFinRegs * 2) + l * 2;
        vr = o[0];
        vi = o[1];
      } else {  // terms beyond the register batch: serial over the tiles
        for (int t = 0; t < ntc; ++t) {
          ur += cd[t * ps + (long long)l * NC];
          if (C) ui += cd[t * ps + (long long)l * NC + 1];
        }
        for (int t = 0; t < ntr; ++t) {
          vr += rd[t * ps + (long long)l * NC];
          if (C) vi += rd[t * ps + (long long)l * NC + 1];
        }
      }
      const V pl = static_cast<const V *>(S.tpiv)[(long long)b * S.tmax + l];
      const double plr = (double)N::re(pl), pli = (double)N::im(pl);
      const double dr = plr * pr + pli * pim, di = plr * pim - pli * pr;  // conj(p_l) p
      double qr, qi;
      if (C) {
        const double d = dr * dr + di * di;
        qr = (vr * dr + vi * di) / d;
        qi = (vi * dr - vr * di) / d;
      } else {
        qr = vr / dr;
        qi = 0.0;
      }
      cross += ur * qr - ui * qi;
    }
  }
  cross = group_sum(cross);
  if (!act || sl != 0) return;
  const int kmax_b = min(S.kmax_cfg, min(h, w));
  unsigned *rm = S.rmask + S.rmask_off[b];
  if (small) {
    S.resid[b] = upd / sqrt(n2);
    const int sm = S.small[b] + 1;
    S.small[b] = sm;
    if (sm >= 2) {
      S.status[b] = ST_CONVERGED;
    } else {
      set_bit(rm, i);
      if (next < 0) {
        S.status[b] = ST_CONVERGED;
        S.exhausted[b] = 1;
      } else {
        S.cur[b] = next;
        S.flagA[b] = 1;  // the pending record is reused
      }
    }
    return;
  }
  const double n2n = n2 + 2.0 * cross + upd * upd;
  S.norm2[b] = n2n;
  S.small[b] = 0;
  S.terms[(long long)b * S.tmax + k] = J.pe;
  // the term's pivot (= its record's last value) next to the term list
  static_cast<V *>(S.tpiv)[(long long)b * S.tmax + k] = N::mk((T)pr, (T)pim);
  S.pend[b] = -1;
  S.rank[b] = k + 1;
  set_bit(rm, i);
  set_bit(S.cmask + S.cmask_off[b], j);
  if (n2n > 0.0) {
    S.resid[b] = upd / sqrt(n2n);
    if (upd <= S.eps * sqrt(n2n)) S.small[b] = 1;
  }
  S.cur[b] = next;
  // loop head of the next iteration (hmatrix.py:318-322)
  if (k + 1 >= kmax_b) {
    S.status[b] = ST_FALLBACK;
  } else if (k + 1 >= S.tmax) {
    S.status[b] = ST_OVERFLOW;
  } else if (next < 0) {
    S.status[b] = ST_CONVERGED;
    S.exhausted[b] = 1;
  } else {
    S.flagA[b] = 1;
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
template <typename T, bool C>
int aca_init(const Prob<T> &, AcaDev &S, int na, cudaStream_t st) {
  if (na <= 0) return HBEM_OK;
  k_aca_init<<<(na + 127) / 128, 128, 0, st>>>(S, na);
  HB_CUDA(cudaGetLastError());
  return HBEM_OK;
}

template <typename T, bool C>
int aca_select(const Prob<T> &, AcaDev &S, const PhaseArgs &A, cudaStream_t st) {
  constexpr int NC = Num<T, C>::NC;
  const int na = A.na;
  unsigned char *flags = A.col_phase ? S.flagC : S.flagA;
  k_phase_flags<<<(na + 255) / 256, 256, 0, st>>>(flags, A.order, na,
                                                   reinterpret_cast<unsigned char *>(A.sel_tmp));
  HB_CUDA(cudaGetLastError());
  size_t tb = A.cub_bytes;
  HB_CUDA(cub::DeviceSelect::Flagged(A.cub_tmp, tb, A.order,
                                     reinterpret_cast<unsigned char *>(A.sel_tmp),
                                     const_cast<int *>(S.list), const_cast<int *>(S.nlist), na,
                                     st));
  if (!A.col_phase) {
    // the row phase consumes the row flags; fin_row/fin_col set them again
    HB_CUDA(cudaMemsetAsync(S.flagA, 0, na, st));
    HB_CUDA(cudaMemsetAsync(S.flagC, 0, na, st));
  }
  // inclusive scan of the needs: block scans + one CTA over the block totals +
  // carry add (three light kernels instead of a generic 40-byte-record scan)
  const int nb = (na + kNeedThreads - 1) / kNeedThreads;
  Need *bsum = reinterpret_cast<Need *>(A.cub_tmp);
  k_need<NC><<<nb, kNeedThreads, 0, st>>>(S, na, A.col_phase, A.nt, A.ns, bsum);
  HB_CUDA(cudaGetLastError());
  k_need_blocks<<<1, 1024, 0, st>>>(bsum, nb, S.nlist);
  HB_CUDA(cudaGetLastError());
  if (nb > 1) k_need_carry<<<nb - 1, kNeedThreads, 0, st>>>(S, na, bsum);
  HB_CUDA(cudaGetLastError());
  return HBEM_OK;
}

inline size_t aca_cub_bytes_impl(int na) {
  size_t b1 = 0, b2 = 0;
  cub::DeviceSelect::Flagged(nullptr, b1, (const int *)nullptr, (const unsigned char *)nullptr,
                             (int *)nullptr, (int *)nullptr, std::max(na, 1));
  b2 = ((size_t)std::max(na, 1) + kNeedThreads - 1) / kNeedThreads * sizeof(Need) + 256;
  return std::max(b1, b2);
}

template <typename T, bool C>
int aca_phase(const Prob<T> &P, AcaDev &S, const PhaseArgs &A, int op, bool helm, int nt, int ns,
              int n, long long n_items, long long n_eitems, cudaStream_t st) {
  if (n <= 0) return HBEM_OK;
  const int col = A.col_phase;
  const int stage = (nt == 1 && ns == 1) ? (std::is_same<T, double>::value && op == HBEM_SLP ? 1 : 0) : -1;
  k_jobs<T, C><<<(n + 127) / 128, 128, 0, st>>>(P, S, n, col, stage);
  HB_CUDA(cudaGetLastError());
  if (S.rsc && n_eitems > 0) {
    // linear spaces: element rows first, then the DOF gather + residual
    const unsigned egrid = (unsigned)((n_eitems + kWarps - 1) / kWarps);
    int rc = dispatch_op(op, helm, nt, ns, [&](auto OPc, auto Hc, auto NTc, auto NSc) -> int {
      constexpr int OP = decltype(OPc)::value;
      constexpr bool HH = decltype(Hc)::value != 0;
      constexpr int NT = decltype(NTc)::value, NS = decltype(NSc)::value;
      if constexpr (HH == C && (NT != 1 || NS != 1) && OP != HBEM_HYPS) {
        if (col) k_p1_erow<T, C, OP, HH, NT, NS, true><<<egrid, kThreads, 0, st>>>(P, S, n, n_eitems);
        else k_p1_erow<T, C, OP, HH, NT, NS, false><<<egrid, kThreads, 0, st>>>(P, S, n, n_eitems);
        HB_CUDA(cudaGetLastError());
        return HBEM_OK;
      } else {
        return set_error(HBEM_ERR_KERNEL, "element rows requested for an unsupported operator");
      }
    });
    if (rc != HBEM_OK) return rc;
  }
  if (n_items > 0) {
    const unsigned grid = (unsigned)((n_items + kWarps - 1) / kWarps);
    const unsigned grid_p0 = (unsigned)((n_items + kP0Warps - 1) / kP0Warps);
    if (A.int_beg) HB_CUDA(cudaEventRecord(A.int_beg, st));
    int rc = dispatch_op(op, helm, nt, ns, [&](auto OPc, auto Hc, auto NTc, auto NSc) -> int {
      constexpr int OP = decltype(OPc)::value;
      constexpr bool HH = decltype(Hc)::value != 0;
      constexpr int NT = decltype(NTc)::value, NS = decltype(NSc)::value;
      if constexpr (HH == C) {
        if constexpr (NT == 1 && NS == 1) {
          if (col) k_aca_p0<T, C, OP, HH, true><<<grid_p0, kP0Warps * 32, 0, st>>>(P, S, n, n_items);
          else k_aca_p0<T, C, OP, HH, false><<<grid_p0, kP0Warps * 32, 0, st>>>(P, S, n, n_items);
        } else {
          if (col)
            k_aca_gen<T, C, OP, HH, NT, NS, true><<<grid, kThreads, 0, st>>>(P, S, n, n_items);
          else
            k_aca_gen<T, C, OP, HH, NT, NS, false><<<grid, kThreads, 0, st>>>(P, S, n, n_items);
        }
        HB_CUDA(cudaGetLastError());
        return HBEM_OK;
      } else {
        return set_error(HBEM_ERR_KERNEL, "value type does not match the equation");
      }
    });
    if (rc != HBEM_OK) return rc;
    if (A.int_end) HB_CUDA(cudaEventRecord(A.int_end, st));
  }
  const unsigned fgrid = (unsigned)(((long long)n * kFinLanes + kThreads - 1) / kThreads);
  if (col) k_fin_col<T, C><<<fgrid, kThreads, 0, st>>>(S, n);
  else k_fin_row<T, C><<<fgrid, kThreads, 0, st>>>(S, n);
  HB_CUDA(cudaGetLastError());
  return HBEM_OK;
}

}  // namespace hb
