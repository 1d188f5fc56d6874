/*
 * hbem_b200 — C ABI of the B200 (sm_100a) Galerkin element-pair integrator
 * and device H-matrix assembler.
 *
 * This is the drop-in boundary for the reference's batched-integrator
 * "device" contract (/root/reference/pkg/src/hbem/backend.py:41-298) and
 * for its H-matrix leaf assembler (/root/reference/pkg/src/hbem/hmatrix.py:
 * 550-811).  Plain pointers and sizes only; no torch types.  Every entry
 * point returns an int status (HBEM_OK = 0); on failure the thread-local
 * message is available from hbem_last_error() and uses the same wording as
 * the reference exceptions so a binding can re-raise them verbatim
 * (ContractViolationError: "not disjoint", "indices"; CapacityError:
 * "weights").
 *
 * Thread safety: a context is read-only after creation; integration calls
 * on one context may be issued from several host threads concurrently
 * (each call uses its own stream and scratch), mirroring
 * backend.py:17 ("integrate_batch is read-only on the context").
 * Determinism: every pair's block is a fixed function of that pair's data
 * (no atomics on values, fixed reduction order), so results are bitwise
 * independent of batch composition and split (backend.py:15-16).
 */
#ifndef HBEM_B200_H
#define HBEM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HBEM_ABI_VERSION 1

/* status codes -> reference exception classes (errors.py:49-71) */
enum {
  HBEM_OK = 0,
  HBEM_ERR_CONTRACT = 1, /* ContractViolationError */
  HBEM_ERR_CAPACITY = 2, /* CapacityError          */
  HBEM_ERR_CONFIG = 3,   /* ConfigError            */
  HBEM_ERR_CUDA = 4,     /* device failure (AssemblyError at the caller) */
  HBEM_ERR_ARG = 5,      /* malformed argument     */
  HBEM_ERR_KERNEL = 6,   /* KernelError            */
  HBEM_ERR_MESH = 7,     /* MeshError              */
  HBEM_ERR_MESH_PARSE = 8 /* MeshParseError (line / section: hbem_gmsh_error_location) */
};

/* OperatorSpec fields (kernels.py:54-96) */
enum { HBEM_LAPLACE = 0, HBEM_HELMHOLTZ = 1 };
enum { HBEM_SLP = 0, HBEM_DLP = 1, HBEM_ADLP = 2, HBEM_HYPS = 3 };
enum { HBEM_DOUBLE = 0, HBEM_SINGLE = 1 };
/* Family (spaces.py:31-34) */
enum { HBEM_P0 = 0, HBEM_P1C = 1, HBEM_P1D = 2 };
/* PairKind (quadrature.py:119-128) */
enum { HBEM_DISJOINT = 0, HBEM_SHARED_VERTEX = 1, HBEM_SHARED_EDGE = 2, HBEM_IDENTICAL = 3 };

#define HBEM_MAX_WEIGHTS 6 /* backend.py:34 */

typedef struct hbem_ctx hbem_ctx;
typedef struct hbem_hmat hbem_hmat;
typedef struct hbem_tree hbem_tree;
typedef struct hbem_blocks hbem_blocks;

/*
 * Everything init_device (backend.py:77-122) and make_integration_context
 * (kernels.py:199-227) stage for one operator on one device.
 * Geometry caches (qpoints/normals/jacobians/curls) are optional: pass NULL
 * and they are computed on the device from vertices/elements with the same
 * float64 operation order as precompute_geometry (mesh.py:338-371) and
 * element_curls (spaces.py:132-143).
 */
typedef struct hbem_ctx_desc {
  int32_t device;
  int32_t equation;   /* HBEM_LAPLACE / HBEM_HELMHOLTZ */
  int32_t op;         /* HBEM_SLP ... HBEM_HYPS        */
  int32_t precision;  /* HBEM_DOUBLE / HBEM_SINGLE     */
  double wavenumber;
  int32_t test_family, trial_family; /* HBEM_P0 / HBEM_P1C / HBEM_P1D */
  int64_t n_vertices;
  const double *vertices;  /* (n_vertices, 3) */
  int64_t n_elements;
  const int64_t *elements; /* (n_elements, 3) */
  int32_t n_q;             /* regular-rule points (<= HBEM_MAX_WEIGHTS) */
  const double *rule_points;  /* (n_q, 2) reference coordinates */
  const double *rule_weights; /* (n_q,)                          */
  const double *qpoints;   /* (m, n_q, 3) or NULL */
  const double *normals;   /* (m, 3) or NULL      */
  const double *jacobians; /* (m,) or NULL        */
  const double *curls;     /* (m, 3, 3) or NULL (hyps only) */
  /* basis tables at the rule points (BasisTable.values, spaces.py:96-129):
     (nt, n_q) and (ns, n_q); NULL = tabulate from rule_points */
  const double *test_values;
  const double *trial_values;
  /* singular tensor rules (quadrature.py:274-312), index = kind-1:
     0 shared vertex, 1 shared edge, 2 identical; points (n, 4) */
  int64_t sing_n[3];
  const double *sing_points[3];
  const double *sing_weights[3];
} hbem_ctx_desc;

int hbem_abi_version(void);
const char *hbem_last_error(void);
int hbem_device_count(int32_t *count);

int hbem_ctx_create(const hbem_ctx_desc *desc, hbem_ctx **out);
int hbem_ctx_destroy(hbem_ctx *ctx);
/* Block shape (nt, ns) and whether the result has an imaginary plane. */
int hbem_ctx_info(const hbem_ctx *ctx, int32_t *nt, int32_t *ns, int32_t *is_complex,
                  int32_t *real_bytes);
/* Copy the device geometry caches back (float64), for verification. */
int hbem_ctx_geometry(const hbem_ctx *ctx, double *qpoints, double *normals, double *jacobians);

/*
 * integrate_batch (backend.py:200-255): disjoint pairs only.
 * pairs (p, 2) int64 test/trial element ids; re/im (p, nt, ns) in the
 * working precision (im may be NULL for Laplace; must be non-NULL for
 * Helmholtz).  Host pointers; synchronous.  Raises CONTRACT on an index out
 * of range ("pair indices must lie in ...") or on the first touching pair
 * ("request pair i = (a, b) is not disjoint; ...").
 */
int hbem_integrate_regular(hbem_ctx *ctx, const int64_t *pairs, int64_t p, void *re, void *im);

/*
 * Any adjacency class (local_matrix, kernels.py:330-347, batched):
 * touching pairs use Sauter-Schwab rules on the device with the canonical
 * test>trial transpose; regular pairs use the 6x6 rule.  Touching pairs are
 * computed in float64 and cast to the working precision, regular pairs in
 * the working precision — exactly the split of _integrate_pairs
 * (hmatrix.py:593-621).  n_singular (optional) receives the touching count.
 */
int hbem_integrate_any(hbem_ctx *ctx, const int64_t *pairs, int64_t p, void *re, void *im,
                       int64_t *n_singular);

/* Device-pointer variants (inputs resident in HBM; asynchronous on stream).
   No contract validation. stream = cudaStream_t (0 = legacy default). */
int hbem_integrate_regular_device(hbem_ctx *ctx, const int64_t *d_pairs, int64_t p, void *d_re,
                                  void *d_im, void *stream);
int hbem_integrate_any_device(hbem_ctx *ctx, const int64_t *d_pairs, int64_t p, void *d_re,
                              void *d_im, void *stream);

/* ---------------------------------------------------------------------
 * Partition (hmatrix.py:105-211): bit-exact cluster and block trees.
 * norm_mode selects the float64 evaluation of np.linalg.norm on a
 * 3-vector that the host numpy performs: 0 = sqrt((x*x + y*y) + z*z),
 * 1 = sqrt(fma(z, z, fma(y, y, x*x))) (OpenBLAS ddot with FMA).
 * --------------------------------------------------------------------- */
int hbem_cluster_tree(const double *points, int64_t n, int32_t n_min, hbem_tree **out);
int hbem_tree_size(const hbem_tree *t, int64_t *n_points, int64_t *n_nodes);
/* perm (n), nodes (n_nodes, 5) [start, stop, level, left, right], bbox (n_nodes, 6) */
int hbem_tree_copy(const hbem_tree *t, int64_t *perm, int64_t *nodes, double *bbox);
int hbem_tree_destroy(hbem_tree *t);
int hbem_block_tree(const hbem_tree *rows, const hbem_tree *cols, double eta, int32_t norm_mode,
                    hbem_blocks **out);
int hbem_blocks_size(const hbem_blocks *b, int64_t *n_leaves);
/* leaves (n_leaves, 3) [row_node, col_node, admissible] in descent order */
int hbem_blocks_copy(const hbem_blocks *b, int64_t *leaves);
int hbem_blocks_destroy(hbem_blocks *b);

/* ---------------------------------------------------------------------
 * Gmsh 2.2 ASCII reader (load_mesh, mesh.py:134-245): 3-node triangles
 * only (other element types counted in n_skipped), referenced vertices
 * compacted in ascending node-tag order.  HBEM_ERR_MESH when the file
 * cannot be read, HBEM_ERR_MESH_PARSE with the reference's message, line
 * number and section otherwise.
 * --------------------------------------------------------------------- */
typedef struct hbem_mesh_file hbem_mesh_file;
int hbem_gmsh_read(const char *path, hbem_mesh_file **out);
int hbem_gmsh_size(const hbem_mesh_file *m, int64_t *n_vertices, int64_t *n_elements,
                   int64_t *n_skipped);
/* vertices (n_vertices, 3) float64, elements (n_elements, 3) int64 */
int hbem_gmsh_copy(const hbem_mesh_file *m, double *vertices, int64_t *elements);
/* line (1-based, -1 if none) and section ("" if none) of the last parse error */
int hbem_gmsh_error_location(int64_t *line, char *section, int32_t cap);
int hbem_gmsh_destroy(hbem_mesh_file *m);

/* ---------------------------------------------------------------------
 * Device H-matrix assembly (assemble_hmatrix, hmatrix.py:759-811) with
 * lock-step batched ACA (hmatrix.py:271-382) over all admissible leaves.
 * --------------------------------------------------------------------- */
typedef struct hbem_hmat_desc {
  /* partition; row/col trees may be the same arrays */
  int64_t n_rows, n_cols;           /* DOF counts */
  const int64_t *row_perm, *col_perm;
  int64_t n_row_nodes, n_col_nodes;
  const int64_t *row_nodes, *col_nodes; /* (n, 5) start, stop, level, left, right */
  int64_t n_leaves;
  const int64_t *leaves;            /* (n_leaves, 3) row_node, col_node, admissible */
  /* spaces */
  const int64_t *test_dofmap;       /* (m, nt) */
  const int64_t *trial_dofmap;      /* (m, ns) */
  /* ACA (AcaConfig, hmatrix.py:219-238) */
  double epsilon;
  int64_t k_max;                    /* <= 0 means None (min(m, n)) */
  int32_t rank_capacity;            /* initial per-block factor capacity, 0 = auto */
  int32_t pointers_on_device;       /* 1: all arrays above are device pointers */
  /* optional host output arenas (page-locked, e.g. hbem_host_alloc), element
     units of the result dtype; when set, execute streams the low-rank
     factors of every wave and the dense leaves into them while the
     assembly runs (hbem_hmat_copy_arenas is then not needed).  A capacity
     smaller than the payload is a CapacityError. */
  void *out_u, *out_v, *out_dense;
  int64_t out_u_cap, out_v_cap, out_dense_cap;
} hbem_hmat_desc;

/* counters returned by hbem_hmat_stats (names as _LeafAssembler.counters,
   hmatrix.py:575-584, plus pair counts) */
typedef struct hbem_hmat_stats {
  int64_t regular_pairs, singular_pairs;
  int64_t aca_converged, aca_exhausted, aca_fallback_dense;
  int64_t dense_leaves, lowrank_leaves;
  int64_t waves, row_jobs, col_jobs, capacity_retries;
  int64_t u_entries, v_entries, dense_entries;
  int64_t launches;          /* kernels launched by the last execute */
  int64_t aca_entries;       /* matrix entries evaluated by ACA row/column jobs */
  double aca_kernel_ms;      /* CUDA-event time of the ACA row+column launches */
  double nearfield_kernel_ms;/* CUDA-event time of the near-field launches (side stream) */
  double seconds;            /* last execute, host wall clock incl. syncs */
  double seconds_setup;      /* one-time partition upload + allocation */
  double seconds_aca;        /* ACA waves (near-field overlapped) */
  double seconds_finalize;   /* payload classification + dense expansion */
  double int_kernel_ms;      /* CUDA-event time of the ACA integration launches (k_aca_*) */
  int64_t int_launches;      /* number of those launches */
  int64_t sing_table_pairs;  /* touching element pairs Sauter-Schwab-integrated per execute
                                (the near-field leaves of this handle only) */
} hbem_hmat_stats;

/* setup (partition upload, state allocation) + one execute */
int hbem_hmat_assemble(hbem_ctx *ctx, const hbem_hmat_desc *desc, void *stream, hbem_hmat **out);
/* re-run the assembly on an existing handle (inputs resident on the device;
   deterministic: identical payloads) */
int hbem_hmat_execute(hbem_hmat *h, void *stream);
int hbem_hmat_stats_get(const hbem_hmat *h, hbem_hmat_stats *stats);
/* per leaf: kind (0 dense, 1 low-rank), rank, converged, exhausted,
   offsets of U (height*rank), V (width*rank) or dense (height*width)
   payloads in their arenas (element units), column-major per rank. */
int hbem_hmat_leaf_meta(const hbem_hmat *h, int32_t *kind, int32_t *rank, int32_t *flags,
                        int64_t *off_u, int64_t *off_v, int64_t *off_dense);
/* per leaf: the ACA residual indicator of LowRankBlock.residual (hmatrix.py:
 * 241-268, 377-382: last rank-1 update relative to the accumulated Frobenius
 * norm; 0 for dense leaves and blocks without terms) */
int hbem_hmat_leaf_residual(const hbem_hmat *h, double *resid);
/* D2H of the factor/dense arenas in the result dtype (complex interleaved). */
int hbem_hmat_copy_arenas(const hbem_hmat *h, void *u, void *v, void *dense);
/* y = H x in original DOF order; x, y host arrays of the result dtype. */
int hbem_hmat_matvec(const hbem_hmat *h, const void *x, void *y);
/* y = H x with x (n_cols) and y (n_rows) DEVICE pointers in the original DOF
 * order, enqueued on `stream` (no host synchronisation); bit-reproducible:
 * every leaf contribution lands in its own slot and rows add them in the
 * reference's fixed (row start, column start) leaf order (hmatrix.py:441-470) */
int hbem_hmat_matvec_device(const hbem_hmat *h, const void *d_x, void *d_y, void *stream);
int hbem_hmat_destroy(hbem_hmat *h);

/* Far-field potential of a surface density, evaluate_far_field
   (scatter.py:362-408): out[i] = sum over elements e and rule points q of
   K_dlp(points[i], y_eq) dens_eq with dens_eq = (sum_l phi[dofmap[e,l]]
   table[l,q]) |J_e| w_q; K_dlp the Helmholtz (wavenumber > 0) or Laplace
   (wavenumber == 0) double-layer kernel of kernel_planes (kernels.py:129-158).
   points (n,3), vertices (nv,3), elements (m,3), rule_points (nq,2),
   rule_weights (nq), table (local_dim,nq), dofmap (m,local_dim) row-major;
   phi_im may be NULL (real density); r_min (n, nullable) receives each point's
   distance to the nearest rule point (the near-field warning test). */
int hbem_far_field(int32_t device, int64_t n_points, const double *points, int64_t n_vertices,
                   const double *vertices, int64_t m, const int64_t *elements, int32_t nq,
                   const double *rule_points, const double *rule_weights, int32_t local_dim,
                   const double *table, const int64_t *dofmap, int64_t n_dofs,
                   const double *phi_re, const double *phi_im, double wavenumber,
                   double *out_re, double *out_im, double *r_min);

/* pinned host buffers for fast D2H of the arenas */
int hbem_host_alloc(int64_t bytes, void **out);
int hbem_host_free(void *p);
/* measured FMA throughput (FLOP/s, 2 per FMA) of this device, FP64 or FP32:
   the live roofline denominator for the FMA-pipe-bound integrators */
int hbem_probe_fma(int32_t device, int32_t precision, double *flops_per_s);

#ifdef __cplusplus
}
#endif
#endif /* HBEM_B200_H */
