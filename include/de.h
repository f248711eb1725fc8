/*
 * de.h — C ABI of the B200-native interface-PCG solver for SIMP-weighted Q1
 * linear elasticity by non-overlapping domain decomposition
 * (arXiv 1501.06211; citations are /root/reference/PAPER.md line numbers).
 *
 * The method (Eq. (7)):
 *   1. K_IiIi u1_Ii = f_Ii                       (interior Dirichlet solves)
 *   2. S u_Gamma = f_Gamma - sum_i K_GammaIi u1_Ii, S = sum_i R_i^T (A_GG,i - A_GI,i A_II,i^-1 A_IG,i) R_i,
 *      solved by PCG preconditioned with H^_theta = (+)_c M_c (M_c^-1 L_c)^(1-theta)
 *      (Eqs. (8)-(9)) applied by inverse Lanczos
 *   3. K_IiIi u2_Ii = -K_IiGamma u_Gamma,   u = (u1_I, 0) + (u2_I, u_Gamma)
 * Material (R1/R2): E_e = Emin + rho_e^p (E0 - Emin); 2D plane stress, 3D isotropic,
 * Hooke's law sigma = 2 mu eps + lambda tr(eps) I. Q1 elements of edge h.
 *
 * Conventions (R4):
 *   node = i + (nx+1)*(j + (ny+1)*k)   (x fastest, k = 0 in 2D)
 *   dof  = dim*node + c                (component fastest)
 *   element e = ex + nx*(ey + ny*ez), density[] in that order
 *   subdomain s = sx + px*(sy + py*sz), each subdomain an axis-aligned box of sub[] elements
 *
 * Ownership: the caller owns every host array passed in; the library copies what it needs
 * during the call and keeps no pointer afterwards. A de_ctx_t owns all device memory it
 * allocates (cudaMalloc on options.device) until de_destroy. Device pointers passed to the
 * *_device entry points are borrowed for the duration of the call only.
 *
 * Errors: every call returns de_status_t (DE_OK = 0). On failure, de_last_error() returns a
 * thread-local message. There is no CPU fallback: without a usable CUDA device, de_setup
 * returns DE_ECUDA.
 *
 * Threading: a context is not thread-safe; distinct contexts are independent.
 * Multi-GPU (nranks > 1): every call is collective over ranks with identical host inputs;
 * every rank returns the full u. Rank r owns subdomain columns sx in
 * [floor(r*px/nranks), floor((r+1)*px/nranks)); interface vectors are replicated and the
 * partial interface sums are combined with one ncclAllReduce per PCG iteration.
 */
#ifndef DE_H_
#define DE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DE_OK = 0,
    DE_EINVAL = -1,      /* invalid argument (partition does not divide mesh, dim not 2/3,
                            rho <= 0 or non-finite, nu not in (-1, 1/2), E0 <= 0, Emin < 0,
                            no Dirichlet dof, unsupported option)                          */
    DE_ENOTSPD = -2,     /* non-positive pivot in an interior factorisation (subdomain id in message) */
    DE_ENOCONV = -3,     /* max_iter reached, or the refined iterate missed rtol (stats.relres_dd);
                            u holds the last iterate                           */
    DE_EBREAKDOWN = -4,  /* p^T S p <= 0, or a non-positive Ritz value (R9)       */
    DE_ESTATE = -5,      /* de_solve before de_factor                                      */
    DE_ENOMEM = -6,
    DE_ECUDA = -7,
    DE_ENCCL = -8
} de_status_t;

typedef struct de_ctx de_ctx_t;   /* opaque */

typedef struct {
    int32_t dim;             /* 2 or 3 */
    int32_t nel[3];          /* elements per axis; nel[2] ignored when dim == 2 */
    double h;                /* element edge length (BASELINE: 1.0); 2D thickness 1 */
    const uint8_t* fixed;    /* host, ndof = dim * prod_a (nel[a]+1) flags; 1 = homogeneous Dirichlet */
} de_mesh_t;

typedef struct {
    int32_t sub[3];          /* elements per subdomain per axis; must divide nel */
} de_partition_t;

typedef struct {
    double theta;            /* fractional index theta of H~_theta; default 0.5 */
    int32_t lanczos_k;       /* inverse-Lanczos basis size k; default 10 */
    int32_t inner_mode;      /* preconditioner: 1 = inverse Lanczos with exact inner solves (mode X,
                                DESIGN.md R10); 0 = inverse Lanczos with SPEC's face-preconditioned PCG
                                inner solves of K (mode F: tol inner_tol, x0 = 0, cap inner_max_iter;
                                PAPER.md:235-237,273); 3 = identity S~ = I */
    double inner_tol;        /* inner_mode 0: relative 2-norm tolerance of the inner PCG; default 1e-3 */
    int32_t inner_max_iter;  /* inner_mode 0: inner PCG iteration cap; default 1000 */
    int32_t max_iter;        /* outer PCG iteration cap; default 20000 */
    int32_t beta_variant;    /* 0 = Fletcher-Reeves (default), 1 = Polak-Ribiere (flexible) */
    int32_t warm_start;      /* 1: start PCG from the previous solve's u_Gamma (config-5 sequence) */
    int32_t rank, nranks;    /* nranks == 1: single GPU, no NCCL */
    int32_t device;          /* CUDA device ordinal */
    const void* nccl_id;     /* 128-byte ncclUniqueId (from de_nccl_unique_id on rank 0), nranks > 1 only */
    void* stream;            /* cudaStream_t to run on, or NULL for a library-owned stream */
    int32_t check_every;     /* convergence poll period in iterations (device-side early exit makes
                                extra launches no-ops); default 8 */
    int32_t use_graph;       /* 1 (default): capture check_every PCG iterations into a CUDA graph */
    int32_t host_only;       /* 1: run only the host setup (topology, DOF map, skeleton queries);
                                no device is touched and de_factor/de_solve return DE_ESTATE */
    int32_t prec_kernels;    /* 0 (default): one persistent cooperative kernel per preconditioner
                                application; 1: one kernel per phase (same arithmetic) */
    int32_t schur_mode;      /* S apply in the PCG loop: 0 = auto (explicit when the dense local S_s take fewer
                                bytes than one pass over the factors, i.e. 2D), 1 = implicit through interior
                                solves, 2 = explicit local Schur complements S_s formed at
                                de_factor; condense/back-substitution always use the solves */
    int32_t weighted_trace;  /* 1: coefficient-weighted trace norm (R19): every trace
                                facet element of M and L is scaled by the mean SIMP modulus of its two adjacent
                                elements; the preconditioner is rebuilt by de_factor after each density update.
                                0 (default): the unweighted norm of PAPER.md:172 (R6) */
    int32_t outer;           /* outer Krylov method of de_solve: 0 (default) = interface PCG on S u_Gamma = g (BASELINE
                                metric); 1 = right-preconditioned flexible GMRES on the full system
                                K u = f with P~ = [[K_II, K_IGamma], [0, S~]],
                                single rank; `iterations` then counts FGMRES iterations */
    int32_t restart;         /* FGMRES restart length m, 1 <= m <= 31 (default 30) */
    void* loopback;          /* nranks > 1 without NCCL: a de_loopback_t* shared by the nranks contexts of one process
                                (see de_loopback_create); NULL (default) = NCCL with nccl_id */
} de_options_t;

/* Single-process loopback group: nranks contexts on one device, each driven by its own host thread, exercise the
 * multi-rank path (owned subdomain slabs, partial interface sums, the cross-rank exchanges) without NCCL. Every
 * all-reduce becomes: copy to this rank's device slot, host barrier, fixed-order sum of slots 0..nranks-1 on this
 * rank's stream, host barrier -- host-synchronised, so no kernel ever waits on another rank's kernel and the PCG
 * loop runs uncaptured (use_graph is ignored). Results are bitwise identical on every rank. Test/verification
 * path of DESIGN.md §8; the owner destroys the group after every context using it. */
typedef struct de_loopback de_loopback_t;
de_status_t de_loopback_create(int32_t nranks, de_loopback_t** out);
void de_loopback_destroy(de_loopback_t* g);

typedef struct {
    int64_t ndof, n_free, n_I, n_Gamma, n_sub, n_sub_local;
    int32_t band;            /* uniform half bandwidth of the interior factors */
    int32_t iterations;      /* outer PCG iterations of the last solve */
    int32_t restarts;        /* iterative-refinement rounds of the last solve (R11) */
    double relres_recursive; /* ||r_Gamma|| / ||f_free|| at exit (recursive residual) */
    double relres_true;      /* ||f - K u||_2 / ||f||_2 over free dofs (matrix-free K) */
    double ms_factor;        /* de_factor: SIMP assembly + band Cholesky */
    double ms_solve;         /* last de_solve, whole call incl. transfers */
    double ms_pcg;           /* PCG loop only */
    double ms_schur;         /* sum of Schur-apply kernel time (event-timed when profiling enabled) */
    double bytes_factor;     /* algorithmic bytes of one pass over the local interior factors */
    double bytes_iter;       /* algorithmic bytes of one PCG iteration on this rank */
    int32_t launches_per_iter; /* kernels launched per PCG iteration (graph nodes) */
    int32_t singular_components; /* bitmask of components using H_theta (R7) */
    int64_t n_cross[3];      /* cross points / wirebasket nodes per component */
    int64_t n_faces[3];
    int64_t n_gamma_c[3];
    double bytes_schur;      /* algorithmic bytes of one Schur-apply launch: one pass over the local
                                factor band + ring blocks A_IG/A_GG + local interface vectors */
    int64_t kernels_launched; /* kernels launched by the last de_solve (graph nodes included) */
    int32_t iterations_pass1; /* PCG iterations before iterative refinement */
    int32_t schur_explicit;  /* 1 if the PCG loop applies explicit local Schur complements */
    double bytes_schur_explicit; /* algorithmic bytes of one explicit S apply: sum_s n_Gamma,s^2 * 8 + vectors */
    double bytes_prec;       /* algorithmic bytes of one preconditioner application (k_prec_coop; per-phase
                                streaming model of DESIGN.md "Kernels and their rooflines"), 0 if none */
    int64_t inner_iterations; /* inner_mode 0: face-PCG iterations of all inner solves since de_setup
                                 (summed over solves and components); 0 otherwise */
    double relres_dd;        /* ||f - K (u_hi + u_lo)||_2 / ||f||_2 of the double-double iterate carried through
                                the iterative refinement (R11/R17); de_solve returns DE_OK iff this is
                                <= rtol. The returned u is fl(u_hi + u_lo), so relres_true exceeds it by at most
                                the FP64 rounding floor of the problem (measured for config 5: 1.35e-10) */
    double bytes_prec_min;   /* distinct bytes one preconditioner application touches, each counted once (operators,
                                r, z, basis written once): the minimum-bytes figure of its roofline */
    int32_t cross_fd;        /* bit 0 / bit 1: the cross-point Schur complement of the K / M elimination is separable
                                and solved by fast diagonalisation instead of the dense S_C^-1 (R23) */
} de_stats_t;

/* Fill *opt with defaults (theta 0.5, k 10, inner_mode 1, max_iter 20000, FR, 1 rank). */
void de_default_options(de_options_t* opt);

/* Setup (host topology + density-independent preconditioner structures, device upload).
 * density: host, prod(nel) values in (0, inf); E0 > 0; Emin >= 0; p > 0; nu in (-1, 1/2).
 * PAPER.md:56 (decomposition), :111-120 (interior-first ordering), :167-181 (trace M, L). */
de_status_t de_setup(const de_mesh_t* mesh, const double* density, double E0, double Emin,
                     double p, double nu, const de_partition_t* part, const de_options_t* opt,
                     de_ctx_t** out);

/* Replace the element densities rho_e (host array, prod(nel), element order of the header comment; every value
 * positive and finite, else DE_EINVAL). The stiffness K(rho) = sum_e E_e(rho_e) K_e^0 changes with them
 * (Eq. (10), read as SIMP: DESIGN.md R1); this is the density update of the topology-optimisation
 * loop between two analyses (BASELINE config 5). Copies the array; the context is marked
 * unfactored, so de_factor must be called before the next de_solve (else DE_ESTATE). With weighted_trace the
 * preconditioner is rebuilt by that de_factor (R19). */
de_status_t de_update_densities(de_ctx_t* ctx, const double* density);
/* Same with a device pointer (float64, prod(nel)) on options.device, borrowed for the call (stream-ordered copy);
 * the values are not validated on the host. */
de_status_t de_update_densities_device(de_ctx_t* ctx, const double* d_density);

/* SIMP scaling + subdomain blocks A_II (band), A_IG, A_GG (ring) + batched band Cholesky
 * A_II,i = L_i L_i^T. Returns DE_ENOTSPD on a non-positive pivot. */
de_status_t de_factor(de_ctx_t* ctx);

/* Solve K(rho) u = f. rhs: host, ndof (Dirichlet entries ignored);
 * u: host, ndof out (0 at Dirichlet dofs). rtol relative to ||rhs_free||_2 (R11).
 * iterations/final_relres may be NULL. final_relres = true ||f - K u|| / ||f|| over free dofs of the
 * returned FP64 u (double-double residual); DE_OK means the refined double-double iterate, whose FP64
 * rounding u is, meets rtol (de_stats_t.relres_dd; R17). */
de_status_t de_solve(de_ctx_t* ctx, const double* rhs, double rtol, double* u,
                     int32_t* iterations, double* final_relres);

/* Same with device-resident rhs and u (float64, ndof, on options.device). */
de_status_t de_solve_device(de_ctx_t* ctx, const double* d_rhs, double rtol, double* d_u,
                            int32_t* iterations, double* final_relres);

/* Bit-exact DOF map (R4/R5): cls[ndof] (0 = I, 1 = Gamma, 2 = Dirichlet),
 * sub[ndof] (owning subdomain of interior dofs, -1 otherwise), reduced[ndof] (canonical index:
 * interior dofs by (s, dof), then Gamma dofs by dof; -1 for Dirichlet). Any pointer may be NULL. */
de_status_t de_get_dofmap(const de_ctx_t* ctx, int8_t* cls, int32_t* sub, int32_t* reduced,
                          int64_t* n_I, int64_t* n_Gamma);

/* Interface skeleton of component c (R6/R8): node ids of Gamma_c (ascending),
 * per node its face id (-1 for a cross point). Arrays sized n_gamma_c[c] (see de_get_stats). */
de_status_t de_get_skeleton(const de_ctx_t* ctx, int32_t c, int32_t* nodes, int32_t* face_of_node);

/* Subdomains owned by this rank (ascending global ids; slab rule in the header comment). ids may be NULL
 * to query the count; available for host_only contexts as well. */
de_status_t de_get_owned(const de_ctx_t* ctx, int32_t* ids, int32_t* n);

/* Fill *stats with the sizes of this context (dof counts, interface skeleton per component: SURVEY.md Appendix A
 * quantities) and the figures of the last de_factor / de_solve (iterations, residuals, times,
 * the algorithmic byte counts of SURVEY.md §8(d) used by bench.py's rooflines). Host bookkeeping, except that with
 * inner_mode 0 the inner face-PCG iteration counter is read from the device (a stream synchronisation).
 * DE_EINVAL on null arguments. */
de_status_t de_get_stats(const de_ctx_t* ctx, de_stats_t* stats);

/* ---- component-level entry points (parity tests and profiling) --------------------------
 * All vectors are device pointers (float64) of the stated lengths. */

/* q = S p over this rank's subdomains, assembled (and all-reduced when nranks > 1); n_Gamma. */
de_status_t de_schur_apply_device(de_ctx_t* ctx, const double* d_p, double* d_q);
/* z = H^_theta^-1 r (or r when inner_mode == 3); n_Gamma. */
de_status_t de_precond_apply_device(de_ctx_t* ctx, const double* d_r, double* d_z);
/* Lower band of the factor of local subdomain sl: out[n_I_s * (band+1)], column-major,
 * out[j*(band+1)+k] = L[j+k][j] (k = 0 holds L[j][j] itself). Host pointer. */
de_status_t de_get_factor_band(const de_ctx_t* ctx, int32_t sl, double* out, int32_t* n_I_s);
/* Same layout for the assembled A_II,s (before factorisation; recomputed on demand). */
de_status_t de_get_assembled_band(de_ctx_t* ctx, int32_t sl, double* out, int32_t* n_I_s);

/* NCCL unique id (128 bytes) for a multi-rank setup; call on rank 0 and broadcast. */
de_status_t de_nccl_unique_id(void* out128);

/* Record per-kernel CUDA-event timing of the Schur apply inside de_solve (bench only). */
de_status_t de_set_profiling(de_ctx_t* ctx, int32_t on);
/* Average device time (ms) of one launch of the Schur-apply kernel over the last solve. */
de_status_t de_get_kernel_time(const de_ctx_t* ctx, double* ms_schur_per_launch, int64_t* launches);
/* Average device time (ms) of one preconditioner application (k_prec_coop, or the multi-kernel path)
   over the last solve with profiling on; same event-pair method inside the captured PCG graph. */
de_status_t de_get_prec_time(const de_ctx_t* ctx, double* ms_prec_per_launch, int64_t* launches);

void de_destroy(de_ctx_t* ctx);
/* ---- Topology-optimisation design update (R20) ----
 * The loop the solver serves: solve K(rho) u = f, then one optimality-criteria (OC) step, then de_factor.
 * The paper states no OC constants; R20 fixes the standard minimum-compliance OC update:
 *   dc_e   = -p rho_e^(p-1) (E0 - Emin) u_e^T KE0 u_e          compliance c = sum_e E_e u_e^T KE0 u_e
 *   rho_e' = clip(rho_e (max(-dc_e,0)/lambda)^eta, max(rho_min, rho_e - move), min(1, rho_e + move))
 *   lambda by bisection on [0, 1e9 max(-dc)] until l2 - l1 <= tol (l1 + l2) or maxit halvings, so that
 *   sum_e rho_e' = volfrac * n_elem (unit element volumes). VTS is p = 1, Emin = 0. */
typedef struct {
    double volfrac;   /* target mean density V, in (0, 1] */
    double move;      /* move limit per step, > 0 */
    double rho_min;   /* lower density bound, in (0, 1); the upper bound is 1 */
    double eta;       /* damping exponent, > 0 (0.5 standard) */
    double tol;       /* relative bisection tolerance on lambda, > 0 */
    int32_t maxit;    /* bisection steps, in [1, 10000] (each is two launches; converged steps are no-ops) */
} de_oc_params_t;

/* volfrac 0.5, move 0.2, rho_min 1e-3, eta 0.5, tol 1e-12, maxit 200. */
void de_default_oc_params(de_oc_params_t* prm);

/* Element sensitivities of the compliance at the context's current densities for the displacement d_u
 * (device, float64, ndof — e.g. de_solve_device's output). d_dc: device, float64, prod(nel) out, or NULL
 * (kept inside the context for de_oc_update_device). compliance: host scalar out, or NULL (no sync). */
de_status_t de_sensitivities_device(de_ctx_t* ctx, const double* d_u, double* d_dc, double* compliance);

/* One OC step from the sensitivities d_dc (device, prod(nel); NULL = those of the last
 * de_sensitivities_device call): the new densities replace the context's (de_factor must be called next)
 * and are copied to d_rho_new (device, prod(nel)) if non-NULL. lambda: host scalar out, or NULL.
 * DE_EINVAL on parameters out of range or when d_dc is NULL and no sensitivities exist. */
de_status_t de_oc_update_device(de_ctx_t* ctx, const double* d_dc, const de_oc_params_t* prm,
                                double* d_rho_new, double* lambda);

/* Host-buffer form of both calls: u host (ndof) in, rho_new host (prod(nel)) out (may be NULL);
 * compliance/lambda host scalars (may be NULL). */
de_status_t de_oc_step(de_ctx_t* ctx, const double* u, const de_oc_params_t* prm, double* rho_new,
                       double* compliance, double* lambda);

const char* de_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* DE_H_ */
