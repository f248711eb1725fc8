// de_internal.h — internal structures of libde (B200-native interface PCG).
// Host setup (topology, trace matrices, preconditioner structures) is plain C++;
// all numerics of the hot path run in the sm_100a kernels declared at the bottom.
#pragma once

#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/de.h"

namespace de {

constexpr int KMAX = 16;            // max inverse-Lanczos basis size supported on device
constexpr int MAXC = 3;             // max displacement components

void set_error(const char* fmt, ...);

// Raise (never lower) a kernel's dynamic shared-memory limit. The limit is one value per kernel for the whole process,
// while the size a launch needs depends on the context (a rank's largest subdomain, its ring entries): two contexts
// driven from different host threads that each SET their own size could lower the limit between another thread's
// set and its launch ("invalid argument"; seen as an intermittent hang of the 8-rank loopback test, whose other
// ranks then waited for the failed ones in an exchange).
inline void raise_dyn_smem(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::map<const void*, size_t> cur;
    std::lock_guard<std::mutex> lk(mu);
    size_t& c = cur[fn];
    if (bytes > c) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
        c = bytes;
    }
}

#define DE_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            ::de::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(e_), __FILE__, \
                            __LINE__, cudaGetErrorString(e_));                          \
            return DE_ECUDA;                                                            \
        }                                                                               \
    } while (0)

// ------------------------------------------------------------------------ host setup

// Sparse matrix in CSR with int32 indices (host side).
struct HCsr {
    int32_t n = 0, m = 0;
    std::vector<int32_t> ptr, col;
    std::vector<double> val;
};

// Exact-elimination structure of one skeleton operator X (X = K_c or M_c), all components
// flattened (R10): faces F (cross points removed), cross points C,
//   x_C = S_C^-1 (b_C - X_CF X_FF^-1 b_F),  x_F = X_FF^-1 (b_F - X_FC x_C),
//   S_C = X_CC - X_CF X_FF^-1 X_FC  (dense, per component, inverted on the GPU).
struct HElim {
    int32_t nfaces = 0;
    std::vector<int32_t> face_off;      // [nfaces+1] into face_nodes
    std::vector<int32_t> face_nodes;    // flattened skeleton index of each face node
    std::vector<int32_t> face_band;     // half bandwidth of X_FF in face order
    std::vector<int64_t> face_fac_off;  // offset of each face factor (column band, ld = band+1)
    std::vector<double> face_fac;       // band Cholesky factors, slot 0 holds 1/L_jj
    int32_t ncross = 0;
    int32_t cross_comp_off[MAXC + 1] = {0, 0, 0, 0};
    std::vector<int32_t> cross_flat;    // flattened skeleton index of each cross point
    HCsr XCF;                           // rows: cross points; cols: flattened skeleton index (face nodes)
    HCsr XFC;                           // rows: face-node slots (face_nodes order); cols: cross index
    std::vector<int64_t> sc_off;        // [ncomp+1] offsets of dense S_C per component
    std::vector<double> SC;             // dense S_C (row-major per component), inverted on device
    // 1 when every component's S_C is bitwise identical to component 0's (same skeleton and Dirichlet rows:
    // the trace norm is componentwise): one S_C^-1 serves all components
    int32_t sc_shared = 0;
    // 3D: G_F = X_FF^-1 X_F,adj per face (dense, column-major: column e over the face's nodes), adj = the face's
    // distinct wirebasket neighbours: the second face phase x_F = y_F - G_F x_C(adj) becomes a streaming pass instead of
    // a second sequential band solve
    std::vector<int64_t> g3_off;        // [nfaces+1] offsets into g3
    std::vector<double> g3;
    std::vector<int32_t> g3_adj_ptr;    // [nfaces+1] into g3_adj
    std::vector<int32_t> g3_adj;        // cross indices
    // 3D, face band <= FB_BS: the face factor L as a block-bidiagonal matrix of FB_BS x FB_BS blocks (D_i on the
    // diagonal, E_i below it). Per face block i four dense FB_BS x FB_BS matrices, column-major (entry (row, col) at
    // col * FB_BS + row): F_i = D_i^-1, G_i = D_i^-1 E_i, F_i^T, H_i = D_i^-T E_{i+1}^T, so that
    //   forward  y_i = F_i r_i - G_i y_{i-1},   backward  x_i = F_i^T y_i - H_i x_{i+1}
    // replace the row-by-row band sweeps (identity padding past the face end). fb_off[F] = first block of face F.
    std::vector<int32_t> fb_off;        // [nfaces+1]
    std::vector<double> fb;             // [blocks][4][FB_BS * FB_BS]
    // Fast diagonalisation of S_C (2D, R23): when the cross points of every component form a full
    // nx x ny tensor grid (index = ix + nx iy) and S_C = A_x (x) I + I (x) A_y exactly (uniform skeleton, unweighted
    // trace norm, Dirichlet rows on whole edges), S_C^-1 = (Q_y (x) Q_x) diag(1 / (lam_a + mu_b)) (Q_y (x) Q_x)^T with
    // A_x = Q_x diag(lam) Q_x^T, A_y = Q_y diag(mu) Q_y^T. Per stored component (one if sc_shared):
    // fd_qx [ix][a] (nx x nx), fd_qy [iy][b] (ny x ny), fd_il [a + nx b] = 1 / (lam_a + mu_b).
    int32_t fd = 0, fd_nx = 0, fd_ny = 0;
    std::vector<double> fd_qx, fd_qy, fd_il;
};

struct HostSetup {
    // mesh / partition
    int dim = 2;
    int nel[3] = {1, 1, 1}, nn[3] = {2, 2, 1}, sub[3] = {1, 1, 1}, ps[3] = {1, 1, 1};
    int64_t nnodes = 0, ndof = 0, nelem = 0;
    int32_t nsub = 0;
    double h = 1.0;
    // dof map (bit-exact contract, R4/R5)
    std::vector<int8_t> cls;          // 0 I, 1 Gamma, 2 D
    std::vector<int32_t> dof_sub;     // owning subdomain of interior dofs, -1 otherwise
    std::vector<int32_t> reduced;     // canonical index or -1
    std::vector<int32_t> gpos;        // Gamma index of a dof or -1
    std::vector<int32_t> lidx;        // local interior index of an interior dof
    std::vector<int32_t> gamma_dofs;  // ascending
    int64_t n_I = 0, n_G = 0, n_free = 0;
    std::vector<int32_t> node_nsub;   // distinct subdomains per node
    std::vector<int32_t> node_subs;   // up to 8 subdomain ids per node (sorted), -1 padded
    // per subdomain
    std::vector<int64_t> ioff;        // offset into idofs (canonical interior start)
    std::vector<int32_t> nI;
    std::vector<int32_t> idofs;       // interior dofs, concatenated by subdomain
    std::vector<int64_t> goff;
    std::vector<int32_t> nGs;
    std::vector<int32_t> gdofs;       // Gamma dofs touched by each subdomain, concatenated
    std::vector<int32_t> band_s;      // per-subdomain half bandwidth
    int32_t band = 0, ld = 0;
    // component skeletons (flattened)
    int ncomp = 0;
    int64_t comp_off[MAXC + 1] = {0, 0, 0, 0};
    std::vector<int32_t> cmap;        // flat -> Gamma index
    std::vector<int32_t> cnode;       // flat -> node id
    std::vector<int32_t> face_of;     // flat -> face id within component, -1 cross
    int64_t n_faces_c[MAXC] = {0, 0, 0}, n_cross_c[MAXC] = {0, 0, 0};
    int singular_mask = 0;
    std::vector<int32_t> flat_of;     // Gamma dof -> flattened skeleton index (-1 otherwise)
    std::vector<double> trace_E;      // element moduli of the weighted trace norm (R19); empty = unweighted
    HCsr M, L, K;                     // block diagonal over components (flattened)
    HElim elimK, elimM;
    double KE0[24 * 24];              // unit-E element stiffness, local order lexicographic
    int nke = 8;
};

// Build everything density-independent. Returns DE_OK or DE_EINVAL with the error set.
de_status_t host_setup(const de_mesh_t* mesh, const de_partition_t* part, double nu,
                       HostSetup& hs);
de_status_t build_trace(HostSetup& hs, const double* Ee);

// Per-subdomain ring structures (A_IG rows over interior, A_GG/A_GI rows over Gamma).
struct HRing {
    std::vector<int32_t> igp;               // per local subdomain: nI+1 row pointers (absolute)
    std::vector<int32_t> ig_col;            // local Gamma column
    std::vector<int32_t> ig_da, ig_db;      // dof pair (row dof, col dof)
    std::vector<int32_t> gxp;               // per local subdomain: nG+1 row pointers (absolute)
    std::vector<int32_t> gx_col;            // >= 0 local Gamma col; < 0: -(interior local)-1
    std::vector<int32_t> gx_da, gx_db;
    std::vector<int64_t> igp_off, gxp_off;  // per local subdomain offsets into igp / gxp
};
void build_ring(const HostSetup& hs, const std::vector<int32_t>& owned, HRing& ring);

// ------------------------------------------------------------------------ device side

struct SubDesc {          // one owned subdomain
    int32_t gid;          // global subdomain id
    int32_t nI;
    int32_t nG;
    int32_t pad;
    int64_t ioff;         // offset into d_idofs / scratch (local concatenation)
    int64_t band_off;     // offset (doubles) into the factor band
    int64_t goff;         // offset into d_Rg / qloc
    int64_t igp_off;      // offset into d_igp (nI+1 entries)
    int64_t gxp_off;      // offset into d_gxp (nG+1 entries)
    int64_t sexp_off;     // offset (doubles) of the explicit local Schur complement S_s (nG x nG), if formed
};

struct MeshDev {
    int dim;
    int nel[3];
    int nn[3];
    int sub[3];
    int ps[3];
    int nke;
};

struct PcgState {
    double rz, pq, alpha, beta, rr, tol2, rz_old;
    int32_t it, done, status, maxit;
};

// optimality-criteria design update (kernels_topopt.cu, R20)
struct OcParams {
    double volfrac, move, rho_min, eta, tol;
    int32_t maxit;
};
struct OcState {
    double compliance, l1, l2, lambda;
    int32_t it, done;
};

struct ElimDev {
    int32_t nfaces, ncross, ncomp, maxface;
    int32_t maxld;               // max face band + 1 (column length of the face factors)
    int32_t face_comp_off[MAXC + 1];   // faces are grouped by component: [face_comp_off[c], face_comp_off[c+1])
    int32_t *face_off, *face_nodes, *face_band;
    int64_t* face_fac_off;
    double* face_fac;
    int32_t* cross_flat;
    int32_t cross_comp_off[MAXC + 1];
    int32_t *xcf_ptr, *xcf_col;
    double* xcf_val;
    int32_t *xfc_ptr, *xfc_col;
    double* xfc_val;
    int64_t sc_off[MAXC + 1];
    double* Sinv;
    int32_t sc_shared;           // 1: all components use the one S_C^-1 at Sinv (HElim::sc_shared)
    // fast diagonalisation of a separable S_C (HElim::fd): tables of stored component cs at fd_qx + cs nx^2,
    // fd_qy + cs ny^2, fd_il + cs nx ny (cs = 0 when sc_shared)
    int32_t fd, fd_nx, fd_ny;
    double *fd_qx, *fd_qy, *fd_il;
    // face-interleaved tridiagonal copy (2D): 32 faces per group, entry (j, lane) at (g*TRI_N + j)*32 + lane
    int32_t tri;                 // 1 if every face block is tridiagonal with <= TRI_N nodes and <= 2 cross couplings
    int32_t* tri_n;              // [nfaces] nodes per face
    int32_t* tri_node;           // flat index of node j (or 0 past the end)
    double* tri_inv;             // 1 / L_jj
    double* tri_sub;             // L_{j+1,j}
    int32_t* tri_xj;             // [2*nfaces] node index j of cross coupling k (or -1)
    int32_t* tri_xc;             // [2*nfaces] cross index of coupling k
    double* tri_xv;              // [2*nfaces] X_{F_j, c}
    // E3 folded into the consumer (tri only): x_i = y_i - g_v0[i] xC[g_c0[i]] - g_v1[i] xC[g_c1[i]] for every
    // flat skeleton index i, with G_F = X_FF^-1 X_FC on face nodes and (v0, c0) = (-1, own cross index), y_i = 0
    // on cross points
    int32_t fuse;
    int32_t *g_c0, *g_c1;
    double *g_v0, *g_v1;
    // X_CF padded to XCF_W entries per cross point ([XCF_W][ncross], col 0 / val 0 padding), tri only
    int32_t* xcf4_col;
    double* xcf4_val;
    // X_CF padded to xcf_w entries per cross point ([xcf_w][ncross], col 0 / val 0 padding), non-tri (3D): the
    // per-block t_C formation issues every load of a chunk together instead of walking CSR rows
    int32_t xcf_w;
    int32_t* xcfw_col;
    double* xcfw_val;
    // G_F = X_FF^-1 X_F,adj per face (HElim::g3), non-tri only: work items (face, 32-node chunk) for the second face phase
    // block-bidiagonal face solves (HElim::fb), non-tri only; null = row-by-row band sweeps
    int32_t* fb_off;
    double* fb;
    int32_t g3_items;
    int32_t *g3_item_face, *g3_item_i0;
    int64_t* g3_off;
    double* g3;
    int32_t *g3_adj_ptr, *g3_adj;
    // warp-per-face parallel cyclic reduction of X_FF y = b (tri only): lane j = face node j, 32 lanes per face
    // (identity rows past the face end); per face [PCR_Q][32] doubles: (alpha, gamma) of the 5 reduction
    // levels, then 1/d after the last level; pcr_node[F*32 + j] = flat index (0 past the end)
    // faces with bitwise-identical coefficient blocks share one: pcr_nt[F] = nodes | (block id << 8)
    double* pcr;
    int32_t* pcr_nt;
    int32_t* pcr_node;
    // G^T = X_CF X_FF^-1 as CSR over cross points (face-node columns): t_C = scale (b_C - G^T b_F) needs only
    // the right-hand side, so the first face phase forms it once per component (fuse only)
    int32_t *gt_ptr, *gt_col;
    double* gt_val;
    // the same rows through face descriptors (faces are contiguous in the flat numbering): cross point ci couples to
    // <= XCF_W faces f, td_start[f * ncross + ci] = flat index of the face's first node, td_len[..] = nodes | end << 8
    // (end = which of the face's two couplings ci is: its G column is g_v0 / g_v1 over the face's nodes); 0 = none.
    // One load level (the descriptors) before the coalesced g and b loads instead of ptr -> (val, col) -> b; null = CSR
    int32_t *td_start, *td_len;
    // fold ELL (fuse only, eK): rows of M and L with <= FELL_W entries, every entry carrying its column's
    // elimination couplings, so the consumer's x = y - G x_C of each neighbour is two dependent load levels
    // instead of four (CSR ptr -> col -> g[col] -> xC[g]); [FELL_W][nflat] each; fell_col[0][i] = -1: CSR row
    int32_t* fell_col;
    // consumer row patterns (fuse only; api.cu up_elim): pat_id[i] >= 0 indexes (pat_code, pat_m[3], pat_l[3]); the
    // row's neighbour values come from flat i-1, i, i+1 and the face's two x_C with row i's own couplings
    int32_t *pat_id, *pat_code;
    double *pat_m, *pat_l;
    // cross-point rows of the consumer (pat_id = -2 - cross index): ELL of width XELL_W over [XELL_W][ncross], every
    // entry with its column's couplings (as the fold ELL); null = CSR walk
    int32_t *xell_col, *xell_c0, *xell_c1;
    double *xell_v0, *xell_v1, *xell_m, *xell_l;
    int32_t *fell_c0, *fell_c1;
    double *fell_v0, *fell_v1, *fell_m, *fell_l;
};
constexpr int FB_BS = 16;            // block size of the block-bidiagonal 3D face solves
constexpr int FELL_W = 3;
constexpr int XELL_W = 5;            // a 2D cross point: itself + four face-end neighbours
constexpr int PCR_L = 5;             // log2(32) reduction levels
constexpr int PCR_Q = 2 * PCR_L + 1;
constexpr int XCF_W = 4;
constexpr int TRI_N = 32;
constexpr int FORM_THREADS = 256;   // columns per pass of the thread-per-column S_s formation
// Explicit S_s storage: the lower triangle of 16 x 16 tiles, tile (I, J) (I >= J) at (I(I+1)/2 + J) * 256,
// row-major inside the tile, zero padding past n_Gamma,s; diagonal tiles are stored whole.
constexpr int STS = 16;
inline int64_t sexp_packed_doubles(int nG) {
    const int64_t nt = (nG + STS - 1) / STS;
    return nt * (nt + 1) / 2 * STS * STS;
}
__host__ __device__ inline int64_t sexp_packed_index(int r, int c) {   // requires r / STS >= c / STS
    const int64_t I = r / STS, J = c / STS;
    return (I * (I + 1) / 2 + J) * (STS * STS) + (r % STS) * STS + (c % STS);
}

struct CsrDev {
    int32_t n;
    int32_t *ptr, *col;
    double* val;
};

struct LzState {                    // per component inverse-Lanczos bookkeeping
    int32_t active, kc, broke, status;
    double nb2, na2, nrm2, rr;
    double h[KMAX];
    double A[KMAX * KMAX], B[KMAX * KMAX];
    double wr[KMAX];
    double coef[KMAX];
    double theta_ritz[KMAX];
    double sc[KMAX];                 // scale of each stored (unnormalised) basis vector (cooperative path)
};

// kernel launchers (implemented in *.cu); all asynchronous on `st`
void launch_simp(const double* rho, double* Ee, int64_t nelem, double E0, double Emin, double p,
                 cudaStream_t st);
void upload_KE0(const double* ke, int nke, cudaStream_t st);
void upload_KE0_oc(const double* ke, int nke, cudaStream_t st);
int oc_blocks(int64_t n);
int launch_sensitivities(const MeshDev& m, const double* u, const double* rho, const double* Ee, double E0,
                         double Emin, double p, int64_t nelem, double* dc, double* part, OcState* st,
                         cudaStream_t s);
int launch_oc_update(const double* rho, const double* dc, int64_t n, const OcParams& prm, double* part,
                     OcState* st, double* rho_new, cudaStream_t s);
void launch_assemble_band(const MeshDev& m, const SubDesc* sd, int nsl, const int32_t* idofs,
                          const double* Ee, double* band, int ld, int band_w, int max_nI,
                          cudaStream_t st);
void launch_assemble_pairs(const MeshDev& m, const int32_t* da, const int32_t* db,
                           const int32_t* sub_of_entry, const double* Ee, double* val, int64_t n,
                           cudaStream_t st);
int launch_band_cholesky(const SubDesc* sd, int nsl, double* band, int ld, int band_w,
                         int* d_fail, cudaStream_t st);
void launch_apply_K(const MeshDev& m, const double* Ee, const double* u, const double* f,
                    const int8_t* cls, double* res, int64_t ndof, cudaStream_t st, const double* ulo = nullptr);
void launch_dd_accum(double* hi, double* lo, const double* d, int64_t n, cudaStream_t st);

enum SchurMode { SCHUR_APPLY = 0, SCHUR_CONDENSE = 1, SCHUR_BACKSUB = 2, SCHUR_COLUMNS = 3 };
struct SchurArgs {
    const SubDesc* sd;
    int nsl;
    const double* band;
    int ld, band_w;
    const int32_t* idofs;
    const int32_t* Rg;
    const int32_t* igp;
    const int32_t* ig_col;
    const double* ig_val;
    const int32_t* gxp;
    const int32_t* gx_col;
    const double* gx_val;
    double* scratch;
    const double* xin;      // interface vector (n_Gamma) gathered through Rg
    const double* f;        // full rhs (ndof) for condense/backsub
    double* qloc;           // per-subdomain local outputs
    double* u;              // full solution (backsub)
    const PcgState* state;  // early exit when state->done (may be null)
    int mode;
    int maxG;
    // SCHUR_COLUMNS (explicit S_s = columns S_s e_t): local subdomains [col_s0, col_s0+nsl)
    double* sexp;
    double* colscratch;     // nsl*maxG*max_nI doubles
    int col_s0, max_nI;
    int max_ig;             // max A_IG entries of one subdomain (shared-memory staging in the formation)
    // wide bands (k_schur_blk): inverses of the bs x bs diagonal blocks of L, [local subdomain][dinv_np][bs][bs]
    // row-major lower triangular (identity padding), formed after the factorisation; null = substitution chain
    const double* dinv;
    int dinv_np, dinv_bs;   // blocks per subdomain, block size (= panel width of the k_schur_blk variant in use)
};
int schur_blk_panel_width(int ld, int max_nI, int maxG);
void launch_blk_diag_inv(const SubDesc* sd, int nsl, const double* band, int ld, double* dinv, int dinv_np, int bs,
                         cudaStream_t st);
int launch_schur_local(const SchurArgs& a, cudaStream_t st);
// q_s = S_s x_s with the explicit column-major S_s (one CTA per subdomain, coalesced over rows)
void launch_schur_explicit(const SubDesc* sd, int nsl, const double* sexp, const int32_t* Rg, const double* xin,
                           double* qloc, int maxG, const PcgState* s, cudaStream_t st);
void prepare_schur_explicit(int maxG);
void prepare_schur_blk(int ld, int band_w, int max_nI, int maxG);

void launch_gather(const int32_t* gptr, const int32_t* gsrc, const double* qloc,
                   const double* add, double* q, int64_t nG, const PcgState* st_done,
                   cudaStream_t st);
// PCG building blocks (deterministic two-level reductions, device-side scalars)
struct RedBuf {
    double* part;
    unsigned int* counter;
    int nblk;
};
void launch_pcg_pq(const double* p, const double* q, int64_t n, RedBuf rb, PcgState* s,
                   cudaStream_t st);
void launch_gather_pq(const int32_t* gptr, const int32_t* gsrc, const double* qloc, const double* p, double* q,
                      int64_t n, RedBuf rb, PcgState* s, cudaStream_t st);
void launch_pcg_update_xr(double* x, double* r, double* r_old, const double* p, const double* q,
                          int64_t n, RedBuf rb, PcgState* s, cudaStream_t st);
void launch_pcg_rz(const double* r, const double* z, const double* r_old, int64_t n, int beta_pr,
                   RedBuf rb, PcgState* s, cudaStream_t st);
void launch_pcg_update_p(double* p, const double* z, int64_t n, PcgState* s, cudaStream_t st);
void launch_pcg_init(double* r, double* p, const double* z, const double* g, const double* Sx,
                     int64_t n, int mode, RedBuf rb, PcgState* s, cudaStream_t st);
void launch_norm2(const double* v, int64_t n, RedBuf rb, double* out, cudaStream_t st);
constexpr int FG_ND = 32;   // max FGMRES restart length + 1 (batched dot products)
void launch_multidot(const double* V, int64_t ld, int nv, const double* w, int64_t n, RedBuf rb, double* out,
                     cudaStream_t st);
void launch_multi_axpy(double* w, const double* V, int64_t ld, int nv, const double* coef, double sign, int64_t n,
                       cudaStream_t st);
void launch_scale_invnorm(double* dst, const double* src, const double* sq, int64_t n, cudaStream_t st);
void launch_copy(double* dst, const double* src, int64_t n, const PcgState* s, cudaStream_t st);
void launch_sum_slots(double* buf, const double* slots, int n, size_t cap, int64_t len, cudaStream_t st);
void launch_axpy(double* y, const double* x, double a, int64_t n, cudaStream_t st);
void launch_scatter_gamma(const int32_t* gamma_dofs, const double* uG, double* u, int64_t nG,
                          cudaStream_t st);
void launch_gather_gamma(const int32_t* gamma_dofs, const double* f, double* fG, int64_t nG,
                         cudaStream_t st);
void launch_zero_dirichlet(const int8_t* cls, double* u, int64_t ndof, cudaStream_t st);

// preconditioner
struct PrecDev {
    int32_t ncomp, nflat, kmax;
    int32_t jacobi_reg;         // Ritz-step Jacobi: 0 = whole CTA (default), 1 = one warp in registers (DE_JACOBI_REG), 2 = one warp from shared memory (DE_JACOBI_WARP)
    int32_t max_face_band;      // max half bandwidth over all face blocks (1: tridiagonal, 2D)
    int64_t comp_off[MAXC + 1];
    int32_t singular[MAXC];
    double theta;
    int32_t* cmap;
    CsrDev M, L, K;
    ElimDev eK, eM;
    double *rf, *s, *v, *w, *Mw, *y, *zf, *W, *LW, *MW;
    LzState* lz;
    double* part;
    unsigned int* counter;
    int nblk;
    // inner_mode 0 (SPEC face-PCG inner solves of K, R10): one cooperative kernel per solve
    int32_t inner_f, fp_nb, fp_maxit;
    size_t fp_smem;
    double fp_tol;
    double *fr, *fz, *fp, *fq, *fpart;
    unsigned long long* fits;   // inner PCG iterations accumulated over all solves (de_stats)
};
int fpcg_prepare(PrecDev& P, int device);   // blocks / smem of k_face_pcg; 0 if no cooperative launch
void prec_apply(const PrecDev& P, const double* r, double* z, const PcgState* s, cudaStream_t st,
                int* nlaunch);
void launch_gauss_jordan(double* A, double* Bbuf, int n, cudaStream_t st);
void prec_prepare(const PrecDev& P);   // one-time kernel attributes (outside graph capture)

// persistent cooperative preconditioner (kernels_prec_coop.cu)
struct CoopBuffers {
    int nb = 0, nsm = 148;
    size_t smem = 0;
    int stage = 0, per_warp = 0, mf = 0, ncmax = 0, nbc_max = 0, tridiag = 0, gram_cgs2 = 1, fold = 0, split = 1, shr = 0, sc_persist = 0;
    size_t sc_persist_bytes = 0;
    double* redf = nullptr;      // fold sums of the shared-row cross-point solve: [2][MAXC][NRED][nb]
    double* ucross = nullptr;   // fold: [KMAX][ncross of eK]
    unsigned int* arrive = nullptr;   // split-phase arrival counter of the fused eliminations (zero between launches)
    double *red = nullptr, *gram = nullptr, *gram_tot = nullptr, *w1 = nullptr, *mw1 = nullptr, *lw1 = nullptr;
    unsigned long long* timers = nullptr;   // phase stamps (diagnostics; env DE_PREC_TIMERS=1)
    const void* kfn = nullptr;              // k_prec_coop instantiation (basis bound, timers)
};
bool prec_coop_prepare(const PrecDev& P, int device, CoopBuffers& B);
size_t prec_coop_red_doubles(const CoopBuffers& B);
size_t prec_coop_gram_doubles(const CoopBuffers& B);
int prec_apply_coop(const PrecDev& P, const CoopBuffers& B, const double* r, double* z, const PcgState* s,
                    cudaStream_t st, bool literal = false);

}  // namespace de
