// kernels_prec_coop.cu — the interface preconditioner z = H^_theta^-1 r as one
// persistent cooperative kernel per application (k_prec_coop: seed, inverse-Lanczos steps, Gram matrices)
// followed by two small launches (k_prec_ritz: the k x k Ritz problems; k_prec_combine: z = W coef).
// Same algorithm as kernels_precond.cu (R7, R9, R10).
//
// Work distribution: block b serves component c = b % ncomp for row-parallel phases (rows
// lo_c + lb*RW + (tid-32), stride nbc*RW; warp 0 hosts the grid-barrier thread and does no row work);
// face solves are warp-per-face over all components; the cross-point GEMV is split over the component's
// blocks. Every scalar (norms, Gram-Schmidt coefficients) is a fixed-order sum of per-block partials that
// EVERY block recomputes after the barrier, so all blocks hold bitwise identical copies and no extra
// barrier is needed to broadcast them.
// Per Lanczos step (2D): exact K-solve (2 barriers: faces by parallel cyclic reduction + t_C; cross-point
// GEMV; the face correction x_F = y_F - G x_C is folded into the next phase) + phase A (M w, L w, dots h) +
// phase C (w - W (2h - G h) with the images by linearity, ||w||_M, Gram row) = 4 barriers: the second
// Gram-Schmidt pass is formed from the Gram matrix G = W^T M W (R21); env DE_CGS2_TWO_PASS runs the
// literal two-pass form (phase B = pass 1 over the rows, phase C = pass 2) for A/B runs and tests. With the fold
// (R22, 2D default) h is summed inside the elimination and phase A merges into C: 3 barriers per step.
#include "de_internal.h"

#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

namespace de {

constexpr int CT = 256;
constexpr int CW = CT / 32;
constexpr int NRED = KMAX + 2;
constexpr int RW = CT - 32;                   // rows per block chunk in row-parallel phases
constexpr int GW = 2 * KMAX + 1;              // Gram row j: G_L[j][t] (t<=j), G_M[j][t] (KMAX+t), (W^T r)[j] (2 KMAX)
constexpr int GRAM_TASKS = KMAX * GW;

struct CoopArgs {
    PrecDev P;
    const double* r;
    double* z;
    const PcgState* s;
    double* red;        // [2][MAXC][NRED][nbc_max]
    double* gram;       // [MAXC][KMAX rows][GW][nbc_max] per-block Gram partials
    double* gram_tot;   // [MAXC][KMAX rows][GW] their fixed-order sums
    double* w1;         // second Lanczos work vector (nflat)
    double* mw1;        // M w1 (nflat)
    double* lw1;        // L w1 (nflat)
    int nbc_max;
    int stage;          // 1: stage face factors in shared memory
    int per_warp;       // doubles of shared memory per warp for face solves
    int mf;             // max face size
    int ncmax;          // max cross points per component
    int tridiag;        // 1: every face block is tridiagonal with <= TRI_MAX nodes (2D) -> thread per face
    int gram_cgs2;      // 1: the second Gram-Schmidt pass is formed from the Gram matrix (one row pass fewer)
    int fold;           // 1 (with gram_cgs2, 2D fused eliminations): h = W^T M w is summed inside the elimination
    int smem_doubles;   // dynamic shared memory of the launch in doubles (fast-diagonalisation tables fit test)
    int shr;            // 1: a shared S_C^-1 (HElim::sc_shared) is applied for ALL components by the block that loads a row
    double* redf;       // [2][MAXC][NRED][nb] fold sums when shr (every block contributes to every component)
    int sc_persist;     // 1: eK's S_C^-1 sits in the persisting L2 set-aside (access-policy window of the launch): plain loads
    int split;          // 1: fused eliminations wait on the arrival counter between t_C and the cross-point solve (no grid barrier)
    double* ucross;     // [KMAX][ncross of eK]: u_t = G^T (M W_t)_F, the face part of M W_t folded onto cross points
    unsigned int* arrive;   // split-phase arrival counter of the fused eliminations (t_C published -> cross-point solve)
    unsigned long long* timers;   // optional phase timestamps (block 0), DE_PREC_TIMERS
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define STAMP(k)                                                        \
    do {                                                                \
        const int k_ = (k);   /* every thread advances its stamp counter */          \
        if (TIM && a.timers && blockIdx.x == 0 && threadIdx.x == 0) a.timers[k_] = gtimer(); \
    } while (0)

__device__ __forceinline__ int ccomp(const int64_t* off, int nc, int64_t i) {
    int c = 0;
    while (c + 1 < nc && i >= off[c + 1]) ++c;
    return c;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block-reduce vals[0..nv) and write this block's partials into red[pp][c][v][lb]
template <int NV>
__device__ void block_partials(const CoopArgs& a, const double (&vals)[NV], int nv, int pp, int c, int lb,
                               double (*sred)[NRED]) {
    static_assert(NV <= NRED, "partials buffer");
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        if (v < nv) {
            const double t = warp_sum(vals[v]);
            if (lane == 0) sred[w][v] = t;
        }
    }
    __syncthreads();
    if (threadIdx.x < nv) {
        double t = 0.0;
        for (int k = 0; k < CW; ++k) t += sred[k][threadIdx.x];
        a.red[((size_t(pp) * MAXC + c) * NRED + threadIdx.x) * a.nbc_max + lb] = t;
    }
    __syncthreads();
}

// totals of all components (fixed order over lb) into tot[c][v]
__device__ void read_totals(const CoopArgs& a, int pp, int nv, int nb, double (*tot)[NRED], bool all = false) {
    // all: the fold sums of the shared-row cross-point solve (a.redf: one slot per block of the WHOLE grid per component)
    // task (c, v) = sum over the component's nbc block partials: lane l adds b = l, l+32, ... in order, then a
    // warp tree (fixed order); TU tasks per warp and QU partials per lane are loaded together
    constexpr int TU = 3, QU = 8;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nc = a.P.ncomp, ntask = nc * nv;
    for (int t0 = w; t0 < ntask; t0 += CW * TU) {
        double acc[TU];
        const double* p[TU];
        int nbc[TU];
#pragma unroll
        for (int u = 0; u < TU; ++u) {
            const int t = min(t0 + u * CW, ntask - 1), c = t / nv, v = t - c * nv;
            nbc[u] = (t0 + u * CW < ntask) ? (all ? nb : (nb - c + nc - 1) / nc) : 0;
            p[u] = all ? a.redf + ((size_t(pp) * MAXC + c) * NRED + v) * nb
                       : a.red + ((size_t(pp) * MAXC + c) * NRED + v) * a.nbc_max;
            acc[u] = 0.0;
        }
        for (int b0 = 0; b0 < (all ? nb : a.nbc_max); b0 += 32 * QU) {
            double x[TU][QU];
#pragma unroll
            for (int u = 0; u < TU; ++u)
#pragma unroll
                for (int q = 0; q < QU; ++q) {
                    const int bb = b0 + lane + 32 * q;
                    x[u][q] = bb < nbc[u] ? *((volatile const double*)(p[u] + bb)) : 0.0;
                }
#pragma unroll
            for (int u = 0; u < TU; ++u)
#pragma unroll
                for (int q = 0; q < QU; ++q) acc[u] += x[u][q];
        }
#pragma unroll
        for (int u = 0; u < TU; ++u) {
            const double sum = warp_sum(acc[u]);
            const int t = t0 + u * CW;
            if (lane == 0 && t < ntask) tot[t / nv][t - (t / nv) * nv] = sum;
        }
    }
    __syncthreads();
}

// per-thread Gram accumulators gacc[v * CT + tid], v < GW
__device__ __forceinline__ void gram_zero(double* gacc) {
#pragma unroll
    for (int v = 0; v < GW; ++v) gacc[v * CT + threadIdx.x] = 0.0;
}

// block sums of gacc (fixed order) -> a.gram partial slots of Gram row j of component c
__device__ void gram_partials(const CoopArgs& a, const double* gacc, int c, int lb, int j) {
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int v = w; v < GW; v += CW) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < CW; ++q) t += gacc[v * CT + q * 32 + lane];
        t = warp_sum(t);
        if (lane == 0) a.gram[((size_t(c) * KMAX + j) * GW + v) * a.nbc_max + lb] = t;
    }
    __syncthreads();
}

// Fixed-order sums of Gram row jr (every accepted component), one entry per warp: entry tasks
// tau = first, first + stride, ...; lanes add the block partials b = lane, lane+32, .. in order, then a warp tree.
__device__ void gram_row_sums(const CoopArgs& a, int jr, const int* kcs, int first, int stride, int nb) {
    constexpr int TU = 6;   // entries per warp in flight
    const int lane = threadIdx.x & 31, nc = a.P.ncomp, per = 2 * (jr + 1) + 1;
    for (int tau0 = first; tau0 < nc * per; tau0 += stride * TU) {
        const double* pg[TU];
        size_t dst[TU];
        int nbcc[TU];
#pragma unroll
        for (int u = 0; u < TU; ++u) {
            const int tau = tau0 + u * stride, cc = min(tau / per, nc - 1), q = tau - cc * per;
            const int v = q <= jr ? q : (q < 2 * (jr + 1) ? KMAX + (q - jr - 1) : 2 * KMAX);
            const bool ok = tau < nc * per && jr < kcs[cc];
            nbcc[u] = ok ? (nb - cc + nc - 1) / nc : 0;
            pg[u] = a.gram + ((size_t(cc) * KMAX + jr) * GW + v) * a.nbc_max;
            dst[u] = ok ? (size_t(cc) * KMAX + jr) * GW + v : ~size_t(0);
        }
        double acc[TU];
#pragma unroll
        for (int u = 0; u < TU; ++u) acc[u] = 0.0;
        for (int b = lane; b < a.nbc_max; b += 32)
#pragma unroll
            for (int u = 0; u < TU; ++u) acc[u] += b < nbcc[u] ? pg[u][b] : 0.0;
#pragma unroll
        for (int u = 0; u < TU; ++u) {
            const double t = warp_sum(acc[u]);
            if (lane == 0 && dst[u] != ~size_t(0)) a.gram_tot[dst[u]] = t;
        }
    }
}

// (M x)_i and (L x)_i by one pass over the shared sparsity pattern (M and L are assembled on the same trace
// facets; host_setup checks that the patterns agree)
__device__ __forceinline__ void spmv_ml(const CsrDev& M, const CsrDev& L, int64_t i, const double* __restrict__ x,
                                        double& yM, double& yL) {
    double am = 0.0, al = 0.0;
    for (int e = M.ptr[i]; e < M.ptr[i + 1]; ++e) {
        const double v = x[M.col[e]];
        am += M.val[e] * v;
        al += L.val[e] * v;
    }
    yM = am;
    yL = al;
}

// x_i of the last exact elimination when its third phase is folded into the consumer (ElimDev::fuse):
// face node y_i - G_i x_C, cross point x_C (v0 = -1, y_i = 0)
__device__ __forceinline__ double elim_value(const ElimDev& E, int64_t i, const double* __restrict__ y,
                                             const double* __restrict__ xC) {
    return y[i] - E.g_v0[i] * xC[E.g_c0[i]] - E.g_v1[i] * xC[E.g_c1[i]];
}

// (M x)_i and (L x)_i with x = elim_value(E, .) (M and L share one sparsity pattern); returns x_i
__device__ __forceinline__ double spmv_elim(const CsrDev& M, const CsrDev& L, int64_t i, const ElimDev& E,
                                            const double* __restrict__ y, const double* __restrict__ xC,
                                            double& yM, double& yL) {
    const int e0 = M.ptr[i], e1 = M.ptr[i + 1];
    double am = 0.0, al = 0.0, xi = 0.0;
    for (int e = e0; e < e1; ++e) {
        const int col = M.col[e];
        const double x = elim_value(E, col, y, xC);
        am += M.val[e] * x;
        al += L.val[e] * x;
        if (col == i) xi = x;
    }
    if (e0 == e1) xi = elim_value(E, i, y, xC);
    yM = am;
    yL = al;
    return xi;
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// spmv_elim through the fold ELL (ElimDev::fell_*): all entry data of row i in one level, then y / x_C in the
// second; rows flagged -1 take the CSR path. Same arithmetic and summation order as spmv_elim.
__device__ __forceinline__ double spmv_elim_fell(const CsrDev& M, const CsrDev& L, int64_t i, const ElimDev& E,
                                                 const double* __restrict__ y, const double* __restrict__ xC,
                                                 int64_t nfl, double& yM, double& yL) {
    const int c0 = E.fell_col[i];
    if (c0 < 0) return spmv_elim(M, L, i, E, y, xC, yM, yL);
    int col[FELL_W], g0[FELL_W], g1[FELL_W];
    double v0[FELL_W], v1[FELL_W], mv[FELL_W], lv[FELL_W];
#pragma unroll
    for (int k = 0; k < FELL_W; ++k) {
        const int64_t at = k * nfl + i;
        col[k] = k == 0 ? c0 : E.fell_col[at];
        g0[k] = E.fell_c0[at];
        g1[k] = E.fell_c1[at];
        v0[k] = E.fell_v0[at];
        v1[k] = E.fell_v1[at];
        mv[k] = E.fell_m[at];
        lv[k] = E.fell_l[at];
    }
    double am = 0.0, al = 0.0, xi = 0.0;
#pragma unroll
    for (int k = 0; k < FELL_W; ++k) {
        const double x = y[col[k]] - v0[k] * xC[g0[k]] - v1[k] * xC[g1[k]];
        am += mv[k] * x;
        al += lv[k] * x;
        if (col[k] == i) xi = x;   // padding repeats column i: the same value
    }
    yM = am;
    yL = al;
    return xi;
}

// spmv_elim through the row patterns (ElimDev::pat_*): every address of the first load level follows from i alone
// (the row's couplings, y and the couplings of its flat neighbours), the second level is the face's two x_C values
// and the pattern table (L1); rows without a pattern (cross points) take the general path. 36 distinct bytes per row
// instead of the fold ELL's 132 + nine gathers.
__device__ __forceinline__ double spmv_elim_pat(const CsrDev& M, const CsrDev& L, int64_t i, const ElimDev& E,
                                                const double* __restrict__ y, const double* __restrict__ xC,
                                                int64_t nfl, double& yM, double& yL) {
    const int pid = E.pat_id[i];
    const int64_t im = i > 0 ? i - 1 : i, ip = i + 1 < nfl ? i + 1 : i;
    const int c0 = E.g_c0[i], c1 = E.g_c1[i];
    const double ym = y[im], y0 = y[i], yp = y[ip];
    const double am0 = E.g_v0[im], a00 = E.g_v0[i], ap0 = E.g_v0[ip];
    const double am1 = E.g_v1[im], a01 = E.g_v1[i], ap1 = E.g_v1[ip];
    if (pid <= -2 && E.xell_col) {   // cross-point row: its ELL (entry data in one level, then y / x_C of each neighbour)
        const int ci = -2 - pid;
        int col[XELL_W], g0[XELL_W], g1[XELL_W];
        double v0[XELL_W], v1[XELL_W], mv[XELL_W], lv[XELL_W];
#pragma unroll
        for (int k = 0; k < XELL_W; ++k) {
            const size_t at = size_t(k) * E.ncross + ci;
            col[k] = E.xell_col[at];
            g0[k] = E.xell_c0[at];
            g1[k] = E.xell_c1[at];
            v0[k] = E.xell_v0[at];
            v1[k] = E.xell_v1[at];
            mv[k] = E.xell_m[at];
            lv[k] = E.xell_l[at];
        }
        double am = 0.0, al = 0.0, xi = 0.0;
#pragma unroll
        for (int k = 0; k < XELL_W; ++k) {
            const double x = y[col[k]] - v0[k] * xC[g0[k]] - v1[k] * xC[g1[k]];
            am += mv[k] * x;
            al += lv[k] * x;
            if (col[k] == i) xi = x;   // padding repeats column i with zero coefficients: the same value
        }
        yM = am;
        yL = al;
        return xi;
    }
    if (pid < 0)
        return E.fell_col ? spmv_elim_fell(M, L, i, E, y, xC, nfl, yM, yL) : spmv_elim(M, L, i, E, y, xC, yM, yL);
    const double xa = xC[c0], xb = xC[c1];
    const int code = E.pat_code[pid];
    double pm[3], pl[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        pm[k] = E.pat_m[3 * pid + k];
        pl[k] = E.pat_l[3 * pid + k];
    }
    const double xm = ym - am0 * xa - am1 * xb, x0 = y0 - a00 * xa - a01 * xb, xp = yp - ap0 * xa - ap1 * xb;
    double am = 0.0, al = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int src = (code >> (3 * k)) & 7;
        const double x = src == 0 ? xm : (src == 1 ? x0 : (src == 2 ? xp : (src == 3 ? xa : (src == 4 ? xb : 0.0))));
        am = fma(pm[k], x, am);
        al = fma(pl[k], x, al);
    }
    yM = am;
    yL = al;
    return x0;
}

// Warp solve of one face block (L then M = P L^T P forward sweeps, b <= 31, row window in registers).
// rhs = scale * b_F (mode 0) or scale * b_F - X_FC xC (mode 1). The factor columns stream through a two-chunk
// shared-memory ring (32 columns per chunk, cp.async issued one chunk ahead), so no load sits on the per-row
// dependency chain (measured: per-row global loads made the 3D face phases 37-92 us).
__device__ void face_warp(const CoopArgs& a, const ElimDev& E, int F, const double* __restrict__ b,
                          const double* scl, const double* __restrict__ xC, double* __restrict__ out, int mode,
                          double* wsm, int lane) {
    __syncwarp();
    const PrecDev& P = a.P;
    const int o = E.face_off[F], n = E.face_off[F + 1] - o, bw = E.face_band[F], ld = bw + 1;
    double* rb = wsm;
    double* ys = wsm + a.mf;
    int* idx = reinterpret_cast<int*>(wsm + 2 * a.mf);
    double* cbuf = wsm + 3 * a.mf;                // [2][32 * ld] column chunks
    const int cstride = 32 * ld;
    const double* gf = E.face_fac + E.face_fac_off[F];
    const double sc = scl[ccomp(P.comp_off, P.ncomp, E.face_nodes[o])];
    for (int i = lane; i < n; i += 32) {
        const int node = E.face_nodes[o + i];
        idx[i] = node;
        double r = sc * b[node];
        if (mode == 1)
            for (int e = E.xfc_ptr[o + i]; e < E.xfc_ptr[o + i + 1]; ++e) r -= E.xfc_val[e] * xC[E.xfc_col[e]];
        rb[i] = r;
    }
    __syncwarp();
    for (int sw = 0; sw < 2; ++sw) {
        const double* __restrict__ fac = gf + (sw == 0 ? 0 : size_t(n) * ld);
        const double* __restrict__ src = sw == 0 ? rb : ys;
        double* dst = sw == 0 ? ys : rb;          // both in shared memory; y reversed, then x reversed back
        const int nch = (n + 31) / 32;
        {   // chunk 0
            const int cnt = min(32, n) * ld;
            for (int i = lane; i < cnt; i += 32) cp_async8(cbuf + i, fac + i);
            cp_async_commit();
        }
        double v = lane < n ? src[lane] : 0.0;
        double outv = 0.0;                        // lane l keeps the solution of rows = l (mod 32)
        __syncwarp();
        for (int ch = 0; ch < nch; ++ch) {
            const int j0 = 32 * ch, jn = min(32, n - j0);
            if (ch + 1 < nch) {                   // next chunk into the other buffer (its last reader was ch - 1)
                const int cnt = min(32, n - j0 - 32) * ld;
                double* nb = cbuf + ((ch + 1) & 1) * cstride;
                const double* gs = fac + size_t(j0 + 32) * ld;
                for (int i = lane; i < cnt; i += 32) cp_async8(nb + i, gs + i);
            }
            cp_async_commit();                    // (possibly empty) group: wait_group 1 then covers chunk ch
            cp_async_wait1();
            __syncwarp();
            const double* cb = cbuf + (ch & 1) * cstride;
#pragma unroll 4
            for (int jj = 0; jj < jn; ++jj) {
                const int j = j0 + jj;
                const double* col = cb + jj * ld;
                const double cl = (lane >= 1 && lane <= bw) ? col[lane] : 0.0;
                const double c0 = col[0];
                const double nxt = (j + 32 < n) ? src[j + 32] : 0.0;   // row entering lane 31 (uniform load)
                const double yj = __shfl_sync(0xffffffffu, v, 0) * c0;
                v = fma(-cl, yj, v);
                const double vs = __shfl_down_sync(0xffffffffu, v, 1);
                v = (lane == 31) ? nxt : vs;                           // branch-free: keeps the warp converged
                outv = (lane == jj) ? yj : outv;
            }
            __syncwarp();
            if (lane < jn) dst[n - 1 - (j0 + lane)] = outv;            // flush this block's solutions
            __syncwarp();
        }
    }
    for (int i = lane; i < n; i += 32) out[idx[i]] = rb[i];
    __syncwarp();
}

// Warp solve of one 3D face block through its block-bidiagonal form (ElimDev::fb): y = X_FF^-1 (scale b_F).
// Lanes 0-15 apply F_i (F_i^T) to the block's right-hand side, lanes 16-31 apply G_i (H_i) to the previous block's
// solution; one shuffle per column broadcasts the vector entry inside each half, a xor-16 shuffle combines the halves.
// 2 ceil(n / 16) steps of 16 independent FMAs instead of 2 n dependent shuffle-FMA rows; the next step's matrix
// columns are loaded before the current step's products.
__device__ void face_warp_blocks(const CoopArgs& a, const ElimDev& E, int F, const double* __restrict__ b,
                                 const double* scl, double* __restrict__ out, double* wsm, int lane) {
    constexpr int BS = FB_BS, BB = BS * BS;
    const unsigned FULL = 0xffffffffu;
    const PrecDev& P = a.P;
    const int o = E.face_off[F], n = E.face_off[F + 1] - o;
    const int nbk = E.fb_off[F + 1] - E.fb_off[F];
    const double* __restrict__ tab = E.fb + size_t(E.fb_off[F]) * 4 * BB;
    const double sc = scl[ccomp(P.comp_off, P.ncomp, E.face_nodes[o])];
    const int row = lane & (BS - 1), half = lane >> 4, hsrc = lane & BS;   // shuffle source base of this half
    double* ys = wsm;   // [nbk * BS] forward solution, per warp
    __syncwarp();
    double m[BS], mn[BS];
#pragma unroll
    for (int c = 0; c < BS; ++c) mn[c] = tab[size_t(half) * BB + c * BS + row];   // step 0: F_0 | G_0
    double yprev = 0.0;
    for (int i = 0; i < nbk; ++i) {
        const int gi = BS * i + row;
        const double r = gi < n ? sc * b[E.face_nodes[o + gi]] : 0.0;
#pragma unroll
        for (int c = 0; c < BS; ++c) m[c] = mn[c];
        if (i + 1 < nbk) {
#pragma unroll
            for (int c = 0; c < BS; ++c) mn[c] = tab[(size_t(i + 1) * 4 + half) * BB + c * BS + row];
        } else {   // first backward step: F^T | H of the last block
#pragma unroll
            for (int c = 0; c < BS; ++c) mn[c] = tab[(size_t(nbk - 1) * 4 + 2 + half) * BB + c * BS + row];
        }
        const double v = half ? yprev : r;
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < BS; ++c) acc = fma(m[c], __shfl_sync(FULL, v, hsrc + c), acc);
        const double t = __shfl_xor_sync(FULL, acc, BS);
        yprev = half ? t - acc : acc - t;   // F r - G y_prev, in both halves
        if (!half) ys[gi] = yprev;
    }
    __syncwarp();
    double xnext = 0.0;
    for (int i = nbk - 1; i >= 0; --i) {
        const int gi = BS * i + row;
#pragma unroll
        for (int c = 0; c < BS; ++c) m[c] = mn[c];
        if (i > 0) {
#pragma unroll
            for (int c = 0; c < BS; ++c) mn[c] = tab[(size_t(i - 1) * 4 + 2 + half) * BB + c * BS + row];
        }
        const double v = half ? xnext : ys[gi];
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < BS; ++c) acc = fma(m[c], __shfl_sync(FULL, v, hsrc + c), acc);
        const double t = __shfl_xor_sync(FULL, acc, BS);
        xnext = half ? t - acc : acc - t;   // F^T y - H x_next
        if (!half && gi < n) out[E.face_nodes[o + gi]] = xnext;
    }
    __syncwarp();
}

// Thread solve of one tridiagonal face block (2D: every face is a path of <= 64 trace nodes):
// forward y_j = (r_j - L_{j,j-1} y_{j-1}) / L_jj, backward x_j = (y_j - L_{j+1,j} x_{j+1}) / L_jj.
// The face data is interleaved over groups of 32 faces (ElimDev::tri_*), so lane l of a warp reads
// entry j of face 32g+l with one coalesced access per step; the 2*n-step recurrence stays in registers.
__device__ void face_thread_tridiag(const CoopArgs& a, const ElimDev& E, int F, const double* __restrict__ b,
                                    const double* scl, const double* __restrict__ xC, double* __restrict__ out,
                                    int mode, double* ysm) {
    const PrecDev& P = a.P;
    const int n = E.tri_n[F];
    const size_t base = size_t(F / 32) * TRI_N * 32 + (F % 32);
    const double sc = scl[ccomp(P.comp_off, P.ncomp, E.tri_node[base])];
    int xj0 = -1, xj1 = -1;
    double xr0 = 0.0, xr1 = 0.0;
    if (mode == 1) {
        xj0 = E.tri_xj[2 * F];
        xj1 = E.tri_xj[2 * F + 1];
        if (xj0 >= 0) xr0 = E.tri_xv[2 * F] * xC[E.tri_xc[2 * F]];
        if (xj1 >= 0) xr1 = E.tri_xv[2 * F + 1] * xC[E.tri_xc[2 * F + 1]];
    }
    constexpr int U = 8;                            // rows per chunk: all loads of a chunk in flight together
    double prev = 0.0, lprev = 0.0;
    for (int j0 = 0; j0 < n; j0 += U) {
        double r[U], inv[U], sub[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = j0 + u;
            r[u] = 0.0;
            inv[u] = 0.0;
            sub[u] = 0.0;
            if (j < n) {
                const size_t at = base + size_t(j) * 32;
                r[u] = sc * b[E.tri_node[at]] - (j == xj0 ? xr0 : 0.0) - (j == xj1 ? xr1 : 0.0);
                inv[u] = E.tri_inv[at];
                sub[u] = E.tri_sub[at];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (j0 + u < n) {
                prev = (r[u] - lprev * prev) * inv[u];
                ysm[(j0 + u) * RW] = prev;
                lprev = sub[u];
            }
        }
    }
    double nxt = 0.0;
    for (int j1 = n - 1; j1 >= 0; j1 -= U) {
        double inv[U], sub[U];
        int node[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = j1 - u;
            inv[u] = 0.0;
            sub[u] = 0.0;
            node[u] = 0;
            if (j >= 0) {
                const size_t at = base + size_t(j) * 32;
                inv[u] = E.tri_inv[at];
                sub[u] = E.tri_sub[at];
                node[u] = E.tri_node[at];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = j1 - u;
            if (j >= 0) {
                nxt = (ysm[j * RW] - sub[u] * nxt) * inv[u];
                out[node[u]] = nxt;
            }
        }
    }
}

// Warp solve of one tridiagonal face block by parallel cyclic reduction (lane j = node j; coefficients
// precomputed per level, ElimDev::pcr): y_F = X_FF^-1 (scale * b_F). Same result as the Cholesky sweeps up to
// rounding (X_FF is diagonally dominant: K = L (+ M) and M on a path).
// NF faces per call (F0 + f * stride, f < NF; F >= fend skipped) with every load issued before the first use.
// KH > 0 (R22 fold): also accumulate this lane's share of the face part of h_t = (M W_t)^T x, i.e.
// hl[t] += MW_t[i] y_i over the face nodes i it solved, t < kc.
template <int NF, int KH>
__device__ __forceinline__ void face_warp_pcr(const PrecDev& P, const ElimDev& E, int F0, int stride, int fend,
                                              const double* __restrict__ b, const double* scl,
                                              double* __restrict__ y, int lane, double* hl = nullptr, int kc = 0,
                                              const int32_t* __restrict__ bmap = nullptr) {
    int n[NF], node[NF];
    double co[NF][PCR_Q], x[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) {
        const int F = F0 + f * stride;
        const bool ok = F < fend;
        const int Fc = ok ? F : 0;
        const int nt = E.pcr_nt[Fc];
        n[f] = ok ? (nt & 0xff) : 0;
        node[f] = E.pcr_node[size_t(Fc) * 32 + lane];
        const double* __restrict__ q = E.pcr + size_t(nt >> 8) * PCR_Q * 32;
#pragma unroll
        for (int k = 0; k < PCR_Q; ++k) co[f][k] = q[k * 32 + lane];
    }
#pragma unroll
    for (int f = 0; f < NF; ++f) {
        const double sc = scl[ccomp(P.comp_off, P.ncomp, __shfl_sync(0xffffffffu, node[f], 0))];
        x[f] = lane < n[f] ? sc * b[bmap ? bmap[node[f]] : node[f]] : 0.0;
    }
    if (KH > 0)   // the fold's M W_t rows of these nodes into L1 now, so their loads after the reduction hit
#pragma unroll
        for (int f = 0; f < NF; ++f)
            if (lane < n[f])
                for (int t = 0; t < kc; ++t)
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(P.MW + size_t(t) * P.nflat + node[f]));
#pragma unroll
    for (int l = 0; l < PCR_L; ++l) {
        const int sg = 1 << l;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            const double xm = __shfl_up_sync(0xffffffffu, x[f], sg), xp = __shfl_down_sync(0xffffffffu, x[f], sg);
            x[f] += co[f][2 * l] * xm + co[f][2 * l + 1] * xp;   // out-of-range neighbours: zero coefficients
        }
    }
#pragma unroll
    for (int f = 0; f < NF; ++f) {
        const double yv = x[f] * co[f][2 * PCR_L];
        if (lane < n[f]) y[node[f]] = yv;
        if (KH > 0 && lane < n[f]) {
            double mw[KH > 0 ? KH : 1];
#pragma unroll
            for (int t = 0; t < KH; ++t) mw[t] = t < kc ? P.MW[size_t(t) * P.nflat + node[f]] : 0.0;
#pragma unroll
            for (int t = 0; t < KH; ++t) hl[t] = fma(mw[t], yv, hl[t]);
        }
    }
}

// Rows [rlo, rhi) of x_C = S_C^-1 t_C: warp w takes the column slice [c0, c1) of all of them, RB rows x NA loads per
// lane in flight; warp partials into part[w][row]. STREAM: evict-first loads (the matrix is streamed once per
// elimination); false: plain loads for a matrix held in the persisting L2 set-aside (CoopArgs::sc_persist).
template <bool STREAM>
__device__ __forceinline__ void sc_rows(const double* __restrict__ S, int ncc, int rlo, int rhi, int nr, int c0, int c1,
                                        int w, int lane, const double* tC, double* part) {
    constexpr int NA = 8, RB = 4;
    for (int r = rlo; r < rhi; r += RB) {
        const double* __restrict__ row[RB];
        double sr[RB];
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            row[u] = S + size_t(r + u < rhi ? r + u : r) * ncc;
            sr[u] = 0.0;
        }
        for (int j = c0 + lane; j < c1; j += 32 * NA) {
            double v[RB][NA], t[NA];
#pragma unroll
            for (int q = 0; q < NA; ++q) {
                const int jj = j + 32 * q;
                const bool ok = jj < c1;
                // streamed once per step (evict-first); a shared S_C^-1 (HElim::sc_shared) is read by the blocks of
                // every component at about the same time, and evict-first lines still serve the partner (measured
                // again in round 2 with the lighter consumer: cached loads 0.615 vs 0.578 ms)
#pragma unroll
                for (int u = 0; u < RB; ++u)
                    v[u][q] = (ok && r + u < rhi) ? (STREAM ? __ldcs(row[u] + jj) : __ldg(row[u] + jj)) : 0.0;
                t[q] = ok ? tC[jj] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < NA; ++q)
#pragma unroll
                for (int u = 0; u < RB; ++u) sr[u] += v[u][q] * t[q];
        }
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            const double su = warp_sum(sr[u]);
            if (lane == 0 && r + u < rhi) part[w * nr + (r + u - rlo)] = su;
        }
    }
}

// which cross-point solve an elimination uses in block component c (the same answer in elim_coop and in the caller)
__device__ __forceinline__ bool use_fd(const CoopArgs& a, const ElimDev& E, int c) {
    const int ncc = E.cross_comp_off[c + 1] - E.cross_comp_off[c];
    return E.tri && E.fuse && E.fd && ncc > 0 &&
           2 * ncc + (ncc & 1) + E.fd_nx * E.fd_nx + E.fd_ny * E.fd_ny <= a.smem_doubles;
}
__device__ __forceinline__ bool use_shr(const CoopArgs& a, const ElimDev& E, int c) {
    const int ncc = E.cross_comp_off[c + 1] - E.cross_comp_off[c];
    return a.shr && E.sc_shared && ncc > 0 && !use_fd(a, E, c) && ((E.tri && E.fuse) || (!E.tri && E.xcf_w > 0));
}

// x = X^-1 (scl * b) by exact elimination (faces -> cross points -> faces); 3 grid barriers.
// fold_j > 0 (K-solve of Lanczos step fold_j, fused 2D path): the first phase also stores u_{j-1} = G^T b_F
// (b = M W_{j-1} raw), and the second phase accumulates the block partials of h_t = (M W_t) . x for t < kc,
// x = X^-1 (scl b) = y - G x_C (R22): h_t = sum_i MW_t[i] y_i + sum_k (MW_t[cf_k] - u_t[k]) x_C[k],
// written to the reduction slots (pp, c, 1 + t) like block_partials.
template <int KM, bool TIM>
__device__ void elim_coop(cg::grid_group& grid, const CoopArgs& a, const ElimDev& E, const double* b,
                          const double* scl, double* out, double* dsm, int c, int lb, int nbc, int& stamp, int& nelim,
                          int fold_j = 0, int kc = 0, int pp = 0, int64_t r0 = 0, int64_t rs = 1,
                          const int32_t* __restrict__ bmap = nullptr, const int* kcs_all = nullptr) {
    // bmap (fused path only): the right-hand side is b[bmap[i]] -- the seed solve reads r through the skeleton map,
    // so no gather phase (and barrier) precedes it
    const PrecDev& P = a.P;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // warp 0 hosts the grid-barrier thread; it comes out of every barrier late, so face solves run
    // on warps 1..CW-1 only (measured: warp 0 otherwise sets the phase time)
    // warp-major over blocks: consecutive face groups land on different SMs (block-major would put every
    // face on the first few dozen blocks); tridiagonal faces: warp gw takes the 32-face group gw
    const int gw = (w - 1) * int(gridDim.x) + blockIdx.x, nwarps = gridDim.x * (CW - 1);
    const int gt = gw * 32 + lane, nthr = nwarps * 32;
    double* y = P.y;
    double* xC = P.y + P.nflat;
    double* wsm = dsm + size_t(w > 0 ? w - 1 : 0) * a.per_warp;   // warp 0 (barrier host) does no face solves
    long long tf0 = clock64();
    const bool fused = E.tri && E.fuse;
    __shared__ double hfw[CW * KMAX];   // fold: the face part of h per warp, read after the cross-point solve
    // fast-diagonalised cross-point solve (HElim::fd): X, Y and the Q tables must fit the dynamic shared memory
    const int nccb = E.cross_comp_off[c + 1] - E.cross_comp_off[c];
    const int fdq = 2 * nccb + (nccb & 1);   // offset of the staged Q tables (16-byte aligned)
    const bool fd = use_fd(a, E, c);
    if (fused) {
        ++nelim;
        if (fd) {   // stage Qx, Qy behind X / Y now (static tables; dsm is free here): they land during the face solves
            const int nx = E.fd_nx, ny = E.fd_ny, cs = E.sc_shared ? 0 : c;
            const double* gx = E.fd_qx + size_t(cs) * nx * nx;
            const double* gy = E.fd_qy + size_t(cs) * ny * ny;
            double* sq = dsm + fdq;
            for (int i = threadIdx.x; i < nx * nx; i += CT) cp_async8(sq + i, gx + i);
            for (int i = threadIdx.x; i < ny * ny; i += CT) cp_async8(sq + nx * nx + i, gy + i);
            cp_async_commit();
        }
        // t_C = scale (b_C - G^T b_F) once per cross point (needs only b), two cross points per warp in flight.
        // Formed FIRST and published through a split-phase arrival counter: the cross-point solve below waits for
        // every block's arrival instead of a grid barrier, and the face solves (which it does not need) run in between.
        if (w > 0 && E.td_start) {   // through the face descriptors: one level, then coalesced g and b loads
            double* tCg = P.y + P.nflat + E.ncross;
            for (int ci0 = gw; ci0 < E.ncross; ci0 += 2 * nwarps) {
                int st[2][XCF_W], ln[2][XCF_W], cf[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int ci = ci0 + u * nwarps;
                    const bool ok = ci < E.ncross;
                    cf[u] = ok ? E.cross_flat[ci] : 0;
#pragma unroll
                    for (int f = 0; f < XCF_W; ++f) {
                        st[u][f] = ok ? E.td_start[size_t(f) * E.ncross + ci] : 0;
                        ln[u][f] = ok ? E.td_len[size_t(f) * E.ncross + ci] : 0;
                    }
                }
                double gv[2][XCF_W], bv[2][XCF_W];
#pragma unroll
                for (int u = 0; u < 2; ++u)
#pragma unroll
                    for (int f = 0; f < XCF_W; ++f) {
                        const int n = ln[u][f] & 0xff, i = st[u][f] + lane;
                        const bool ok = lane < n;
                        gv[u][f] = ok ? ((ln[u][f] >> 8) ? E.g_v1[i] : E.g_v0[i]) : 0.0;
                        bv[u][f] = ok ? b[bmap ? bmap[i] : i] : 0.0;
                    }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int ci = ci0 + u * nwarps;
                    double acc = 0.0;
#pragma unroll
                    for (int f = 0; f < XCF_W; ++f) acc = fma(gv[u][f], bv[u][f], acc);
                    const double sgt = warp_sum(acc);
                    if (lane == 0 && ci < E.ncross) {
                        tCg[ci] = scl[ccomp(P.comp_off, P.ncomp, cf[u])] * (b[bmap ? bmap[cf[u]] : cf[u]] - sgt);
                        if (fold_j > 0) a.ucross[size_t(fold_j - 1) * E.ncross + ci] = sgt;
                    }
                }
            }
        } else if (w > 0) {
            double* tCg = P.y + P.nflat + E.ncross;
            for (int ci0 = gw; ci0 < E.ncross; ci0 += 2 * nwarps) {
                double acc[2] = {0.0, 0.0};
                int e0[2], e1[2], cf[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int ci = ci0 + u * nwarps;
                    const bool ok = ci < E.ncross;
                    e0[u] = ok ? E.gt_ptr[ci] : 0;
                    e1[u] = ok ? E.gt_ptr[ci + 1] : 0;
                    cf[u] = ok ? E.cross_flat[ci] : 0;
                }
                const int len = max(e1[0] - e0[0], e1[1] - e0[1]);
                for (int k = lane; k < len; k += 64) {
                    double v[2][2], x[2][2];
#pragma unroll
                    for (int u = 0; u < 2; ++u)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int e = e0[u] + k + 32 * h;
                            const bool ok = e < e1[u];
                            v[u][h] = ok ? E.gt_val[e] : 0.0;
                            x[u][h] = ok ? b[bmap ? bmap[E.gt_col[e]] : E.gt_col[e]] : 0.0;
                        }
#pragma unroll
                    for (int u = 0; u < 2; ++u) acc[u] += v[u][0] * x[u][0] + v[u][1] * x[u][1];
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int ci = ci0 + u * nwarps;
                    const double sgt = warp_sum(acc[u]);
                    if (lane == 0 && ci < E.ncross) {
                        tCg[ci] = scl[ccomp(P.comp_off, P.ncomp, cf[u])] * (b[bmap ? bmap[cf[u]] : cf[u]] - sgt);
                        if (fold_j > 0) a.ucross[size_t(fold_j - 1) * E.ncross + ci] = sgt;
                    }
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 32) {   // publish this block's share of t_C (release: fence, then the arrival)
            __threadfence();
            atomicAdd(a.arrive, 1u);
        }
        // warp per face (PCR); each face lies in one component, solved by that component's blocks
        const int lw = (w - 1) * nbc + lb, nwc = (CW - 1) * nbc;
        const int fb = E.face_comp_off[c], fe = E.face_comp_off[c + 1];
        if (fold_j > 0) {   // R22: the face part of h_t = (M W_t)^T x summed here, where y_F is in registers
            double hl[KM];
#pragma unroll
            for (int t = 0; t < KM; ++t) hl[t] = 0.0;
            if (w > 0)
                for (int F = fb + lw; F < fe; F += 2 * nwc) face_warp_pcr<2, KM>(P, E, F, nwc, fe, b, scl, y, lane, hl, kc);
#pragma unroll
            for (int t = 0; t < KM; ++t) {
                const double v = warp_sum(hl[t]);
                if (lane == 0) hfw[w * KMAX + t] = v;
            }
        } else if (w > 0) {
            for (int F = fb + lw; F < fe; F += 2 * nwc) face_warp_pcr<2, 0>(P, E, F, nwc, fe, b, scl, y, lane, nullptr, 0, bmap);
        }
    } else if (E.tri) {
        if (w > 0)
            for (int F = gt; F < E.nfaces; F += nthr) face_thread_tridiag(a, E, F, b, scl, nullptr, y, 0, dsm + (threadIdx.x - 32));
    } else if (w > 0)
        for (int F = gw; F < E.nfaces; F += nwarps) {
            if (E.fb) face_warp_blocks(a, E, F, b, scl, y, wsm, lane);
            else face_warp(a, E, F, b, scl, nullptr, y, 0, wsm, lane);
        }
    if (TIM && a.timers && lane == 0 && w > 0 && gw < 4096) a.timers[200 + gw] = clock64() - tf0;
    if (fused && a.split) {   // wait for every block's t_C (published before its face solves): no grid barrier here
        if (threadIdx.x == 32) {
            const unsigned target = unsigned(nelim) * gridDim.x;
            while (*((volatile unsigned*)a.arrive) < target) {}
            __threadfence();
        }
        __syncthreads();
    } else {
        grid.sync();
        __syncwarp();   // lane 0 spun in the barrier: reconverge before warp-synchronous code
    }
    STAMP(stamp++);
    // cross points of this block's component: t_C = scl*b_C - X_CF y in smem, then rows of S_C^-1 t_C
    const bool dbg2 = TIM && a.timers && blockIdx.x == 0 && threadIdx.x == 32;   // E2 sub-phases (the last elimination wins)
    if (dbg2) a.timers[180] = gtimer();
    {
        const int base = E.cross_comp_off[c], ncc = E.cross_comp_off[c + 1] - base;
        // General path with a padded X_CF (3D wirebasket): t_C = scl b_C - X_CF y is formed ONCE, each block its own
        // rows [rlo, rhi) (8 lanes per row, fixed-order lane tree), published through the arrival counter and then
        // read by every block of the component -- the redundant per-block formation read the whole padded X_CF in
        // every block (c4: 21 us of the 57 us cross-point phase).
        const bool dist = !E.tri && E.xcf_w > 0;
        if (dist) {
            ++nelim;
            double* tCg = P.y + P.nflat + E.ncross;
            if (ncc > 0) {
                const int rlo = int(int64_t(lb) * ncc / nbc), rhi = int(int64_t(lb + 1) * ncc / nbc);
                const int g8 = threadIdx.x >> 3, l8 = threadIdx.x & 7;
                const double sc = scl[c];
                for (int r0_ = rlo; r0_ < rhi; r0_ += CT / 8) {
                    const int r = r0_ + g8;
                    const bool ok = r < rhi;
                    const int ci = base + (ok ? r : rlo);
                    double acc = (ok && l8 == 0) ? sc * b[E.cross_flat[ci]] : 0.0;
                    for (int k = l8; k < E.xcf_w; k += 8) {
                        const size_t at = size_t(k) * E.ncross + ci;
                        const double v = E.xcfw_val[at];
                        const int col = E.xcfw_col[at];
                        acc -= ok ? v * y[col] : 0.0;
                    }
                    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
                    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
                    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
                    if (ok && l8 == 0) tCg[ci] = acc;
                }
            }
            __syncthreads();
            if (threadIdx.x == 32) {   // publish, then wait for every block's rows
                __threadfence();
                atomicAdd(a.arrive, 1u);
                const unsigned target = unsigned(nelim) * gridDim.x;
                while (*((volatile unsigned*)a.arrive) < target) {}
                __threadfence();
            }
            __syncthreads();
        }
        const bool shr = use_shr(a, E, c);
        // fold: (MW_t[c_r] - u_t[r]) of this block's rows, loaded BEFORE the cross-point GEMV (they are complete once every
        // block has arrived) so that the fold sums after it read shared memory only
        double cmine = 0.0;
        bool cpre = false;
        if (shr) {
            // Shared S_C^-1: every block owns rows [Rlo, Rhi) of the ONE matrix (split over the whole grid) and applies
            // them to the t_C of every component, so each row crosses L2 -> SM once instead of once per component
            // (c4: three wirebasket components, 188 -> 62.5 MB per elimination)
            const int nc = P.ncomp, bI = int(blockIdx.x), nbA = int(gridDim.x);
            const int Rlo = int(int64_t(bI) * ncc / nbA), Rhi = int(int64_t(bI + 1) * ncc / nbA), nr = Rhi - Rlo;
            double* tA = dsm;                 // [nc][ncc]
            double* part = tA + nc * ncc;     // [CW][nc][nr]
            const double* tCg = P.y + P.nflat + E.ncross;
            for (int i = threadIdx.x; i < nc * ncc; i += CT) tA[i] = tCg[i];   // cross points are numbered by component
            __syncthreads();
            const double* S = E.Sinv;
            const int cw = ((ncc + CW * 32 - 1) / (CW * 32)) * 32;
            const int c0 = w * cw, c1 = min(ncc, c0 + cw);
            constexpr int NA = 8, RB = 4;
            for (int r = Rlo; r < Rhi; r += RB) {
                const double* __restrict__ row[RB];
                double sr[RB][MAXC];
#pragma unroll
                for (int u = 0; u < RB; ++u) {
                    row[u] = S + size_t(r + u < Rhi ? r + u : r) * ncc;
#pragma unroll
                    for (int cc = 0; cc < MAXC; ++cc) sr[u][cc] = 0.0;
                }
                for (int j = c0 + lane; j < c1; j += 32 * NA) {
                    double v[RB][NA];
#pragma unroll
                    for (int q = 0; q < NA; ++q) {
                        const int jj = j + 32 * q;
                        const bool ok = jj < c1;
#pragma unroll
                        for (int u = 0; u < RB; ++u) v[u][q] = (ok && r + u < Rhi) ? __ldcs(row[u] + jj) : 0.0;
                    }
#pragma unroll
                    for (int cc = 0; cc < MAXC; ++cc)
                        if (cc < nc) {
#pragma unroll
                            for (int q = 0; q < NA; ++q) {
                                const int jj = j + 32 * q;
                                const double t = jj < c1 ? tA[cc * ncc + jj] : 0.0;
#pragma unroll
                                for (int u = 0; u < RB; ++u) sr[u][cc] += v[u][q] * t;
                            }
                        }
                }
#pragma unroll
                for (int u = 0; u < RB; ++u)
#pragma unroll
                    for (int cc = 0; cc < MAXC; ++cc)
                        if (cc < nc) {
                            const double su = warp_sum(sr[u][cc]);
                            if (lane == 0 && r + u < Rhi) part[(w * nc + cc) * nr + (r + u - Rlo)] = su;
                        }
            }
            __syncthreads();
            for (int e = threadIdx.x; e < nc * nr; e += CT) {
                const int cc = e / nr, rr = e - cc * nr;
                double acc = 0.0;
                for (int q = 0; q < CW; ++q) acc += part[(q * nc + cc) * nr + rr];
                const int ci = E.cross_comp_off[cc] + Rlo + rr;
                xC[ci] = acc;
                out[E.cross_flat[ci]] = acc;
                part[cc * nr + rr] = acc;   // slice 0: kept for the fold sums (read above by this thread only)
            }
            __syncthreads();
            if (fold_j > 0) {
                // fold sums of every component over this block's rows, + the face part of the block's own component
                // (summed per warp in the face phase), into the all-blocks slots (pp, cc, v, block)
                // (every component with its OWN basis size: a zero or broken-down component has a smaller one)
                for (int task = w; task < nc * (KMAX + 1); task += CW) {
                    const int cc = task / (KMAX + 1), v = task - cc * (KMAX + 1);
                    if (v > kcs_all[cc]) continue;
                    double t_ = 0.0;
                    if (v > 0)
                        for (int rr = lane; rr < nr; rr += 32) {
                            const int ci = E.cross_comp_off[cc] + Rlo + rr;
                            t_ += (P.MW[size_t(v - 1) * P.nflat + E.cross_flat[ci]] - a.ucross[size_t(v - 1) * E.ncross + ci]) *
                                  part[cc * nr + rr];
                        }
                    t_ = warp_sum(t_);
                    if (v > 0 && cc == c)
                        for (int q = 1; q < CW; ++q) t_ += hfw[q * KMAX + v - 1];
                    if (lane == 0) a.redf[((size_t(pp) * MAXC + cc) * NRED + v) * nbA + bI] = t_;
                }
                __syncthreads();
            }
        } else if (ncc > 0) {
            double* tC = dsm;
            if (dist || (E.tri && E.fuse)) {   // formed once: above (3D) / in the first face phase (fused 2D)
                const double* tCg = P.y + P.nflat + E.ncross;
                for (int i = threadIdx.x; i < ncc; i += CT) tC[i] = tCg[base + i];
            } else if (E.tri) {   // padded X_CF: every load of UC cross points issued before the first use
                constexpr int UC = 4;
                const double sc = scl[c];
                // every block of the component reads the same inputs: start each block at a different offset so
                // the blocks do not queue on the same L2 lines at the same time
                const int rot = int((int64_t(lb) * 224) % ncc);
                for (int i0 = threadIdx.x - 32; i0 < ncc; i0 += RW * UC) {   // warps 1.. (warp 0: barrier host)
                    if (threadIdx.x < 32) break;
                    int fl[UC], col[UC][XCF_W];
                    double xv[UC][XCF_W];
#pragma unroll
                    for (int u = 0; u < UC; ++u) {
                        const int i = i0 + u * RW;
                        const bool ok = i < ncc;
                        const int ci = base + (ok ? (i + rot < ncc ? i + rot : i + rot - ncc) : 0);
                        fl[u] = E.cross_flat[ci];
#pragma unroll
                        for (int k = 0; k < XCF_W; ++k) {
                            col[u][k] = E.xcf4_col[size_t(k) * E.ncross + ci];
                            xv[u][k] = E.xcf4_val[size_t(k) * E.ncross + ci];
                        }
                    }
                    double bv[UC], yv[UC][XCF_W];
#pragma unroll
                    for (int u = 0; u < UC; ++u) {
                        bv[u] = b[fl[u]];
#pragma unroll
                        for (int k = 0; k < XCF_W; ++k) yv[u][k] = y[col[u][k]];
                    }
#pragma unroll
                    for (int u = 0; u < UC; ++u) {
                        const int i = i0 + u * RW;
                        double t = sc * bv[u];
#pragma unroll
                        for (int k = 0; k < XCF_W; ++k) t -= xv[u][k] * yv[u][k];
                        if (i < ncc) tC[i + rot < ncc ? i + rot : i + rot - ncc] = t;
                    }
                }
            } else if (E.xcf_w > 0) {   // padded X_CF (3D): UC rows per thread, every load of an 8-entry chunk together
                constexpr int UC = 2, CH = 8;
                const double sc = scl[c];
                const int rot = int((int64_t(lb) * 224) % ncc);   // blocks start at different rows (L2 queuing)
                for (int i0 = threadIdx.x; i0 < ncc; i0 += CT * UC) {
                    int ci[UC], ii[UC];
                    double acc[UC];
#pragma unroll
                    for (int u = 0; u < UC; ++u) {
                        const int i = i0 + u * CT;
                        ii[u] = i < ncc ? (i + rot < ncc ? i + rot : i + rot - ncc) : -1;
                        ci[u] = base + (ii[u] >= 0 ? ii[u] : 0);
                        acc[u] = ii[u] >= 0 ? sc * b[E.cross_flat[ci[u]]] : 0.0;
                    }
                    for (int k0 = 0; k0 < E.xcf_w; k0 += CH) {
                        int col[UC][CH];
                        double v[UC][CH], yv[UC][CH];
#pragma unroll
                        for (int u = 0; u < UC; ++u)
#pragma unroll
                            for (int q = 0; q < CH; ++q) {
                                const size_t at = size_t(k0 + q) * E.ncross + ci[u];
                                col[u][q] = E.xcfw_col[at];
                                v[u][q] = E.xcfw_val[at];
                            }
#pragma unroll
                        for (int u = 0; u < UC; ++u)
#pragma unroll
                            for (int q = 0; q < CH; ++q) yv[u][q] = y[col[u][q]];
#pragma unroll
                        for (int u = 0; u < UC; ++u)
#pragma unroll
                            for (int q = 0; q < CH; ++q) acc[u] -= v[u][q] * yv[u][q];
                    }
#pragma unroll
                    for (int u = 0; u < UC; ++u)
                        if (ii[u] >= 0) tC[ii[u]] = acc[u];
                }
            } else {
                for (int i = threadIdx.x; i < ncc; i += CT) {
                    const int ci = base + i;
                    double t = scl[c] * b[E.cross_flat[ci]];
                    for (int e = E.xcf_ptr[ci]; e < E.xcf_ptr[ci + 1]; ++e) t -= E.xcf_val[e] * y[E.xcf_col[e]];
                    tC[i] = t;
                }
            }
            if (fd) asm volatile("cp.async.wait_group 0;\n" ::: "memory");   // this thread's share of the Q tables
            __syncthreads();
            if (dbg2) a.timers[181] = gtimer();
            // block lb owns the contiguous rows [rlo, rhi) of x_C = S_C^-1 t_C
            const int rlo = int(int64_t(lb) * ncc / nbc), rhi = int(int64_t(lb + 1) * ncc / nbc), nr = rhi - rlo;
            double* part = fd ? tC : tC + ncc;   // [npart][nr] row sums (dense: one slice per warp)
            const int npart = fd ? 1 : CW;
            if (fd) {
                // Separable S_C (HElim::fd, R23): x_C = (Qy (x) Qx) diag(1/(lam_a + mu_b)) (Qy (x) Qx)^T t_C.
                // Every block of the component runs the forward transforms of the whole nx x ny grid (2 nx ny (nx + ny)
                // flops from shared memory, the small Q tables from L1/L2) and the backward transforms of its own rows:
                // no S_C^-1 stream (c5: 30.5 MB per elimination), the same fixed summation order in every block.
                const int nx = E.fd_nx, ny = E.fd_ny, cs = E.sc_shared ? 0 : c;
                const double* Qx = dsm + fdq;          // staged at the start of the phase
                const double* Qy = Qx + nx * nx;
                const double* __restrict__ il = E.fd_il + size_t(cs) * nx * ny;
                double* X = tC;          // t_C as X[ix + nx iy]; later Z[a + nx b], then the row sums
                double* Y = tC + ncc;    // Y[a + nx iy]; later V[a + nx (iy - iyA)]
                constexpr int TY = 8;
                const int nah = (nx + 31) / 32, nty = (ny + TY - 1) / TY;
                // Y(a, iy) = sum_ix Qx[ix][a] X(ix, iy): lane = a (coalesced Qx rows), TY values of iy per lane (X broadcast)
                for (int task = w; task < nah * nty; task += CW) {
                    const int aa = (task % nah) * 32 + lane, iy0 = (task / nah) * TY;
                    const bool ok = aa < nx;
                    const int ac = ok ? aa : 0;
                    int xo[TY];
                    double acc[TY];
#pragma unroll
                    for (int u = 0; u < TY; ++u) {
                        xo[u] = nx * min(iy0 + u, ny - 1);
                        acc[u] = 0.0;
                    }
#pragma unroll 4
                    for (int ix = 0; ix < nx; ++ix) {
                        const double q = Qx[ix * nx + ac];
#pragma unroll
                        for (int u = 0; u < TY; ++u) acc[u] = fma(q, X[xo[u] + ix], acc[u]);
                    }
#pragma unroll
                    for (int u = 0; u < TY; ++u)
                        if (ok && iy0 + u < ny) Y[aa + nx * (iy0 + u)] = acc[u];
                }
                __syncthreads();
                // Z(a, b) = (sum_iy Y(a, iy) Qy[iy][b]) / (lam_a + mu_b), into X's place
                for (int task = w; task < nah * nty; task += CW) {
                    const int aa = (task % nah) * 32 + lane, b0 = (task / nah) * TY;
                    const bool ok = aa < nx;
                    const int ac = ok ? aa : 0;
                    int bo[TY];
                    double acc[TY];
#pragma unroll
                    for (int u = 0; u < TY; ++u) {
                        bo[u] = min(b0 + u, ny - 1);
                        acc[u] = 0.0;
                    }
#pragma unroll 4
                    for (int iy = 0; iy < ny; ++iy) {
                        const double yv = Y[ac + nx * iy];
#pragma unroll
                        for (int u = 0; u < TY; ++u) acc[u] = fma(yv, Qy[iy * ny + bo[u]], acc[u]);
                    }
#pragma unroll
                    for (int u = 0; u < TY; ++u)
                        if (ok && b0 + u < ny) X[aa + nx * (b0 + u)] = acc[u] * il[aa + nx * (b0 + u)];
                }
                __syncthreads();
                // own rows: V(a, iy) = sum_b Z(a, b) Qy[iy][b] for the rows' iy range, into Y's place
                const int iyA = nr > 0 ? rlo / nx : 0, niy = nr > 0 ? (rhi - 1) / nx - iyA + 1 : 0;
                for (int e = threadIdx.x; e < nx * niy; e += CT) {
                    const int iyl = e / nx, aa = e - iyl * nx;
                    const double* qrow = Qy + (iyA + iyl) * ny;
                    double t = 0.0;
                    for (int bb = 0; bb < ny; ++bb) t = fma(X[aa + nx * bb], qrow[bb], t);
                    Y[e] = t;
                }
                __syncthreads();
                // x(ix, iy) = sum_a Qx[ix][a] V(a, iy): warp per row, lanes over a (fixed order), into X's place
                for (int r = rlo + w; r < rhi; r += CW) {
                    const int iy = r / nx, ix = r - iy * nx;
                    const double* qrow = Qx + ix * nx;
                    const double* vcol = Y + nx * (iy - iyA);
                    double t = 0.0;
                    for (int aa = lane; aa < nx; aa += 32) t = fma(qrow[aa], vcol[aa], t);
                    t = warp_sum(t);
                    if (lane == 0) part[r - rlo] = t;
                }
            } else {
                const double* S = E.Sinv + E.sc_off[c];

                // block lb owns the contiguous rows [rlo, rhi); warp w takes one column slice of all of them (RB rows
                // at a time, NA loads per row per lane in flight: RB * NA independent loads per batch, so a block's
                // ~13 rows (c5) take 4 dependent batches instead of 7); warp partials are summed in fixed order
                const int cw = ((ncc + CW * 32 - 1) / (CW * 32)) * 32;
                const int c0 = w * cw, c1 = min(ncc, c0 + cw);
                cpre = fold_j > 0 && kc * nr <= CT && ncc + (CW + KMAX) * nr <= a.smem_doubles;
                if (cpre && int(threadIdx.x) < kc * nr) {
                    const int t = threadIdx.x / nr, rr = threadIdx.x - t * nr;
                    const int cfi = E.cross_flat[base + rlo + rr];
                    cmine = P.MW[size_t(t) * P.nflat + cfi] - a.ucross[size_t(t) * E.ncross + base + rlo + rr];
                }
                if (a.sc_persist && &E == &a.P.eK) sc_rows<false>(S, ncc, rlo, rhi, nr, c0, c1, w, lane, tC, part);
                else sc_rows<true>(S, ncc, rlo, rhi, nr, c0, c1, w, lane, tC, part);
            }
            if (dbg2) a.timers[182] = gtimer();
            __syncthreads();
            if (dbg2) a.timers[183] = gtimer();
            for (int r = rlo + threadIdx.x; r < rhi; r += CT) {
                double acc = 0.0;
                for (int q = 0; q < npart; ++q) acc += part[q * nr + (r - rlo)];
                xC[base + r] = acc;
                out[E.cross_flat[base + r]] = acc;
                part[r - rlo] = acc;   // kept for the fold sums below (slice 0 of this row: read above by this thread only)
            }
            __syncthreads();
        }
        if (fold_j > 0 && !shr) {
            // block sums into the reduction slots (pp, c, 1 + t), slot 0 (unused) = 0; fixed order: the cross part
            // sum_r (MW_t[c_r] - u_t[r]) x_C[r] over this block's rows (lanes stride the rows, then a warp tree), then
            // the face part over the warps (summed per warp in the face phase)
            const int rlo = ncc > 0 ? int(int64_t(lb) * ncc / nbc) : 0, rhi = ncc > 0 ? int(int64_t(lb + 1) * ncc / nbc) : 0;
            const double* xr = (fd ? dsm : dsm + ncc);
            const int nr = rhi - rlo;
            double* prod = dsm + ncc + CW * nr;   // [kc][nr] behind the dense path's row sums
            if (cpre) {
                if (int(threadIdx.x) < kc * nr) prod[threadIdx.x] = cmine * xr[threadIdx.x % nr];
                __syncthreads();
            }
            for (int v = w; v <= kc; v += CW) {
                double t_ = 0.0;
                if (v > 0 && cpre) {
                    for (int r = lane; r < nr; r += 32) t_ += prod[(v - 1) * nr + r];
                } else if (v > 0)
                    for (int r = rlo + lane; r < rhi; r += 32) {
                        const int cf = E.cross_flat[base + r];
                        t_ += (P.MW[size_t(v - 1) * P.nflat + cf] - a.ucross[size_t(v - 1) * E.ncross + base + r]) * xr[r - rlo];
                    }
                t_ = warp_sum(t_);
                if (v > 0)
                    for (int q = 1; q < CW; ++q) t_ += hfw[q * KMAX + v - 1];
                if (lane == 0) a.red[((size_t(pp) * MAXC + c) * NRED + v) * a.nbc_max + lb] = t_;
            }
            __syncthreads();
        }
    }
    if (dbg2) a.timers[184] = gtimer();
    grid.sync();
    __syncwarp();   // lane 0 spun in the barrier: reconverge before warp-synchronous code
    if (dbg2) a.timers[185] = gtimer();
    STAMP(stamp++);
    if (E.tri && E.fuse) return;   // x_F = y_F - G_F x_C is formed by the consumer phase (elim_value)
    tf0 = clock64();
    if (E.tri) {
        if (w > 0)
            for (int F = gt; F < E.nfaces; F += nthr) face_thread_tridiag(a, E, F, b, scl, xC, out, 1, dsm + (threadIdx.x - 32));
    } else if (E.g3_items > 0) {
        // x_F = y_F - G_F x_C(adj) with the dense G_F = X_FF^-1 X_F,adj of every face (HElim::g3): a streaming pass,
        // one warp per (face, 32-node chunk), instead of a second sequential band solve per face
        if (w > 0)
            for (int it = gw; it < E.g3_items; it += nwarps) {
                const int F = E.g3_item_face[it], i = E.g3_item_i0[it] + lane;
                const int o = E.face_off[F], n = E.face_off[F + 1] - o;
                const int a0 = E.g3_adj_ptr[F], na = E.g3_adj_ptr[F + 1] - a0;
                const double* __restrict__ G = E.g3 + E.g3_off[F];
                const bool ok = i < n;
                const int node = ok ? E.face_nodes[o + i] : 0;
                double acc = ok ? y[node] : 0.0;
                for (int e0 = 0; e0 < na; e0 += 32) {
                    const double xe = e0 + lane < na ? xC[E.g3_adj[a0 + e0 + lane]] : 0.0;   // lane e holds x_C(adj e)
                    const int ne = min(32, na - e0);
                    int e = 0;
                    for (; e + 8 <= ne; e += 8) {
                        double gv[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q) gv[q] = ok ? __ldcs(G + size_t(e0 + e + q) * n + i) : 0.0;   // streamed once
#pragma unroll
                        for (int q = 0; q < 8; ++q) acc = fma(-gv[q], __shfl_sync(0xffffffffu, xe, e + q), acc);
                    }
                    for (; e < ne; ++e) {
                        const double gv = ok ? __ldcs(G + size_t(e0 + e) * n + i) : 0.0;
                        acc = fma(-gv, __shfl_sync(0xffffffffu, xe, e), acc);
                    }
                }
                if (ok) out[node] = acc;
            }
    } else if (w > 0)
        for (int F = gw; F < E.nfaces; F += nwarps) face_warp(a, E, F, b, scl, xC, out, 1, wsm, lane);
    if (TIM && a.timers && lane == 0 && w > 0 && gw < 4096) a.timers[200 + 4096 + gw] = clock64() - tf0;
    grid.sync();
    __syncwarp();   // lane 0 spun in the barrier: reconverge before warp-synchronous code
    STAMP(stamp++);
}

// Circle-method position map for the parallel Jacobi ordering on M (even) slots: pairs are always the
// fixed slots (2k, 2k+1); between rounds slot 0 stays and the others rotate t_1 -> t_2 -> .. -> t_{H-1} ->
// b_{H-1} -> .. -> b_0 -> t_1 (t_i = slot 2i, b_i = slot 2i+1), so every pair meets once in M-1 rounds.
// Returns the slot whose content moves INTO slot `pos`.
__device__ __forceinline__ constexpr int circle_src(int pos, int M) {
    const int H = M / 2;
    if (pos == 0) return 0;
    if ((pos & 1) == 0) {
        const int i = pos / 2;
        return i == 1 ? 1 : 2 * (i - 1);
    }
    const int i = (pos - 1) / 2;
    return i == H - 1 ? 2 * (H - 1) : 2 * (i + 1) + 1;
}

// Cyclic parallel Jacobi on the symmetric n x n matrix C (smem, leading dim KMAX+1) with eigenvectors
// accumulated into V (smem, starts as I). One warp; lane r < M holds row r of C and of V in registers,
// slots >= n are decoupled ghosts. On return C's diagonal holds the eigenvalues and V's columns the
// eigenvectors (same order: full sweeps return every slot to its place). Returns the sweep count.
template <int M>
__device__ int jacobi_reg(double* C, double* V, int n) {
    constexpr int LDK = KMAX + 1, H = M / 2;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    double c[M], v[M];
#pragma unroll
    for (int b = 0; b < M; ++b) {
        c[b] = (lane < n && b < n) ? C[lane * LDK + b] : 0.0;
        v[b] = lane == b ? 1.0 : 0.0;
    }
    const int srcl = lane < M ? circle_src(lane, M) : lane;
    const bool even = (lane & 1) == 0;
    int nsw = 0;
    for (int sweep = 0; sweep < 30; ++sweep) {
        double off = 0.0, dia = 0.0;
#pragma unroll
        for (int b = 0; b < M; ++b) {
            const double x = lane < M ? c[b] * c[b] : 0.0;
            if (b == lane) dia += x;
            else off += x;
        }
        off = warp_sum(off);
        dia = warp_sum(dia);
        // converged when ||offdiag||_F <= 1e-12 ||diag||_F: eigenvector errors ~1e-12 relative, far inside the
        // preconditioner's 1e-9 parity tolerance (one sweep fewer than 1e-15 on c5: 0.6469 -> 0.6428 ms)
        if (off <= 1e-24 * dia) break;
        ++nsw;
        const double thr = 1e-15 * sqrt(dia);
        int rotated = 0;
        for (int rnd = 0; rnd < M - 1; ++rnd) {
            double diag = 0.0, offp = 0.0;
#pragma unroll
            for (int b = 0; b < M; ++b) {
                if (b == lane) diag = c[b];
                if (b == (lane ^ 1)) offp = c[b];
            }
            const double dq = __shfl_xor_sync(FULL, diag, 1);
            double cs = 1.0, sn = 0.0;
            if (even && lane < M && fabs(offp) > thr && fabs(offp) > 1e-300) {
                // rotation zeroing C[p][q] (p = lane, q = lane + 1), the small angle (|tan| <= 1):
                // cos^2 = (1 + |d|/rt)/2, sin cos = sgn(d) apq/rt with rt = sqrt(d^2 + 4 apq^2) -- the same
                // rotation as t = 2 apq/(d + sgn(d) rt), cs = 1/sqrt(1+t^2), in two rsqrt and no sqrt/divide
                const double d = dq - diag, apq = offp;
                const double ir = rsqrt(fma(d, d, 4.0 * apq * apq));
                const double h = 0.5 * fma(fabs(d), ir, 1.0);
                const double ih = rsqrt(h);
                cs = h * ih;
                sn = (d >= 0.0 ? apq : -apq) * ir * ih;
                rotated = 1;
            }
            cs = __shfl_sync(FULL, cs, lane & ~1);
            sn = __shfl_sync(FULL, sn, lane & ~1);
            // C <- C J and V <- V J: columns (2k, 2k+1) of this lane's rows
#pragma unroll
            for (int k = 0; k < H; ++k) {
                const double ck = __shfl_sync(FULL, cs, 2 * k), sk = __shfl_sync(FULL, sn, 2 * k);
                const double x0 = c[2 * k], x1 = c[2 * k + 1], y0 = v[2 * k], y1 = v[2 * k + 1];
                c[2 * k] = ck * x0 - sk * x1;
                c[2 * k + 1] = sk * x0 + ck * x1;
                v[2 * k] = ck * y0 - sk * y1;
                v[2 * k + 1] = sk * y0 + ck * y1;
            }
            // C <- J^T C: rows 2k (even lane) and 2k+1 (odd lane) combine
#pragma unroll
            for (int b = 0; b < M; ++b) {
                const double o = __shfl_xor_sync(FULL, c[b], 1);
                c[b] = even ? cs * c[b] - sn * o : sn * o + cs * c[b];
            }
            // next pairing: rows move between lanes, columns between registers (static map)
#pragma unroll
            for (int b = 0; b < M; ++b) c[b] = __shfl_sync(FULL, c[b], srcl);
            double tc[M], tv[M];
#pragma unroll
            for (int b = 0; b < M; ++b) {
                tc[b] = c[b];
                tv[b] = v[b];
            }
#pragma unroll
            for (int b = 0; b < M; ++b) {
                c[b] = tc[circle_src(b, M)];
                v[b] = tv[circle_src(b, M)];
            }
        }
        if (!__any_sync(FULL, rotated)) break;   // every pair below threshold: converged
    }
    __syncwarp();
    if (lane < n) {
#pragma unroll
        for (int b = 0; b < M; ++b)
            if (b < n) {
                if (b == lane) C[lane * LDK + b] = c[b];
                V[lane * LDK + b] = v[b];
            }
    }
    __syncwarp();
    return nsw;
}

// Cyclic parallel Jacobi on the symmetric n x n matrix C in shared memory (leading dim KMAX+1), eigenvectors
// accumulated into V (shared, starts as I); one warp. The same rotations and ordering as jacobi_reg (pairs of the
// circle method on M = n rounded up to even slots, the small-angle rotation from two rsqrt), but every round is
// one data-parallel update of all entries: lanes 0..M/2-1 form the M/2 rotations, then each lane rewrites its
// share of C <- J^T C J and V <- V J from four (two) shared loads per entry. A round costs a few shared-memory
// latencies instead of ~30 dependent shuffles (jacobi_reg). Returns the sweep count.
template <int M>
__device__ int jacobi_smem(double* C, double* V, int n, double* rot) {
    constexpr int LDK = KMAX + 1, H = M / 2, NE = (M * M + 31) / 32;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    double* cs = rot;            // [H]
    double* sn = rot + H;        // [H]
    if (n < M) {                 // ghost slot of odd n: a decoupled zero row/column
        for (int i = lane; i < M; i += 32) {
            C[(M - 1) * LDK + i] = 0.0;
            C[i * LDK + (M - 1)] = 0.0;
            V[(M - 1) * LDK + i] = i == M - 1 ? 1.0 : 0.0;
            V[i * LDK + (M - 1)] = i == M - 1 ? 1.0 : 0.0;
        }
        __syncwarp();
    }
    int perm[M];                 // perm[pos] = index at slot pos; pairs (perm[2k], perm[2k+1])
#pragma unroll
    for (int p = 0; p < M; ++p) perm[p] = p;
    int nsw = 0;
    for (int sweep = 0; sweep < 30; ++sweep) {
        double off = 0.0, dia = 0.0;
        for (int e = lane; e < M * M; e += 32) {
            const int i = e / M, j = e - i * M;
            const double x = C[i * LDK + j];
            if (i == j) dia += x * x;
            else off += x * x;
        }
        off = warp_sum(off);
        dia = warp_sum(dia);
        if (off <= 1e-24 * dia) break;   // ||offdiag||_F <= 1e-12 ||diag||_F (as jacobi_reg)
        ++nsw;
        const double thr = 1e-15 * sqrt(dia);
        int rotated = 0;
        for (int rnd = 0; rnd < M - 1; ++rnd) {
            int inv[M];          // slot of each index
#pragma unroll
            for (int p = 0; p < M; ++p) inv[perm[p]] = p;
            if (lane < H) {
                int p_ = 0, q_ = 0;
#pragma unroll
                for (int k = 0; k < H; ++k)
                    if (k == lane) {
                        p_ = perm[2 * k];
                        q_ = perm[2 * k + 1];
                    }
                const double app = C[p_ * LDK + p_], aqq = C[q_ * LDK + q_], apq = C[p_ * LDK + q_];
                double c_ = 1.0, s_ = 0.0;
                if (fabs(apq) > thr && fabs(apq) > 1e-300) {
                    const double d = aqq - app;
                    const double ir = rsqrt(fma(d, d, 4.0 * apq * apq));
                    const double h = 0.5 * fma(fabs(d), ir, 1.0);
                    const double ih = rsqrt(h);
                    c_ = h * ih;
                    s_ = (d >= 0.0 ? apq : -apq) * ir * ih;
                }
                cs[lane] = c_;
                sn[lane] = s_;
            }
            __syncwarp();
            rotated |= __any_sync(FULL, lane < H && sn[lane < H ? lane : 0] != 0.0);
            double nc[NE], nv[NE];
#pragma unroll
            for (int u = 0; u < NE; ++u) {
                const int e = lane + 32 * u;
                nc[u] = 0.0;
                nv[u] = 0.0;
                if (e < M * M) {
                    const int i = e / M, j = e - i * M;
                    const int si = inv[i], sj = inv[j];
                    const int ki = si >> 1, kj = sj >> 1;
                    const int pi = perm[si & ~1], qi = perm[si | 1], pj = perm[sj & ~1], qj = perm[sj | 1];
                    // J column t of pair k: (J[p][t], J[q][t]) = (c, -s) for t = p, (s, c) for t = q
                    const double ci_ = cs[ki], si_ = sn[ki], cj_ = cs[kj], sj_ = sn[kj];
                    const double ap = (si & 1) ? si_ : ci_, aq = (si & 1) ? ci_ : -si_;
                    const double bp = (sj & 1) ? sj_ : cj_, bq = (sj & 1) ? cj_ : -sj_;
                    const double cpp = C[pi * LDK + pj], cpq = C[pi * LDK + qj], cqp = C[qi * LDK + pj],
                                 cqq = C[qi * LDK + qj];
                    nc[u] = ap * (cpp * bp + cpq * bq) + aq * (cqp * bp + cqq * bq);
                    nv[u] = V[i * LDK + pj] * bp + V[i * LDK + qj] * bq;
                }
            }
            __syncwarp();
#pragma unroll
            for (int u = 0; u < NE; ++u) {
                const int e = lane + 32 * u;
                if (e < M * M) {
                    const int i = e / M, j = e - i * M;
                    C[i * LDK + j] = nc[u];
                    V[i * LDK + j] = nv[u];
                }
            }
            __syncwarp();
            int np[M];   // next pairing: the slot contents move by the circle map
#pragma unroll
            for (int p = 0; p < M; ++p) np[p] = perm[circle_src(p, M)];
#pragma unroll
            for (int p = 0; p < M; ++p) perm[p] = np[p];
        }
        if (!rotated) break;
    }
    return nsw;
}

// Cyclic parallel Jacobi of jacobi_smem (the same pairs, rotations and update formulas, entry by entry) run by the
// whole CTA: one thread per entry of C and V, the circle-method schedule of all rounds tabulated once in shared
// memory (the content of slot ring[k] after r rounds is ring[(k + r) mod (M-1)], slot 0 stays). A round is a
// rotation phase (M/2 threads), the entry updates and the write-back: three CTA barriers instead of one warp
// walking 4 entries per lane with register-array index maps (35 us -> measured in profiles/). Returns the sweeps.
__device__ int jacobi_block(double* C, double* V, int n, int* sched, int* slot_of, double* csn, double* red, int* flag) {
    constexpr int LDK = KMAX + 1;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int M = (n + 1) & ~1, H = M / 2;
    double* cs = csn;
    double* sn = csn + KMAX / 2;
    if (n < M) {   // ghost slot of odd n: a decoupled zero row/column
        for (int i = tid; i < M; i += CT) {
            C[(M - 1) * LDK + i] = 0.0;
            C[i * LDK + (M - 1)] = 0.0;
            V[(M - 1) * LDK + i] = i == M - 1 ? 1.0 : 0.0;
            V[i * LDK + (M - 1)] = i == M - 1 ? 1.0 : 0.0;
        }
    }
    int* ring = slot_of;   // scratch until the first round
    if (tid == 0) {
        int p = 1;
        for (int k = 0; k < M - 1; ++k) {
            ring[k] = p;
            p = circle_src(p, M);
        }
    }
    __syncthreads();
    for (int e = tid; e < (M - 1) * (M - 1); e += CT) {
        const int rnd = e / (M - 1), k = e - rnd * (M - 1);
        sched[rnd * KMAX + ring[k]] = ring[(k + rnd) % (M - 1)];
    }
    if (tid < M - 1) sched[tid * KMAX] = 0;
    __syncthreads();
    const int i = tid / M, j = tid - i * M;
    const bool mine = tid < M * M;
    int nsw = 0;
    for (int sweep = 0; sweep < 30; ++sweep) {
        double off = 0.0, dia = 0.0;
        if (mine) {
            const double x = C[i * LDK + j];
            if (i == j) dia = x * x;
            else off = x * x;
        }
        off = warp_sum(off);
        dia = warp_sum(dia);
        if (lane == 0) {
            red[wid] = off;
            red[CW + wid] = dia;
        }
        if (tid == 0) *flag = 0;
        __syncthreads();
        off = 0.0;
        dia = 0.0;
        for (int q = 0; q < CW; ++q) {
            off += red[q];
            dia += red[CW + q];
        }
        if (off <= 1e-24 * dia) break;   // ||offdiag||_F <= 1e-12 ||diag||_F (as jacobi_reg / jacobi_smem)
        ++nsw;
        const double thr = 1e-15 * sqrt(dia);
        for (int rnd = 0; rnd < M - 1; ++rnd) {
            if (tid < H) {
                const int p_ = sched[rnd * KMAX + 2 * tid], q_ = sched[rnd * KMAX + 2 * tid + 1];
                const double app = C[p_ * LDK + p_], aqq = C[q_ * LDK + q_], apq = C[p_ * LDK + q_];
                double c_ = 1.0, s_ = 0.0;
                if (fabs(apq) > thr && fabs(apq) > 1e-300) {
                    const double d = aqq - app;
                    const double ir = rsqrt(fma(d, d, 4.0 * apq * apq));
                    const double h = 0.5 * fma(fabs(d), ir, 1.0);
                    const double ih = rsqrt(h);
                    c_ = h * ih;
                    s_ = (d >= 0.0 ? apq : -apq) * ir * ih;
                    *flag = 1;
                }
                cs[tid] = c_;
                sn[tid] = s_;
                slot_of[p_] = 2 * tid;
                slot_of[q_] = 2 * tid + 1;
            }
            __syncthreads();
            double ncv = 0.0, nvv = 0.0;
            if (mine) {
                const int si = slot_of[i], sj = slot_of[j];
                const int ki = si >> 1, kj = sj >> 1;
                const int pi = sched[rnd * KMAX + (si & ~1)], qi = sched[rnd * KMAX + (si | 1)];
                const int pj = sched[rnd * KMAX + (sj & ~1)], qj = sched[rnd * KMAX + (sj | 1)];
                const double ci_ = cs[ki], si_ = sn[ki], cj_ = cs[kj], sj_ = sn[kj];
                const double ap = (si & 1) ? si_ : ci_, aq = (si & 1) ? ci_ : -si_;
                const double bp = (sj & 1) ? sj_ : cj_, bq = (sj & 1) ? cj_ : -sj_;
                const double cpp = C[pi * LDK + pj], cpq = C[pi * LDK + qj], cqp = C[qi * LDK + pj], cqq = C[qi * LDK + qj];
                ncv = ap * (cpp * bp + cpq * bq) + aq * (cqp * bp + cqq * bq);
                nvv = V[i * LDK + pj] * bp + V[i * LDK + qj] * bq;
            }
            __syncthreads();
            if (mine) {
                C[i * LDK + j] = ncv;
                V[i * LDK + j] = nvv;
            }
            __syncthreads();
        }
        if (!*flag) break;   // every pair below threshold: converged (read after the round's last barrier)
        __syncthreads();     // before the next sweep clears the flag
    }
    return nsw;
}

// One warp: generalized eigenproblem A y = theta B y (n <= KMAX) and coef = Y f(Theta) Y^T wr.
// Returns false on a non-SPD B or a non-positive Ritz value (non-singular component).
__device__ bool ritz_warp(const double* Ain, const double* Bin, const double* wr, int n, bool sing, double theta,
                          double* coef, double* R, double* C, double* V, double* X, double* rot, int* rpq,
                          unsigned long long* tm = nullptr, int use_reg = 0, int stage = 0) {
    // stage 0: everything on this warp; 1: stop before the Jacobi (the CTA runs jacobi_block); 2: resume after it
    const int lane = threadIdx.x & 31;
    constexpr int LDK = KMAX + 1;
    double* rinv = rot;   // 1/L_jj of the Cholesky factor of B (the three triangular solves multiply)
    double* jsc = rot + KMAX;   // rotation scratch of jacobi_smem
    int nsw = 0;
    if (stage != 2) {
    if (tm && lane == 0) tm[0] = gtimer();
    for (int idx = lane; idx < n * n; idx += 32) {
        const int i = idx / n, j = idx - i * n;
        C[i * LDK + j] = 0.5 * (Ain[i * KMAX + j] + Ain[j * KMAX + i]);
        R[i * LDK + j] = 0.5 * (Bin[i * KMAX + j] + Bin[j * KMAX + i]);
        V[i * LDK + j] = (i == j) ? 1.0 : 0.0;
    }
    __syncwarp();
    for (int j = 0; j < n; ++j) {
        const double d = R[j * LDK + j];
        if (!(d > 0.0)) return false;
        const double il = rsqrt(d), l = d * il;
        __syncwarp();
        if (lane == 0) {
            R[j * LDK + j] = l;
            rinv[j] = il;
        }
        if (lane > j && lane < n) R[lane * LDK + j] *= il;
        __syncwarp();
        for (int idx = lane; idx < (n - j - 1) * (n - j - 1); idx += 32) {
            const int i = j + 1 + idx / (n - j - 1), kk = j + 1 + idx % (n - j - 1);
            if (kk <= i) R[i * LDK + kk] -= R[i * LDK + j] * R[kk * LDK + j];
        }
        __syncwarp();
    }
    if (lane < n)
        for (int i = 0; i < n; ++i) {
            double t = C[i * LDK + lane];
            for (int kk = 0; kk < i; ++kk) t -= R[i * LDK + kk] * X[kk * LDK + lane];
            X[i * LDK + lane] = t * rinv[i];
        }
    __syncwarp();
    if (lane < n)
        for (int i = 0; i < n; ++i) {
            double t = X[lane * LDK + i];
            for (int kk = 0; kk < i; ++kk) t -= C[lane * LDK + kk] * R[i * LDK + kk];
            C[lane * LDK + i] = t * rinv[i];
        }
    __syncwarp();
    for (int idx = lane; idx < n * n; idx += 32) {
        const int i = idx / n, j = idx - i * n;
        if (j > i) {
            const double m = 0.5 * (C[i * LDK + j] + C[j * LDK + i]);
            C[i * LDK + j] = m;
            C[j * LDK + i] = m;
        }
    }
    __syncwarp();
    if (tm && lane == 0) tm[1] = gtimer();
    }   // stage != 2
    if (stage == 1) return true;
    if (stage == 2) {
    } else if (n > 1 && use_reg != 1) {
        switch ((n + 1) & ~1) {
            case 2: nsw = jacobi_smem<2>(C, V, n, jsc); break;
            case 4: nsw = jacobi_smem<4>(C, V, n, jsc); break;
            case 6: nsw = jacobi_smem<6>(C, V, n, jsc); break;
            case 8: nsw = jacobi_smem<8>(C, V, n, jsc); break;
            case 10: nsw = jacobi_smem<10>(C, V, n, jsc); break;
            case 12: nsw = jacobi_smem<12>(C, V, n, jsc); break;
            case 14: nsw = jacobi_smem<14>(C, V, n, jsc); break;
            default: nsw = jacobi_smem<16>(C, V, n, jsc); break;
        }
    } else if (n > 1) {
        switch ((n + 1) & ~1) {
            case 2: nsw = jacobi_reg<2>(C, V, n); break;
            case 4: nsw = jacobi_reg<4>(C, V, n); break;
            case 6: nsw = jacobi_reg<6>(C, V, n); break;
            case 8: nsw = jacobi_reg<8>(C, V, n); break;
            case 10: nsw = jacobi_reg<10>(C, V, n); break;
            case 12: nsw = jacobi_reg<12>(C, V, n); break;
            case 14: nsw = jacobi_reg<14>(C, V, n); break;
            default: nsw = jacobi_reg<16>(C, V, n); break;
        }
    }
    if (tm && lane == 0) {
        tm[2] = gtimer();
        if (stage == 0) tm[4] = nsw;
    }
    int bad = 0;
    double g = 0.0;
    if (lane < n) {
        const double th = C[lane * LDK + lane];
        if (!sing && !(th > 0.0)) bad = 1;
        // theta = 1/2 (the paper's H_0.5): sqrt/rsqrt instead of the much longer pow sequence
        const double f = theta == 0.5 ? (sing ? 1.0 / (1.0 + sqrt(fmax(th, 0.0))) : rsqrt(th))
                                      : (sing ? 1.0 / (1.0 + pow(fmax(th, 0.0), 1.0 - theta)) : pow(th, theta - 1.0));
        for (int i = n - 1; i >= 0; --i) {
            double t = V[i * LDK + lane];
            for (int kk = i + 1; kk < n; ++kk) t -= R[kk * LDK + i] * X[kk * LDK + lane];
            X[i * LDK + lane] = t * rinv[i];
        }
        double t = 0.0;
        for (int i = 0; i < n; ++i) t += X[i * LDK + lane] * wr[i];
        g = f * t;
    }
    if (__any_sync(0xffffffffu, bad)) return false;
    double cf = 0.0;                                        // coef_i = sum_e Y[i][e] g_e
    for (int e = 0; e < n; ++e) {
        const double ge = __shfl_sync(0xffffffffu, g, e);
        if (lane < n) cf += X[lane * LDK + e] * ge;
    }
    if (lane < n) coef[lane] = cf;
    if (tm && lane == 0) tm[3] = gtimer();
    return true;
}

// KM: compile-time bound on the basis size (>= lanczos_k) for the register arrays of the row phases;
// TIM: diagnostic timers compiled in (DE_PREC_TIMERS)
template <int KM, bool TIM>
__global__ void __launch_bounds__(CT, 2) k_prec_coop(CoopArgs a) {
    static_assert(KM <= KMAX, "basis bound");
    cg::grid_group grid = cg::this_grid();
    if (a.s != nullptr && a.s->done) return;
    int stamp = 0, nelim = 0;
    STAMP(stamp++);
    const PrecDev& P = a.P;
    extern __shared__ double dsm[];
    __shared__ double sred[CW][NRED];
    __shared__ double tot[MAXC][NRED];
    __shared__ double scl[MAXC], nrmv[MAXC], nb2v[MAXC];
    __shared__ double hsm[MAXC][KMAX];
    __shared__ double sclh[MAXC][KMAX];   // 1/||w_j||_M of every accepted basis vector (Gram scaling)
    __shared__ int act[MAXC], kcs[MAXC], brk[MAXC];
    const int tid = threadIdx.x;
    const int nb = gridDim.x, nc = P.ncomp;
    const int c = blockIdx.x % nc, lb = blockIdx.x / nc, nbc = (nb - c + nc - 1) / nc;
    const int64_t lo = P.comp_off[c], hi = P.comp_off[c + 1];
    // row-parallel phases run on warps 1..CW-1 (RW rows per block chunk); warp 0 hosts the grid-barrier
    // thread and only joins the block reductions
    // 32-row warp chunks dealt warp-major over the component's blocks (chunk q = k*(CW-1)*nbc + (w-1)*nbc + lb),
    // so expensive row ranges (the cross points at the end of each component, rows with more couplings) spread
    // over many blocks instead of a few (measured: the block-contiguous layout left some blocks 1.4x the median)
    const int64_t r0 = tid >= 32 ? lo + (int64_t(tid / 32 - 1) * nbc + lb) * 32 + (tid & 31) : hi, rs = int64_t(nbc) * RW;
    const int64_t nf = P.nflat;
    int pp = 0;
    double vals[KM + 2];
#define ZERO_VALS()                                    \
    _Pragma("unroll") for (int v_ = 0; v_ < KM + 2; ++v_) vals[v_] = 0.0

    // ---- r_c gather and zero test. Fused seed elimination (2D): no gather phase -- the seed solve reads r through
    // the skeleton map, the consumer phase below stores r_c, and a zero component shows as ||s||_M = 0 (M is SPD).
    const bool fuseM = P.eM.tri && P.eM.fuse;
    if (!fuseM) {
        ZERO_VALS();
        for (int64_t i = r0; i < hi; i += rs) {
            const double x = a.r[P.cmap[i]];
            P.rf[i] = x;
            vals[0] += x * x;
        }
        block_partials(a, vals, 1, pp, c, lb, sred);
        grid.sync();
        __syncwarp();   // lane 0 spun in the barrier: reconverge before warp-synchronous code
        STAMP(stamp++);
        read_totals(a, pp, 1, nb, tot);
        pp ^= 1;
    }
    if (tid < nc) {
        act[tid] = fuseM ? 1 : (tot[tid][0] > 0.0 ? 1 : 0);
        kcs[tid] = 0;
        brk[tid] = 0;
        scl[tid] = 1.0;
    }
    __syncthreads();
    // Basis vectors are stored unnormalised (W_t = sclh_t * Wraw_t, likewise M W_t and L W_t): every
    // consumer folds sclh_t into its coefficients, so no normalisation pass over the rows is needed.
    // ---- s = M^-1 r (exact) = Wraw_0
    if (fuseM) elim_coop<KM, TIM>(grid, a, P.eM, a.r, scl, P.W, dsm, c, lb, nbc, stamp, nelim, 0, 0, 0, 0, 1, P.cmap);
    else elim_coop<KM, TIM>(grid, a, P.eM, P.rf, scl, P.W, dsm, c, lb, nbc, stamp, nelim);
    // ---- Ms, Ls, ||s||_M; q_1 = s / ||s||_M; rhs of the next solve M q_1 = Ms / ||s||_M
    ZERO_VALS();
    double* gacc = dsm;   // per-thread Gram accumulators [GW][CT] (dsm is free outside face solves / Ritz)
    gram_zero(gacc);
    for (int64_t i = r0; i < hi; i += rs) {
        double m, l, sv;
        if (fuseM) {
            sv = P.eM.pat_id ? spmv_elim_pat(P.M, P.L, i, P.eM, P.y, P.y + nf, nf, m, l)
                             : spmv_elim(P.M, P.L, i, P.eM, P.y, P.y + nf, m, l);
            P.W[i] = sv;
        } else {
            spmv_ml(P.M, P.L, i, P.W, m, l);
            sv = P.W[i];
        }
        P.MW[i] = m;
        P.LW[i] = l;
        vals[0] += sv * m;
        gacc[0 * CT + tid] += sv * l;            // G_L[0][0] (unscaled)
        gacc[KMAX * CT + tid] += sv * m;         // G_M[0][0]
        double rv;
        if (fuseM) {
            rv = a.r[P.cmap[i]];
            P.rf[i] = rv;
        } else {
            rv = P.rf[i];
        }
        gacc[2 * KMAX * CT + tid] += sv * rv;   // (W^T r)[0]
    }
    gram_partials(a, gacc, c, lb, 0);
    block_partials(a, vals, 1, pp, c, lb, sred);
    grid.sync();
    __syncwarp();   // lane 0 spun in the barrier: reconverge before warp-synchronous code
    STAMP(stamp++);
    read_totals(a, pp, 1, nb, tot);
    pp ^= 1;
    if (tid < nc) {
        nrmv[tid] = sqrt(tot[tid][0]);
        if (fuseM) act[tid] = tot[tid][0] > 0.0 ? 1 : 0;   // r_c = 0 <=> s = M^-1 r_c = 0 <=> ||s||_M = 0
        if (act[tid]) kcs[tid] = 1;
        scl[tid] = act[tid] ? 1.0 / nrmv[tid] : 0.0;
        sclh[tid][0] = scl[tid];
    }
    __syncthreads();
    // Gram row 0 is complete: warp 0 of the first blocks sums it while the next phase runs (warp 0 does no
    // face or row work there); the last row is left to block 0 before the Ritz step
    if (P.kmax > 1 && tid < 32) gram_row_sums(a, 0, kcs, blockIdx.x, nb, nb);
    // ---- inverse Lanczos steps
    const bool fuseK = P.eK.tri && P.eK.fuse;
    for (int j = 1; j < P.kmax; ++j) {
        const bool fold = a.fold && fuseK;   // h summed inside the elimination (R22): no phase A, no barrier
        elim_coop<KM, TIM>(grid, a, P.eK, P.MW + size_t(j - 1) * nf, scl, P.w, dsm, c, lb, nbc, stamp, nelim,
                       fold ? j : 0, kcs[c], pp, r0, rs, nullptr, kcs);   // w = K^-1 M q_j
        const bool part = act[c] && !brk[c];
        const int kc = kcs[c];
        const bool dbg = TIM && a.timers && blockIdx.x == 0 && tid == 32 && j == 5;
        if (fold) {
            read_totals(a, pp, 1 + kc, nb, tot, use_shr(a, P.eK, c));
            pp ^= 1;
            if (tid < KMAX) hsm[c][tid] = tid < kc ? tot[c][1 + tid] * sclh[c][tid] * sclh[c][tid] : 0.0;
            __syncthreads();
        } else {
        // A: (M w, L w) by one SpMV over the shared pattern; ||w||_M^2 and h_t = W_t . M w
#define DBGT(k) do { if (dbg) a.timers[k] = gtimer(); } while (0)
        DBGT(120);
        if (TIM && a.timers && j == 5 && tid == 32) a.timers[200 + 4096 + 1024 + blockIdx.x] = gtimer();   // A start
        const long long tA0 = clock64();
        ZERO_VALS();
        if (part)
            for (int64_t i = r0; i < hi; i += rs) {
                double wt[KM];   // basis loads first (the stores below may alias them for the compiler)
#pragma unroll
                for (int t = 0; t < KM; ++t) wt[t] = t < kc ? P.W[size_t(t) * nf + i] : 0.0;
                double m, l, wi;
                if (fuseK) {
                    wi = spmv_elim(P.M, P.L, i, P.eK, P.y, P.y + nf, m, l);
                    P.w[i] = wi;
                } else {
                    spmv_ml(P.M, P.L, i, P.w, m, l);
                    wi = P.w[i];
                }
                a.mw1[i] = m;
                a.lw1[i] = l;
                vals[0] += wi * m;
#pragma unroll
                for (int t = 0; t < KM; ++t) vals[1 + t] += wt[t] * m;
            }
        DBGT(121);
        if (TIM && a.timers && j == 5 && blockIdx.x < 4 && (tid & 31) == 0) a.timers[140 + blockIdx.x * CW + (tid >> 5)] = clock64() - tA0;
        block_partials(a, vals, 1 + KM, pp, c, lb, sred);
        DBGT(122);
        if (TIM && a.timers && j == 5 && tid == 32) {
            a.timers[200 + 4096 + 1536 + blockIdx.x] = gtimer();   // A arrival
            unsigned sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            a.timers[200 + 4096 + 2048 + blockIdx.x] = sm;
        }
        grid.sync();
    __syncwarp();   // lane 0 spun in the barrier: reconverge before warp-synchronous code
    STAMP(stamp++);
        DBGT(123);
        read_totals(a, pp, 1 + kc, nb, tot);   // every component's first 1+kc (kc uniform enough: use own)
        DBGT(124);
        pp ^= 1;
        if (tid < nc) nb2v[tid] = tot[tid][0];
        if (tid < KMAX) hsm[c][tid] = tid < kc ? tot[c][1 + tid] * sclh[c][tid] * sclh[c][tid] : 0.0;
        __syncthreads();
        }   // !fold
        if (a.gram_cgs2) {
            // second Gram-Schmidt pass from the Gram matrix (R21): h' = W^T M (w - W h) = h - G h with
            // G = W^T M W from the Gram rows 0..kc-1 (summed by now), so w2 = w - W (2h - G h) in one pass over the
            // rows; per raw basis vector the coefficient is 2 hsm_t - sclh_t^2 sum_s Graw_M[t][s] hsm_s
            double* gsm = dsm;   // [KMAX][KMAX] raw M-Gram of this component (dsm is free between phases)
            for (int e = tid; e < kc * kc; e += CT) {
                const int t = e / kc, u = e - t * kc, hi_ = t > u ? t : u, lo_ = t > u ? u : t;
                gsm[t * KMAX + u] = *((volatile const double*)(a.gram_tot + (size_t(c) * KMAX + hi_) * GW + KMAX + lo_));
            }
            __syncthreads();
            double hn = 0.0;
            if (tid < kc) {
                double g = 0.0;
                for (int u = 0; u < kc; ++u) g += gsm[tid * KMAX + u] * hsm[c][u];
                hn = 2.0 * hsm[c][tid] - sclh[c][tid] * sclh[c][tid] * g;
            }
            __syncthreads();
            if (tid < kc) hsm[c][tid] = hn;
            __syncthreads();
        }
        // B: w1 = w - W h; M w1 = M w - (M W) h and L w1 = L w - (L W) h by linearity (own rows only);
        // dots h'_t = W_t . M w1
        if (!a.gram_cgs2) {
        DBGT(130);
        ZERO_VALS();
        if (part)
            for (int64_t i = r0; i < hi; i += rs) {
                double wt[KM], mt[KM], lt[KM];
#pragma unroll
                for (int t = 0; t < KM; ++t) {
                    const bool ok = t < kc;
                    wt[t] = ok ? P.W[size_t(t) * nf + i] : 0.0;
                    mt[t] = ok ? P.MW[size_t(t) * nf + i] : 0.0;
                    lt[t] = ok ? P.LW[size_t(t) * nf + i] : 0.0;
                }
                double x = P.w[i], m = a.mw1[i], l = a.lw1[i];
#pragma unroll
                for (int t = 0; t < KM; ++t) {
                    x -= hsm[c][t] * wt[t];
                    m -= hsm[c][t] * mt[t];
                    l -= hsm[c][t] * lt[t];
                }
                a.w1[i] = x;
                a.mw1[i] = m;
                a.lw1[i] = l;
#pragma unroll
                for (int t = 0; t < KM; ++t) vals[t] += wt[t] * m;
            }
        DBGT(131);
        block_partials(a, vals, KM, pp, c, lb, sred);
        DBGT(132);
        grid.sync();
    __syncwarp();   // lane 0 spun in the barrier: reconverge before warp-synchronous code
    STAMP(stamp++);
        DBGT(133);
        read_totals(a, pp, kc > 0 ? kc : 1, nb, tot);
        DBGT(134);
        pp ^= 1;
        if (tid < KMAX) hsm[c][tid] = tid < kc ? tot[c][tid] * sclh[c][tid] * sclh[c][tid] : 0.0;
        __syncthreads();
        }   // !a.gram_cgs2
        // C: w2 = w1 - W h' with M w2, L w2 by linearity (M w2 is the next solve's rhs); ||w2||_M^2; row j of
        // the Rayleigh-Ritz Gram matrices before normalisation: w2.(L W_t), w2.(M W_t) (t < j), w2.L w2,
        // w2.M w2, w2.r
        if (dbg) a.timers[110] = gtimer();
        if (TIM && a.timers && j == 5 && tid == 32 && fold) a.timers[200 + 4096 + 1024 + blockIdx.x] = gtimer();   // C start
        ZERO_VALS();
        gram_zero(gacc);
        if (part)
            for (int64_t i = r0; i < hi; i += rs) {
                double wt[KM], mt[KM], lt[KM];
#pragma unroll
                for (int t = 0; t < KM; ++t) {
                    const bool ok = t < kc;
                    wt[t] = ok ? P.W[size_t(t) * nf + i] : 0.0;
                    mt[t] = ok ? P.MW[size_t(t) * nf + i] : 0.0;
                    lt[t] = ok ? P.LW[size_t(t) * nf + i] : 0.0;
                }
                double x, m, l;
                if (fold) {   // the former phase A on the same row: w_i and (M w)_i, (L w)_i by the fused SpMV
                    x = P.eK.pat_id ? spmv_elim_pat(P.M, P.L, i, P.eK, P.y, P.y + nf, nf, m, l)
                        : (P.eK.fell_col ? spmv_elim_fell(P.M, P.L, i, P.eK, P.y, P.y + nf, nf, m, l)
                                         : spmv_elim(P.M, P.L, i, P.eK, P.y, P.y + nf, m, l));
                    vals[1] += x * m;   // ||w||_M^2 before the orthogonalisation (breakdown test)
                } else {
                    x = a.gram_cgs2 ? P.w[i] : a.w1[i];
                    m = a.mw1[i];
                    l = a.lw1[i];
                }
                const double rv = P.rf[i];
#pragma unroll
                for (int t = 0; t < KM; ++t) {
                    x -= hsm[c][t] * wt[t];
                    m -= hsm[c][t] * mt[t];
                    l -= hsm[c][t] * lt[t];
                }
                P.W[size_t(j) * nf + i] = x;
                P.MW[size_t(j) * nf + i] = m;   // also the next solve's right-hand side (unnormalised, scaled by scl)
                P.LW[size_t(j) * nf + i] = l;
                vals[0] += x * m;
#pragma unroll
                for (int t = 0; t < KM; ++t)
                    if (t < kc) {
                        gacc[t * CT + tid] += x * lt[t];
                        gacc[(KMAX + t) * CT + tid] += x * mt[t];
                    }
                gacc[kc * CT + tid] += x * l;
                gacc[(KMAX + kc) * CT + tid] += x * m;
                gacc[2 * KMAX * CT + tid] += x * rv;
            }
        if (dbg) a.timers[111] = gtimer();
        if (part) gram_partials(a, gacc, c, lb, j);
        block_partials(a, vals, fold ? 2 : 1, pp, c, lb, sred);
        if (dbg) a.timers[112] = gtimer();
        if (TIM && a.timers && j == 5 && tid == 32 && fold) {   // per-block arrival at the phase-C barrier (tools/prec_timers.py)
            a.timers[200 + 4096 + 1536 + blockIdx.x] = gtimer();
            unsigned sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            a.timers[200 + 4096 + 2048 + blockIdx.x] = sm;
        }
        grid.sync();
    __syncwarp();   // lane 0 spun in the barrier: reconverge before warp-synchronous code
    STAMP(stamp++);
        if (dbg) a.timers[113] = gtimer();
        read_totals(a, pp, fold ? 2 : 1, nb, tot);
        if (dbg) a.timers[114] = gtimer();
        pp ^= 1;
        if (fold && tid < nc) nb2v[tid] = tot[tid][1];
        __syncthreads();
        if (tid < nc) {
            const bool pt = act[tid] && !brk[tid];
            const double na = sqrt(fmax(tot[tid][0], 0.0)), nbn = sqrt(fmax(nb2v[tid], 0.0));
            if (pt) {
                if (na > 1e-12 * nbn) {
                    kcs[tid] = j + 1;
                    scl[tid] = 1.0 / na;
                    sclh[tid][j] = scl[tid];
                } else {
                    brk[tid] = 1;
                    scl[tid] = 0.0;
                }
            } else {
                scl[tid] = 0.0;
            }
        }
        __syncthreads();
        if (j + 1 < P.kmax && tid < 32) gram_row_sums(a, j, kcs, blockIdx.x, nb, nb);
    }
    // block 0: per component the basis size, activity and the scales; the last Gram row's fixed-order sums and the
    // scaled Gram matrices are formed by k_prec_ritz (one CTA per component) instead of serially here
    if (blockIdx.x == 0) {
        if (tid < nc * KMAX) {
            const int cc = tid / KMAX, t = tid - cc * KMAX;
            LzState& zs = P.lz[cc];
            zs.sc[t] = t < kcs[cc] ? sclh[cc][t] : 0.0;
            if (t == 0) {
                zs.kc = kcs[cc];
                zs.active = act[cc];
            }
        }
        STAMP(stamp++);
    }
    // every elimination's arrivals lie before the last grid barrier above: leave the counter at zero for the next launch
    if (blockIdx.x == 0 && tid == 0) *a.arrive = 0u;
    // the k x k Ritz problems (k_prec_ritz) and the combine (k_prec_combine) follow as two small launches: the
    // Ritz code runs there without this kernel's register cap, and one grid barrier is saved
}

#undef ZERO_VALS

// One CTA per component: the last Gram row's fixed-order sums (rows < kmax-1 were summed inside k_prec_coop), the
// Gram matrices scaled by the basis normalisation, then the k x k Ritz problem on warp 0 -> coefficients
// (no register cap here: the Jacobi and the triangular solves stay in registers / shared memory).
template <bool TIM>
__global__ void __launch_bounds__(CT) k_prec_ritz(PrecDev P, const double* __restrict__ gram,
                                                  const double* __restrict__ gram_tot, int nbc_max, int nb,
                                                  const PcgState* s, unsigned long long* timers) {
    if (s != nullptr && s->done) return;
    extern __shared__ double rsm[];
    __shared__ double As[KMAX * KMAX], Bs[KMAX * KMAX], wrs[KMAX], lastrow[GW], scs[KMAX];
    const int w = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;   // CTA w = component w
    if (w >= P.ncomp) return;
    LzState& zs = P.lz[w];
    if (tid < KMAX) zs.coef[tid] = 0.0;
    if (!zs.active) return;
    const int kc = zs.kc, nc = P.ncomp;
    if (tid < KMAX) scs[tid] = zs.sc[tid];
    if (TIM && timers && w == 0 && tid == 0) timers[100] = gtimer();
    if (kc == P.kmax) {   // row kmax-1: lanes add the block partials b = lane, lane+32, .. in order, then a warp tree
        const int jr = kc - 1, per = 2 * (jr + 1) + 1, nbcc = (nb - w + nc - 1) / nc;
        for (int q = wid; q < per; q += CW) {
            const int v = q <= jr ? q : (q < 2 * (jr + 1) ? KMAX + (q - jr - 1) : 2 * KMAX);
            const double* pg = gram + ((size_t(w) * KMAX + jr) * GW + v) * nbc_max;
            double acc = 0.0;
            for (int b = lane; b < nbc_max; b += 32) acc += b < nbcc ? pg[b] : 0.0;
            acc = warp_sum(acc);
            if (lane == 0) lastrow[v] = acc;
        }
    }
    __syncthreads();
    for (int e = tid; e < KMAX * GW; e += CT) {
        const int jr = e / GW, v = e - jr * GW;
        if (jr >= kc) continue;
        const int kind = v < KMAX ? 0 : (v < 2 * KMAX ? 1 : 2), t = kind == 0 ? v : v - KMAX;
        if (kind < 2 && t > jr) continue;
        const double acc = jr == P.kmax - 1 ? lastrow[v] : gram_tot[(size_t(w) * KMAX + jr) * GW + v];
        if (kind == 2) {
            wrs[jr] = scs[jr] * acc;
        } else {
            const double g = scs[jr] * scs[t] * acc;   // (sc_j Wraw_j)^T L (sc_t Wraw_t)
            double* G = kind == 0 ? As : Bs;
            G[jr * KMAX + t] = g;
            G[t * KMAX + jr] = g;
        }
    }
    __syncthreads();
    double* R = rsm;
    double* Cm = R + KMAX * (KMAX + 1);
    double* V = Cm + KMAX * (KMAX + 1);
    double* X = V + KMAX * (KMAX + 1);
    double* rot = X + KMAX * (KMAX + 1);
    int* rpq = reinterpret_cast<int*>(rot + KMAX);
    unsigned long long* tm = (TIM && timers && w == 0) ? timers + 102 : nullptr;
    bool ok;
    if (P.jacobi_reg == 0 && kc > 1) {   // default: Cholesky / C = L^-1 A L^-T on warp 0, the Jacobi by the whole CTA
        __shared__ int sched[KMAX * KMAX], slot_of[KMAX], jflag, okf;
        __shared__ double csn[KMAX], jred[2 * CW];
        if (wid == 0) {
            const bool o1 = ritz_warp(As, Bs, wrs, kc, P.singular[w] != 0, P.theta, zs.coef, R, Cm, V, X, rot, rpq, tm, 0, 1);
            if (lane == 0) okf = o1 ? 1 : 0;
        }
        __syncthreads();
        int nsw = 0;
        if (okf) nsw = jacobi_block(Cm, V, kc, sched, slot_of, csn, jred, &jflag);
        __syncthreads();
        if (wid != 0) return;
        if (tm && lane == 0) tm[4] = nsw;
        ok = okf && ritz_warp(As, Bs, wrs, kc, P.singular[w] != 0, P.theta, zs.coef, R, Cm, V, X, rot, rpq, tm, 0, 2);
    } else {
        if (wid != 0) return;
        ok = ritz_warp(As, Bs, wrs, kc, P.singular[w] != 0, P.theta, zs.coef, R, Cm, V, X, rot, rpq, tm, P.jacobi_reg);
    }
    if (TIM && timers && w == 0 && lane == 0) timers[101] = gtimer();
    if (!ok && lane == 0) {
        zs.status = DE_EBREAKDOWN;
        for (int e = 0; e < KMAX; ++e) zs.coef[e] = 0.0;
        if (s) {
            PcgState* sm = const_cast<PcgState*>(s);
            sm->status = DE_EBREAKDOWN;
            sm->done = 1;
        }
    }
}

// z = sum_t coef_t W_t = sum_t (coef_t sc_t) Wraw_t, scattered back to interface order
__global__ void __launch_bounds__(256) k_prec_combine(PrecDev P, double* __restrict__ z, const PcgState* s) {
    if (s != nullptr && s->done) return;
    __shared__ double cs[MAXC][KMAX];
    __shared__ int kc[MAXC];
    if (threadIdx.x < P.ncomp * KMAX) {
        const int c = threadIdx.x / KMAX, t = threadIdx.x - c * KMAX;
        const LzState& zs = P.lz[c];
        cs[c][t] = zs.active ? zs.coef[t] * zs.sc[t] : 0.0;
        if (t == 0) kc[c] = zs.active ? zs.kc : 0;
    }
    __syncthreads();
    const size_t nf = size_t(P.nflat);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P.nflat; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = ccomp(P.comp_off, P.ncomp, i);
        double acc = 0.0;
        for (int t = 0; t < kc[c]; ++t) acc += cs[c][t] * P.W[size_t(t) * nf + i];
        z[P.cmap[i]] = acc;
    }
}

// ------------------------------------------------------------------ host side
bool prec_coop_prepare(const PrecDev& P, int device, CoopBuffers& B) {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    int coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
    if (!coop) return false;
    const int mf = std::max(P.eK.maxface & 0xffff, P.eM.maxface & 0xffff);
    int ncmax = 1;
    for (const ElimDev* E : {&P.eK, &P.eM})
        for (int c = 0; c < P.ncomp; ++c) ncmax = std::max(ncmax, E->cross_comp_off[c + 1] - E->cross_comp_off[c]);
    // per face-solving warp (warps 1..CW-1): rhs / y / node ids (mf each) + the two-chunk column ring of face_warp
    int maxld = 1;
    for (const ElimDev* E : {&P.eK, &P.eM}) maxld = std::max(maxld, E->maxld);
    const bool stage = false;
    const int per_warp = 3 * mf + 2 * 32 * maxld;
    size_t smem = size_t(CW - 1) * per_warp * 8;
    {   // t_C plus the per-warp partials of the rows one block owns in the cross-point GEMV (>= 1 block per SM)
        const int nbc_lo = std::max(1, nsm / std::max(1, P.ncomp));
        smem = std::max(smem, (size_t(ncmax) + size_t(CW) * ((ncmax + nbc_lo - 1) / nbc_lo)) * 8);
    }
    smem = std::max(smem, size_t(GW) * CT * 8);      // per-thread Gram accumulators
    for (const ElimDev* E : {&P.eK, &P.eM})          // fast-diagonalised cross-point solve: X, Y and the staged Q tables
        if (E->fd) {
            const size_t need = (size_t(2) * ncmax + 1 + size_t(E->fd_nx) * E->fd_nx + size_t(E->fd_ny) * E->fd_ny) * 8;
            if (need <= 96 * 1024) smem = std::max(smem, need);   // larger grids keep the dense S_C^-1 path
        }
    smem = std::max(smem, size_t(RW) * TRI_N * 8);   // per-thread forward solutions of tridiagonal faces
    smem = std::max(smem, size_t(CW) * (4 * KMAX * (KMAX + 1) + 2 * KMAX + 4 * KMAX) * 8);
    if (smem > 200 * 1024) return false;
    typedef void (*coop_fn)(CoopArgs);
    const bool tim = getenv("DE_PREC_TIMERS") != nullptr;
    coop_fn kfn = P.kmax <= 10 ? (tim ? k_prec_coop<10, true> : k_prec_coop<10, false>) : k_prec_coop<KMAX, false>;
    if (tim && P.kmax > 10) kfn = k_prec_coop<KMAX, true>;
    raise_dyn_smem(reinterpret_cast<const void*>(kfn), smem);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, CT, smem) != cudaSuccess || per_sm < 1)
        return false;
    int bps = 2;   // blocks per SM; DE_COOP_BPS overrides (tuning experiments only)
    if (const char* e = getenv("DE_COOP_BPS")) bps = std::max(1, atoi(e));
    const int nb = nsm * std::min(per_sm, bps);
    if (nb < P.ncomp) return false;
    {   // guaranteed by the sizing above (nb >= nsm)
        const int nbc_min = nb / P.ncomp;
        const size_t need = (size_t(ncmax) + size_t(CW) * ((ncmax + nbc_min - 1) / nbc_min)) * 8;
        if (need > smem) return false;
    }
    if (getenv("DE_VERBOSE"))
        fprintf(stderr, "[de] k_prec_coop: %d blocks (%d resident/SM possible), %zu B smem\n", nb, per_sm, smem);
    B.nb = nb;
    B.nsm = nsm;
    B.kfn = reinterpret_cast<const void*>(kfn);
    B.smem = smem;
    B.stage = stage ? 1 : 0;
    B.per_warp = per_warp;
    B.mf = mf;
    B.ncmax = ncmax;
    B.tridiag = (P.eK.tri && P.eM.tri) ? 1 : 0;   // informational; each ElimDev carries its own flag
    B.nbc_max = (nb + P.ncomp - 1) / P.ncomp;
    B.gram_cgs2 = getenv("DE_CGS2_TWO_PASS") ? 0 : 1;   // A/B switch: the literal two-pass CGS2
    // fold h into the elimination (R22): 2D fused eliminations, one-pass Gram-Schmidt, room for the accumulators
    B.fold = (B.gram_cgs2 && P.eK.tri && P.eK.fuse && !getenv("DE_NO_FOLD")) ? 1 : 0;
    {   // shared-row cross-point solve: t_C of every component + the per-warp row sums must fit
        const size_t need = (size_t(P.ncomp) * ncmax + size_t(CW) * P.ncomp * (ncmax / nb + 2)) * 8;
        // two components (2D): measured slower on c5 (0.569 vs 0.547 ms: the partner block's reads of the same rows hit
        // L2 anyway); three (3D wirebasket): c4 cross-point phase 34 -> 31.8 us
        B.shr = ((P.ncomp > 2 || getenv("DE_SHR")) && need <= B.smem && !getenv("DE_NO_SHR")) ? 1 : 0;
    }
    B.sc_persist = 0;
    B.sc_persist_bytes = 0;
    if (getenv("DE_SC_PERSIST") && !P.eK.fd) {   // opt-in A/B: persisting-L2 window over eK's S_C^-1 (<= 40 MB)
        size_t bytes = 0;
        for (int c = 0; c < (P.eK.sc_shared ? 1 : P.ncomp); ++c) {
            const size_t n = size_t(P.eK.cross_comp_off[c + 1] - P.eK.cross_comp_off[c]);
            bytes += n * n * 8;
        }
        int maxp = 0;
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, device);
        if (bytes > 0 && bytes <= size_t(40) << 20 && bytes <= size_t(maxp)) {
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes);
            B.sc_persist = 1;
            B.sc_persist_bytes = bytes;
        }
        if (getenv("DE_VERBOSE")) fprintf(stderr, "[de] S_C^-1 persisting window: %zu bytes (max %d) -> %d\n", bytes, maxp, B.sc_persist);
    }
    B.split = getenv("DE_NO_SPLIT") ? 0 : 1;   // A/B switch: a grid barrier between t_C and the cross-point solve
    if (getenv("DE_VERBOSE")) fprintf(stderr, "[de] k_prec_coop: fold %d (R22) split %d\n", B.fold, B.split);
    return true;
}

size_t prec_coop_red_doubles(const CoopBuffers& B) { return size_t(2) * MAXC * NRED * B.nbc_max; }
size_t prec_coop_gram_doubles(const CoopBuffers& B) { return size_t(MAXC) * GRAM_TASKS * B.nbc_max; }

int prec_apply_coop(const PrecDev& P, const CoopBuffers& B, const double* r, double* z, const PcgState* s,
                    cudaStream_t st, bool literal) {
    CoopArgs a{};
    a.P = P;
    a.r = r;
    a.z = z;
    a.s = s;
    a.red = B.red;
    a.gram = B.gram;
    a.gram_tot = B.gram_tot;
    a.w1 = B.w1;
    a.mw1 = B.mw1;
    a.lw1 = B.lw1;
    a.nbc_max = B.nbc_max;
    a.stage = B.stage;
    a.per_warp = B.per_warp;
    a.mf = B.mf;
    a.ncmax = B.ncmax;
    a.tridiag = B.tridiag;
    a.gram_cgs2 = literal ? 0 : B.gram_cgs2;   // literal: SPEC's two-pass CGS2 (used under FGMRES)
    a.fold = literal ? 0 : B.fold;
    a.ucross = B.ucross;
    a.arrive = B.arrive;
    a.split = B.split;
    a.sc_persist = B.sc_persist;
    a.shr = B.shr;
    a.redf = B.redf;
    a.smem_doubles = int(B.smem / sizeof(double));
    a.timers = B.timers;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(B.nb);
    cfg.blockDim = dim3(CT);
    cfg.dynamicSmemBytes = B.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (B.sc_persist) {   // eK's S_C^-1 (re-read by every K-elimination) held in the persisting L2 set-aside
        attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[1].val.accessPolicyWindow.base_ptr = const_cast<double*>(P.eK.Sinv);
        attr[1].val.accessPolicyWindow.num_bytes = B.sc_persist_bytes;
        attr[1].val.accessPolicyWindow.hitRatio = 1.0f;
        attr[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.numAttrs = 2;
    }
    cudaError_t e = cudaLaunchKernelEx(&cfg, reinterpret_cast<void (*)(CoopArgs)>(const_cast<void*>(B.kfn)), a);
    if (e != cudaSuccess) return -1;
    const size_t rsm = size_t(4 * KMAX * (KMAX + 1) + 6 * KMAX) * sizeof(double);
    if (B.timers) k_prec_ritz<true><<<P.ncomp, CT, rsm, st>>>(P, B.gram, B.gram_tot, B.nbc_max, B.nb, s, B.timers);
    else k_prec_ritz<false><<<P.ncomp, CT, rsm, st>>>(P, B.gram, B.gram_tot, B.nbc_max, B.nb, s, nullptr);
    k_prec_combine<<<B.nsm * 4, 256, 0, st>>>(P, z, s);
    e = cudaGetLastError();
    return e == cudaSuccess ? 3 : -1;
}

}  // namespace de
