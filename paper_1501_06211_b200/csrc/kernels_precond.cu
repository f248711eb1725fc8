// kernels_precond.cu — SURVEY.md §8(a) row C5: the interface preconditioner z = H^_theta^-1 r
// (Eqs. (8)-(9); inverse Lanczos PAPER.md:181,191; R7,R9,R10).
// All displacement components are batched in one flattened skeleton index space (block-diagonal).
//
// Per component c (skipped when r_c = 0):
//   s = M^-1 r_c                            (exact: faces -> cross-point Schur complement -> faces)
//   q_1 = s / ||s||_M
//   q_{j+1} ~ K^-1 M q_j, CGS2 in the M inner product, breakdown if ||w||_M <= 1e-12 ||w_0||_M
//   A_k = W^T L W, B_k = W^T M W;  (Theta, Y) = eig(A_k, B_k), Y^T B_k Y = I
//   z_c = W Y f(Theta) Y^T W^T r_c,   f = Theta^(theta-1)   (or 1/(1+Theta^(1-theta)) if singular, R7)
// K = L_c (or L_c + M_c when singular). Exact inner solves with X in {K, M} (mode X, R10):
//   y_F = X_FF^-1 b_F (warp per face, band factor in smem);  x_C = S_C^-1 (b_C - X_CF y_F) (dense GEMV);
//   x_F = X_FF^-1 (b_F - X_FC x_C).
// Reductions are fixed-shape (deterministic), segmented per component and per task.
#include "de_internal.h"

namespace de {

constexpr int PB = 256;

__device__ __forceinline__ int comp_of(const int64_t* off, int ncomp, int64_t i) {
    int c = 0;
    while (c + 1 < ncomp && i >= off[c + 1]) ++c;
    return c;
}

__device__ __forceinline__ bool lz_part(const LzState& z) { return z.active && !z.broke; }

// Block reduce + segmented last-block finalisation. Partials part[(slot)*nblk + bx].
__device__ __forceinline__ double pblock_sum(double v, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = (l < int(blockDim.x >> 5)) ? sh[l] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    __syncthreads();
    return r;
}

// returns true in thread 0 of the last block of this slot; *tot holds the total
__device__ bool seg_reduce(double v, int slot, int nblk, double* part, unsigned int* counter, double* tot) {
    __shared__ double sh[32];
    __shared__ bool last;
    const double bs = pblock_sum(v, sh);
    if (threadIdx.x == 0) {
        part[size_t(slot) * nblk + blockIdx.x] = bs;
        __threadfence();
        last = (atomicAdd(counter + slot, 1u) == unsigned(nblk - 1));
    }
    __syncthreads();
    if (!last) return false;
    __threadfence();
    double acc = 0.0;
    for (int b = threadIdx.x; b < nblk; b += blockDim.x) acc += *((volatile double*)&part[size_t(slot) * nblk + b]);
    const double t = pblock_sum(acc, sh);
    if (threadIdx.x == 0) {
        counter[slot] = 0u;
        *tot = t;
    }
    return threadIdx.x == 0;
}

// ------------------------------------------------------------------ gather r -> rf, zero test
__global__ void k_prec_init(PrecDev P, const double* __restrict__ r, const PcgState* s) {
    if (s && s->done) return;
    const int c = blockIdx.y;
    const int64_t lo = P.comp_off[c], hi = P.comp_off[c + 1];
    double v = 0.0;
    for (int64_t i = lo + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < hi; i += int64_t(gridDim.x) * blockDim.x) {
        const double x = r[P.cmap[i]];
        P.rf[i] = x;
        v += x * x;
    }
    double tot;
    if (seg_reduce(v, c, gridDim.x, P.part, P.counter, &tot)) {
        LzState& z = P.lz[c];
        z.rr = tot;
        z.active = tot > 0.0 ? 1 : 0;
        z.kc = 0;
        z.broke = 0;
        z.status = 0;
    }
}

// ------------------------------------------------------------------ exact elimination solves
// mode 0: y_F = X_FF^-1 b_F ; mode 1: x_F = X_FF^-1 (b_F - X_FC xC)
__global__ void k_face_solve(ElimDev E, const double* __restrict__ b, const double* __restrict__ xC,
                             double* __restrict__ out, int mode, int maxf, int maxfac, const PcgState* s) {
    if (s && s->done) return;
    extern __shared__ double fsm[];
    const int wpb = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int F = blockIdx.x * wpb + w;
    if (F >= E.nfaces) return;
    double* v = fsm + size_t(w) * (maxf + maxfac);
    double* fac = v + maxf;
    const int o = E.face_off[F], n = E.face_off[F + 1] - o, bw = E.face_band[F], ld = bw + 1;
    const double* gf = E.face_fac + E.face_fac_off[F];
    for (int i = lane; i < n * ld; i += 32) fac[i] = gf[i];
    for (int i = lane; i < n; i += 32) {
        double r = b[E.face_nodes[o + i]];
        if (mode == 1)
            for (int e = E.xfc_ptr[o + i]; e < E.xfc_ptr[o + i + 1]; ++e) r -= E.xfc_val[e] * xC[E.xfc_col[e]];
        v[i] = r;
    }
    __syncwarp();
    for (int j = 0; j < n; ++j) {
        const double vj = v[j] * fac[j * ld];
        for (int k = lane + 1; k <= bw && j + k < n; k += 32) v[j + k] -= fac[j * ld + k] * vj;
        __syncwarp();
        if (lane == 0) v[j] = vj;
        __syncwarp();
    }
    for (int j = n - 1; j >= 0; --j) {
        double t = 0.0;
        for (int k = lane + 1; k <= bw && j + k < n; k += 32) t += fac[j * ld + k] * v[j + k];
        for (int off = 1; off < min(bw, 32); off <<= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
        t = __shfl_sync(0xffffffffu, t, 0);
        const double vj = (v[j] - t) * fac[j * ld];
        __syncwarp();
        if (lane == 0) v[j] = vj;
        __syncwarp();
    }
    for (int i = lane; i < n; i += 32) out[E.face_nodes[o + i]] = v[i];
}

// x_C = S_C^-1 (b_C - X_CF y): each CTA rebuilds t_C of its component in smem, warps do rows.
__global__ void k_cross_solve(ElimDev E, const double* __restrict__ b, const double* __restrict__ y,
                              double* __restrict__ xC, double* __restrict__ x, int rows_per_cta, const PcgState* s) {
    if (s && s->done) return;
    extern __shared__ double tC[];
    const int c = blockIdx.y;
    const int base = E.cross_comp_off[c], nc = E.cross_comp_off[c + 1] - base;
    const int r0 = blockIdx.x * rows_per_cta;
    if (r0 >= nc) return;
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
        const int ci = base + i;
        double t = b[E.cross_flat[ci]];
        for (int e = E.xcf_ptr[ci]; e < E.xcf_ptr[ci + 1]; ++e) t -= E.xcf_val[e] * y[E.xcf_col[e]];
        tC[i] = t;
    }
    __syncthreads();
    const int wpb = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double* S = E.Sinv + E.sc_off[c];
    for (int rr = r0 + w; rr < min(r0 + rows_per_cta, nc); rr += wpb) {
        const double* row = S + size_t(rr) * nc;
        double acc = 0.0;
        for (int j = lane; j < nc; j += 32) acc += row[j] * tC[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            xC[base + rr] = acc;
            x[E.cross_flat[base + rr]] = acc;
        }
    }
}

static void elim_solve(const PrecDev& P, const ElimDev& E, const double* b, double* x, const PcgState* s,
                       cudaStream_t st, int* nl) {
    const int maxf = P.nblk;   // unused placeholder
    (void)maxf;
    // sizes for the face kernel are stashed in E.maxface (max nodes) and derived factor size
    const int mf = E.maxface & 0xffff, mfac = E.maxface >> 16;
    const int wpb = 4;
    const size_t smem_face = size_t(wpb) * (mf + mfac) * sizeof(double);
    double* y = P.y;
    double* xC = P.y + P.nflat;   // cross solution scratch (ncross entries)
    if (E.nfaces > 0) {
        k_face_solve<<<(E.nfaces + wpb - 1) / wpb, 32 * wpb, smem_face, st>>>(E, b, xC, y, 0, mf, mfac, s);
        ++*nl;
    }
    if (E.ncross > 0) {
        int ncmax = 0;
        for (int c = 0; c < P.ncomp; ++c) ncmax = std::max(ncmax, E.cross_comp_off[c + 1] - E.cross_comp_off[c]);
        const int rows = 16;
        dim3 grid((ncmax + rows - 1) / rows, P.ncomp);
        k_cross_solve<<<grid, 256, size_t(ncmax) * sizeof(double), st>>>(E, b, y, xC, x, rows, s);
        ++*nl;
    }
    if (E.nfaces > 0) {
        k_face_solve<<<(E.nfaces + wpb - 1) / wpb, 32 * wpb, smem_face, st>>>(E, b, xC, x, 1, mf, mfac, s);
        ++*nl;
    }
}

// ------------------------------------------------------------------ SpMV (+ fused M-norm)
// field: 0 -> nrm2 (seed), 1 -> nb2, 2 -> na2 (breakdown test), -1 -> no dot
__global__ void k_spmv_dot(PrecDev P, CsrDev A, const double* __restrict__ x, double* __restrict__ y, int field,
                           int j, const PcgState* s) {
    if (s && s->done) return;
    const int c = blockIdx.y;
    const int64_t lo = P.comp_off[c], hi = P.comp_off[c + 1];
    double v = 0.0;
    for (int64_t i = lo + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < hi; i += int64_t(gridDim.x) * blockDim.x) {
        double acc = 0.0;
        for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) acc += A.val[e] * x[A.col[e]];
        y[i] = acc;
        v += x[i] * acc;
    }
    if (field < 0) return;
    double tot;
    if (seg_reduce(v, c, gridDim.x, P.part, P.counter, &tot)) {
        LzState& z = P.lz[c];
        if (field == 0) {
            z.nrm2 = tot;
            if (z.active) z.kc = 1;
        } else if (field == 1) {
            z.nb2 = tot;
        } else {
            z.na2 = tot;
            if (lz_part(z)) {
                const double na = sqrt(fmax(tot, 0.0)), nb = sqrt(fmax(z.nb2, 0.0));
                if (na > 1e-12 * nb) z.kc = j + 1;
                else z.broke = 1;
            }
        }
    }
}

// W_j = w / ||w||_M, v = Mw / ||w||_M for participating components (j = 0: w = s, norm = nrm2)
__global__ void k_lz_normalize(PrecDev P, const double* __restrict__ w, const double* __restrict__ Mw, int j,
                               const PcgState* s) {
    if (s && s->done) return;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P.nflat; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = comp_of(P.comp_off, P.ncomp, i);
        const LzState& z = P.lz[c];
        if (!z.active || z.kc != j + 1) continue;   // kc was advanced iff q_{j} is accepted
        const double inv = 1.0 / sqrt(j == 0 ? z.nrm2 : z.na2);
        P.W[size_t(j) * P.nflat + i] = w[i] * inv;
        P.v[i] = Mw[i] * inv;
    }
}

// h_t = W_t . vec for t < kc (one task per blockIdx.z... tasks in blockIdx.y, components in z)
__global__ void k_mdot_h(PrecDev P, const double* __restrict__ vec, const PcgState* s) {
    if (s && s->done) return;
    const int t = blockIdx.y, c = blockIdx.z;
    const LzState& z = P.lz[c];
    if (!lz_part(z) || t >= z.kc) return;
    const int64_t lo = P.comp_off[c], hi = P.comp_off[c + 1];
    const double* Wt = P.W + size_t(t) * P.nflat;
    double v = 0.0;
    for (int64_t i = lo + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < hi; i += int64_t(gridDim.x) * blockDim.x)
        v += Wt[i] * vec[i];
    double tot;
    if (seg_reduce(v, 8 + c * KMAX + t, gridDim.x, P.part, P.counter, &tot)) P.lz[c].h[t] = tot;
}

__global__ void k_axpy_basis(PrecDev P, double* __restrict__ w, const PcgState* s) {
    if (s && s->done) return;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P.nflat; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = comp_of(P.comp_off, P.ncomp, i);
        const LzState& z = P.lz[c];
        if (!lz_part(z)) continue;
        double acc = w[i];
        for (int t = 0; t < z.kc; ++t) acc -= z.h[t] * P.W[size_t(t) * P.nflat + i];
        w[i] = acc;
    }
}

// out_t = A W_t for t < kc (t in blockIdx.y)
__global__ void k_spmv_multi(PrecDev P, CsrDev A, double* __restrict__ out, const PcgState* s) {
    if (s && s->done) return;
    const int t = blockIdx.y;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P.nflat; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = comp_of(P.comp_off, P.ncomp, i);
        if (!P.lz[c].active || t >= P.lz[c].kc) continue;
        const double* Wt = P.W + size_t(t) * P.nflat;
        double acc = 0.0;
        for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e) acc += A.val[e] * Wt[A.col[e]];
        out[size_t(t) * P.nflat + i] = acc;
    }
}

// Rayleigh-Ritz dots: tasks (i <= j) A_ij = W_i.LW_j, B_ij = W_i.MW_j, and wr_i = W_i.rf
__global__ void k_mdot_rr(PrecDev P, int kmax, const PcgState* s) {
    if (s && s->done) return;
    const int task = blockIdx.y, c = blockIdx.z;
    const LzState& z = P.lz[c];
    if (!z.active) return;
    const int kc = z.kc;
    const int npair = kc * (kc + 1) / 2;
    int kind, i = 0, j = 0;
    if (task < npair) kind = 0;
    else if (task < 2 * npair) kind = 1;
    else if (task < 2 * npair + kc) kind = 2;
    else return;
    int t = kind == 0 ? task : (kind == 1 ? task - npair : task - 2 * npair);
    if (kind < 2) {
        while (t >= kc - i) {
            t -= kc - i;
            ++i;
        }
        j = i + t;
    } else {
        i = t;
    }
    const int64_t lo = P.comp_off[c], hi = P.comp_off[c + 1];
    const double* a = P.W + size_t(i) * P.nflat;
    const double* b = kind == 0 ? P.LW + size_t(j) * P.nflat : (kind == 1 ? P.MW + size_t(j) * P.nflat : P.rf);
    double v = 0.0;
    for (int64_t x = lo + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; x < hi; x += int64_t(gridDim.x) * blockDim.x)
        v += a[x] * b[x];
    const int ntask = kmax * (kmax + 1) + kmax;
    double tot;
    if (seg_reduce(v, 8 + MAXC * KMAX + c * ntask + task, gridDim.x, P.part, P.counter, &tot)) {
        LzState& zz = P.lz[c];
        if (kind == 0) zz.A[i * KMAX + j] = zz.A[j * KMAX + i] = tot;
        else if (kind == 1) zz.B[i * KMAX + j] = zz.B[j * KMAX + i] = tot;
        else zz.wr[i] = tot;
    }
}

// Small generalized symmetric eigenproblem A y = theta B y per component (one thread each):
// Cholesky B = R R^T, C = R^-1 A R^-T, cyclic Jacobi, Y = R^-T V; coef = Y f(Theta) Y^T wr.
__global__ void k_lz_eig(PrecDev P, PcgState* s) {
    if (s && s->done) return;
    const int c = threadIdx.x;
    if (c >= P.ncomp) return;
    LzState& z = P.lz[c];
    for (int i = 0; i < KMAX; ++i) z.coef[i] = 0.0;
    if (!z.active) return;
    const int n = z.kc;
    double R[KMAX][KMAX], C[KMAX][KMAX], V[KMAX][KMAX];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) R[i][j] = (j <= i) ? z.B[i * KMAX + j] : 0.0;
    for (int j = 0; j < n; ++j) {          // Cholesky (lower)
        double d = R[j][j];
        for (int k = 0; k < j; ++k) d -= R[j][k] * R[j][k];
        if (!(d > 0.0)) {
            z.status = DE_EBREAKDOWN;
            if (s) { s->status = DE_EBREAKDOWN; s->done = 1; }
            return;
        }
        R[j][j] = sqrt(d);
        for (int i = j + 1; i < n; ++i) {
            double t = R[i][j];
            for (int k = 0; k < j; ++k) t -= R[i][k] * R[j][k];
            R[i][j] = t / R[j][j];
        }
    }
    // X = R^-1 A (column by column), then C = X R^-T  (i.e. C^T = R^-1 X^T)
    double X[KMAX][KMAX];
    for (int col = 0; col < n; ++col)
        for (int i = 0; i < n; ++i) {
            double t = z.A[i * KMAX + col];
            for (int k = 0; k < i; ++k) t -= R[i][k] * X[k][col];
            X[i][col] = t / R[i][i];
        }
    for (int row = 0; row < n; ++row)
        for (int i = 0; i < n; ++i) {
            double t = X[row][i];
            for (int k = 0; k < i; ++k) t -= R[i][k] * C[row][k];
            C[row][i] = t / R[i][i];
        }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const double m = 0.5 * (C[i][j] + C[j][i]);
            C[i][j] = m;
            V[i][j] = (i == j) ? 1.0 : 0.0;
        }
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0, dia = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) (i == j ? dia : off) += C[i][j] * C[i][j];
        if (off <= 1e-32 * dia) break;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = C[p][q];
                if (apq == 0.0) continue;
                const double tau = (C[q][q] - C[p][p]) / (2.0 * apq);
                const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                const double cs = 1.0 / sqrt(1.0 + t * t), sn = t * cs;
                for (int k = 0; k < n; ++k) {
                    const double ckp = C[k][p], ckq = C[k][q];
                    C[k][p] = cs * ckp - sn * ckq;
                    C[k][q] = sn * ckp + cs * ckq;
                }
                for (int k = 0; k < n; ++k) {
                    const double cpk = C[p][k], cqk = C[q][k];
                    C[p][k] = cs * cpk - sn * cqk;
                    C[q][k] = sn * cpk + cs * cqk;
                }
                for (int k = 0; k < n; ++k) {
                    const double vkp = V[k][p], vkq = V[k][q];
                    V[k][p] = cs * vkp - sn * vkq;
                    V[k][q] = sn * vkp + cs * vkq;
                }
            }
    }
    const bool sing = P.singular[c] != 0;
    double Y[KMAX][KMAX], f[KMAX];
    for (int e = 0; e < n; ++e) {
        const double th = C[e][e];
        z.theta_ritz[e] = th;
        if (!sing && !(th > 0.0)) {
            z.status = DE_EBREAKDOWN;
            if (s) { s->status = DE_EBREAKDOWN; s->done = 1; }
            return;
        }
        f[e] = sing ? 1.0 / (1.0 + pow(fmax(th, 0.0), 1.0 - P.theta)) : pow(th, P.theta - 1.0);
        for (int i = n - 1; i >= 0; --i) {   // Y(:,e) = R^-T V(:,e)
            double t = V[i][e];
            for (int k = i + 1; k < n; ++k) t -= R[k][i] * Y[k][e];
            Y[i][e] = t / R[i][i];
        }
    }
    double g[KMAX];
    for (int e = 0; e < n; ++e) {
        double t = 0.0;
        for (int i = 0; i < n; ++i) t += Y[i][e] * z.wr[i];
        g[e] = f[e] * t;
    }
    for (int i = 0; i < n; ++i) {
        double t = 0.0;
        for (int e = 0; e < n; ++e) t += Y[i][e] * g[e];
        z.coef[i] = t;
    }
}

__global__ void k_lz_combine(PrecDev P, double* __restrict__ zout, const PcgState* s) {
    if (s && s->done) return;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P.nflat; i += int64_t(gridDim.x) * blockDim.x) {
        const int c = comp_of(P.comp_off, P.ncomp, i);
        const LzState& z = P.lz[c];
        double acc = 0.0;
        if (z.active)
            for (int t = 0; t < z.kc; ++t) acc += z.coef[t] * P.W[size_t(t) * P.nflat + i];
        zout[P.cmap[i]] = acc;
    }
}

void prec_apply(const PrecDev& P, const double* r, double* z, const PcgState* s, cudaStream_t st, int* nlaunch) {
    int nl = 0;
    const int64_t maxc = [&] {
        int64_t m = 0;
        for (int c = 0; c < P.ncomp; ++c) m = std::max(m, P.comp_off[c + 1] - P.comp_off[c]);
        return m;
    }();
    const int nb = P.nblk;   // blocks per component for segmented reductions
    const dim3 gseg(nb, P.ncomp);
    const int eb = int(std::min<int64_t>((P.nflat + 255) / 256, 148 * 4));
    (void)maxc;
    k_prec_init<<<gseg, PB, 0, st>>>(P, r, s); ++nl;
    elim_solve(P, P.eM, P.rf, P.s, s, st, &nl);                                    // s = M^-1 r
    k_spmv_dot<<<gseg, PB, 0, st>>>(P, P.M, P.s, P.Mw, 0, 0, s); ++nl;            // ||s||_M
    k_lz_normalize<<<eb, 256, 0, st>>>(P, P.s, P.Mw, 0, s); ++nl;                  // q_1, v = M q_1
    for (int j = 1; j < P.kmax; ++j) {
        elim_solve(P, P.eK, P.v, P.w, s, st, &nl);                                 // w = K^-1 M q_j
        k_spmv_dot<<<gseg, PB, 0, st>>>(P, P.M, P.w, P.Mw, 1, j, s); ++nl;        // ||w||_M before
        for (int pass = 0; pass < 2; ++pass) {                                     // CGS2
            if (pass == 1) { k_spmv_dot<<<gseg, PB, 0, st>>>(P, P.M, P.w, P.Mw, -1, j, s); ++nl; }
            k_mdot_h<<<dim3(nb, j, P.ncomp), PB, 0, st>>>(P, P.Mw, s); ++nl;
            k_axpy_basis<<<eb, 256, 0, st>>>(P, P.w, s); ++nl;
        }
        k_spmv_dot<<<gseg, PB, 0, st>>>(P, P.M, P.w, P.Mw, 2, j, s); ++nl;        // ||w||_M after
        k_lz_normalize<<<eb, 256, 0, st>>>(P, P.w, P.Mw, j, s); ++nl;
    }
    k_spmv_multi<<<dim3(eb, P.kmax), 256, 0, st>>>(P, P.L, P.LW, s); ++nl;
    k_spmv_multi<<<dim3(eb, P.kmax), 256, 0, st>>>(P, P.M, P.MW, s); ++nl;
    const int ntask = P.kmax * (P.kmax + 1) + P.kmax;
    k_mdot_rr<<<dim3(nb, ntask, P.ncomp), PB, 0, st>>>(P, P.kmax, s); ++nl;
    k_lz_eig<<<1, 32, 0, st>>>(P, const_cast<PcgState*>(s)); ++nl;
    k_lz_combine<<<eb, 256, 0, st>>>(P, z, s); ++nl;
    if (nlaunch) *nlaunch = nl;
}

void prec_prepare(const PrecDev& P) {
    for (const ElimDev* E : {&P.eK, &P.eM}) {
        const int mf = E->maxface & 0xffff, mfac = E->maxface >> 16;
        const size_t smem = size_t(4) * (mf + mfac) * sizeof(double);
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(k_face_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    }
}

// ------------------------------------------------------------------ Gauss-Jordan SPD inverse (setup)
__global__ void k_gj_step(const double* __restrict__ A, double* __restrict__ Bo, int n, int k) {
    const int i = blockIdx.y;
    const double p = A[size_t(k) * n + k];
    const double aik = A[size_t(i) * n + k];
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const double akj = A[size_t(k) * n + j];
        double v;
        if (i == k) v = (j == k) ? 1.0 / p : akj / p;
        else v = (j == k) ? -aik / p : A[size_t(i) * n + j] - aik * akj / p;
        Bo[size_t(i) * n + j] = v;
    }
}

void launch_gauss_jordan(double* A, double* Bbuf, int n, cudaStream_t st) {
    double* src = A;
    double* dst = Bbuf;
    for (int k = 0; k < n; ++k) {
        dim3 grid((n + 255) / 256, n);
        k_gj_step<<<grid, 256, 0, st>>>(src, dst, n, k);
        std::swap(src, dst);
    }
    if (src != A) cudaMemcpyAsync(A, src, sizeof(double) * size_t(n) * n, cudaMemcpyDeviceToDevice, st);
}

}  // namespace de
