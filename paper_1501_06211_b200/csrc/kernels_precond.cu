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

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

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
// mode 0: y_F = X_FF^-1 b_F ; mode 1: x_F = X_FF^-1 (b_F - X_FC xC).
// Warp per face; both triangular solves are forward column sweeps (L, then M = P L^T P) with the
// b+1 active rows in registers (lane l holds row j+l; b <= 31), one shuffle per row on the chain.
__global__ void k_face_solve(ElimDev E, const double* __restrict__ b, const double* __restrict__ xC,
                             double* __restrict__ out, int mode, int per_warp, int mf, const PcgState* s) {
    if (s && s->done) return;
    extern __shared__ double fsh[];
    const int wpb = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int F = blockIdx.x * wpb + w;
    if (F >= E.nfaces) return;
    double* rb = fsh + size_t(w) * per_warp;
    double* ys = rb + mf;
    int* idx = reinterpret_cast<int*>(ys + mf);
    double* fs = ys + 2 * mf;                   // staged [L | M] factor of this face
    const int o = E.face_off[F], n = E.face_off[F + 1] - o, bw = E.face_band[F], ld = bw + 1;
    const double* gf = E.face_fac + E.face_fac_off[F];
    for (int i = lane; i < 2 * n * ld; i += 32) fs[i] = gf[i];
    const double* Lf = fs;
    const double* Mf = fs + size_t(n) * ld;
    for (int i = lane; i < n; i += 32) {
        const int node = E.face_nodes[o + i];
        idx[i] = node;
        double r = b[node];
        if (mode == 1)
            for (int e = E.xfc_ptr[o + i]; e < E.xfc_ptr[o + i + 1]; ++e) r -= E.xfc_val[e] * xC[E.xfc_col[e]];
        rb[i] = r;
    }
    __syncwarp();
#pragma unroll 1
    for (int sw = 0; sw < 2; ++sw) {
        const double* fac = sw == 0 ? Lf : Mf;
        const double* src = sw == 0 ? rb : ys;
        double* dst = sw == 0 ? ys : rb;
        double v = lane < n ? src[lane] : 0.0;   // ys already holds P y
        __syncwarp();
#pragma unroll 4
        for (int j = 0; j < n; ++j) {
            const double* col = fac + size_t(j) * ld;
            const double cl = (lane >= 1 && lane <= bw) ? col[lane] : 0.0;
            const double nxt = (j + 32 < n) ? src[j + 32] : 0.0;   // row entering lane 31 (uniform load)
            const double yj = __shfl_sync(0xffffffffu, v, 0) * col[0];
            v = fma(-cl, yj, v);
            const double vs = __shfl_down_sync(0xffffffffu, v, 1);
            v = (lane == 31) ? nxt : vs;                           // branch-free: keeps the warp converged
            dst[n - 1 - j] = yj;                                   // same value from every lane
        }
        __syncwarp();
    }
    for (int i = lane; i < n; i += 32) out[idx[i]] = rb[i];
}

static int face_warps_per_block(int per_warp_doubles) {
    const int bytes = per_warp_doubles * 8;
    int w = 4;
    while (w > 1 && w * bytes > 160 * 1024) --w;
    return w;
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

// ------------------------------------------------------------------ mode F: face-preconditioned inner PCG
// SPEC's inner solve of K x = b (R10), every component at
// once: textbook PCG from x0 = 0, preconditioner = K restricted to each face (cross points removed) solved
// exactly with the face band factors + Jacobi (diag K) at the cross points, stop when ||r||_2 <= tol ||b||_2
// (per component) or after maxit iterations. One cooperative kernel per solve, four grid barriers per
// iteration (p update | q = K p, p.q | x, r update, r.r | z = P r, r.z); per-component scalars are fixed-order
// sums of per-block partials that every block recomputes after the barrier (bitwise identical everywhere).
constexpr int FP_T = 256;

struct FpcgArgs {
    PrecDev P;
    const double* b;
    double* x;
    const PcgState* s;
};

// z_F = K_FF^-1 r_F for face F (warp; both band sweeps as in k_face_solve, factor read from global memory);
// returns this lane's share of r_F . z_F
__device__ double fp_face(const ElimDev& E, int F, const double* __restrict__ r, double* __restrict__ z,
                          double* rb, double* ys, int* idx, int lane) {
    const int o = E.face_off[F], n = E.face_off[F + 1] - o, bw = E.face_band[F], ld = bw + 1;
    const double* Lf = E.face_fac + E.face_fac_off[F];
    const double* Mf = Lf + size_t(n) * ld;
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
        const int node = E.face_nodes[o + i];
        idx[i] = node;
        rb[i] = r[node];
    }
    __syncwarp();
#pragma unroll 1
    for (int sw = 0; sw < 2; ++sw) {
        const double* fac = sw == 0 ? Lf : Mf;
        const double* src = sw == 0 ? rb : ys;   // the second sweep writes rb[n, 2n) (r_F stays for the dot)
        double v = lane < n ? src[lane] : 0.0;
        __syncwarp();
        for (int j = 0; j < n; ++j) {
            const double* col = fac + size_t(j) * ld;
            const double cl = (lane >= 1 && lane <= bw) ? col[lane] : 0.0;
            const double nxt = (j + 32 < n) ? src[j + 32] : 0.0;
            const double yj = __shfl_sync(0xffffffffu, v, 0) * col[0];
            v = fma(-cl, yj, v);
            const double vs = __shfl_down_sync(0xffffffffu, v, 1);
            v = (lane == 31) ? nxt : vs;
            if (sw == 0) ys[n - 1 - j] = yj;
            else if (lane == 0) rb[n + n - 1 - j] = yj;
        }
        __syncwarp();
    }
    double acc = 0.0;
    for (int i = lane; i < n; i += 32) {
        const double zi = rb[n + i];
        z[idx[i]] = zi;
        acc += rb[i] * zi;
    }
    return acc;
}

__device__ __forceinline__ double fp_diag(const CsrDev& K, int64_t i) {
    for (int e = K.ptr[i]; e < K.ptr[i + 1]; ++e)
        if (K.col[e] == i) return K.val[e];
    return 1.0;
}

// block partial of acc[0..nc) into part[(slot*MAXC + c)*nb + block]; fixed-order totals into tot[c]
__device__ void fp_reduce(const FpcgArgs& a, double (&acc)[MAXC], int slot, double* tot, double (*sred)[MAXC]) {
    const int nc = a.P.ncomp, lane = threadIdx.x & 31, w = threadIdx.x >> 5, nb = gridDim.x;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
        double t = acc[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) sred[w][c] = t;
    }
    __syncthreads();
    if (threadIdx.x < nc) {
        double t = 0.0;
        for (int k = 0; k < FP_T / 32; ++k) t += sred[k][threadIdx.x];
        a.P.fpart[(size_t(slot) * MAXC + threadIdx.x) * nb + blockIdx.x] = t;
    }
    __syncthreads();
    cg::this_grid().sync();
    if (w < nc) {
        const double* pp = a.P.fpart + (size_t(slot) * MAXC + w) * nb;
        double t = 0.0;
        for (int k = lane; k < nb; k += 32) t += *((volatile const double*)(pp + k));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) tot[w] = t;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(FP_T) k_face_pcg(FpcgArgs a) {
    if (a.s && a.s->done) return;
    const PrecDev& P = a.P;
    const ElimDev& E = P.eK;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double fsm[];
    __shared__ double sred[FP_T / 32][MAXC];
    __shared__ double tot[MAXC], nb2[MAXC], rz[MAXC], al[MAXC], be[MAXC];
    __shared__ int done[MAXC];
    const int nc = P.ncomp, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t n = P.nflat, gt = blockIdx.x * int64_t(FP_T) + threadIdx.x, gs = int64_t(gridDim.x) * FP_T;
    const int gw = blockIdx.x * (FP_T / 32) + w, nw = gridDim.x * (FP_T / 32);
    const int mf = E.maxface & 0xffff;
    double* rb = fsm + size_t(w) * (4 * mf);        // [0, n) r_F, [n, 2n) z_F
    double* ys = rb + 2 * mf;
    int* idx = reinterpret_cast<int*>(fsm + size_t(FP_T / 32) * 4 * mf) + w * mf;
    double* x = a.x;
    double *r = P.fr, *z = P.fz, *p = P.fp, *q = P.fq;
    double acc[MAXC];
    int slot = 0;
    // x = 0, r = b, ||b||^2
#pragma unroll
    for (int c = 0; c < MAXC; ++c) acc[c] = 0.0;
    for (int64_t i = gt; i < n; i += gs) {
        const double bi = a.b[i];
        x[i] = 0.0;
        r[i] = bi;
        acc[comp_of(P.comp_off, nc, i)] += bi * bi;
    }
    fp_reduce(a, acc, slot, tot, sred);
    slot ^= 1;
    if (threadIdx.x < MAXC) {
        nb2[threadIdx.x] = threadIdx.x < nc ? tot[threadIdx.x] : 0.0;
        done[threadIdx.x] = threadIdx.x < nc ? (tot[threadIdx.x] == 0.0) : 1;
    }
    __syncthreads();
    int it = 0;
    for (;;) {
        // z = P r (faces: warp each; cross points: Jacobi), r.z
#pragma unroll
        for (int c = 0; c < MAXC; ++c) acc[c] = 0.0;
        for (int F = gw; F < E.nfaces; F += nw) {
            const int c = comp_of(P.comp_off, nc, E.face_nodes[E.face_off[F]]);
            if (done[c]) continue;
            const double t = fp_face(E, F, r, z, rb, ys, idx, lane);
#pragma unroll
            for (int cc = 0; cc < MAXC; ++cc)
                if (cc == c) acc[cc] += t;
        }
        for (int64_t k = gt; k < E.ncross; k += gs) {
            const int64_t i = E.cross_flat[k];
            const int c = comp_of(P.comp_off, nc, i);
            if (done[c]) continue;
            const double zi = r[i] / fp_diag(P.K, i);
            z[i] = zi;
#pragma unroll
            for (int cc = 0; cc < MAXC; ++cc)
                if (cc == c) acc[cc] += r[i] * zi;
        }
        fp_reduce(a, acc, slot, tot, sred);
        slot ^= 1;
        if (threadIdx.x < nc && !done[threadIdx.x]) {
            be[threadIdx.x] = it == 0 ? 0.0 : tot[threadIdx.x] / rz[threadIdx.x];
            rz[threadIdx.x] = tot[threadIdx.x];
        }
        __syncthreads();
        ++it;
        // p = z + beta p
        for (int64_t i = gt; i < n; i += gs) {
            const int c = comp_of(P.comp_off, nc, i);
            if (!done[c]) p[i] = it == 1 ? z[i] : z[i] + be[c] * p[i];
        }
        grid.sync();
        // q = K p, p.q
#pragma unroll
        for (int c = 0; c < MAXC; ++c) acc[c] = 0.0;
        for (int64_t i = gt; i < n; i += gs) {
            const int c = comp_of(P.comp_off, nc, i);
            if (done[c]) continue;
            double t = 0.0;
            for (int e = P.K.ptr[i]; e < P.K.ptr[i + 1]; ++e) t += P.K.val[e] * p[P.K.col[e]];
            q[i] = t;
#pragma unroll
            for (int cc = 0; cc < MAXC; ++cc)
                if (cc == c) acc[cc] += p[i] * t;
        }
        fp_reduce(a, acc, slot, tot, sred);
        slot ^= 1;
        if (threadIdx.x < nc && !done[threadIdx.x]) al[threadIdx.x] = rz[threadIdx.x] / tot[threadIdx.x];
        __syncthreads();
        // x += alpha p, r -= alpha q, r.r
#pragma unroll
        for (int c = 0; c < MAXC; ++c) acc[c] = 0.0;
        for (int64_t i = gt; i < n; i += gs) {
            const int c = comp_of(P.comp_off, nc, i);
            if (done[c]) continue;
            x[i] += al[c] * p[i];
            const double ri = r[i] - al[c] * q[i];
            r[i] = ri;
#pragma unroll
            for (int cc = 0; cc < MAXC; ++cc)
                if (cc == c) acc[cc] += ri * ri;
        }
        fp_reduce(a, acc, slot, tot, sred);
        slot ^= 1;
        if (threadIdx.x < nc && !done[threadIdx.x]) {
            const double t = sqrt(tot[threadIdx.x]), bn = sqrt(nb2[threadIdx.x]);
            if (t <= P.fp_tol * bn || it >= P.fp_maxit) {
                done[threadIdx.x] = 1;
                if (blockIdx.x == 0) atomicAdd(P.fits, (unsigned long long)it);
            }
        }
        __syncthreads();
        bool all = true;
        for (int c = 0; c < nc; ++c) all = all && done[c];
        if (all) break;
    }
}

int fpcg_prepare(PrecDev& P, int device) {
    int nsm = 0, coop = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
    if (!coop) return 0;
    const int mf = std::max(1, P.eK.maxface & 0xffff);
    const size_t smem = size_t(FP_T / 32) * (4 * mf * sizeof(double) + mf * sizeof(int));
    if (smem > 200 * 1024) return 0;
    if (smem > 48 * 1024) raise_dyn_smem(reinterpret_cast<const void*>(k_face_pcg), smem);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_face_pcg, FP_T, smem) != cudaSuccess || per_sm < 1)
        return 0;
    P.fp_nb = nsm * std::min(per_sm, 2);
    P.fp_smem = smem;
    return P.fp_nb;
}

static void face_pcg_solve(const PrecDev& P, const double* b, double* x, const PcgState* s, cudaStream_t st,
                           int* nl) {
    FpcgArgs a{P, b, x, s};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(P.fp_nb);
    cfg.blockDim = dim3(FP_T);
    cfg.dynamicSmemBytes = P.fp_smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_face_pcg, a);
    ++*nl;
}

static void elim_solve(const PrecDev& P, const ElimDev& E, const double* b, double* x, const PcgState* s,
                       cudaStream_t st, int* nl) {
    const int mf = E.maxface & 0xffff, mfac = E.maxface >> 16;
    const int per_warp = 3 * mf + mfac;
    const int wpb = face_warps_per_block(per_warp);
    auto face = [&](const double* xc, double* o, int mode) {
        const int g = (E.nfaces + wpb - 1) / wpb;
        k_face_solve<<<g, 32 * wpb, size_t(wpb) * per_warp * sizeof(double), st>>>(E, b, xc, o, mode, per_warp, mf, s);
    };
    double* y = P.y;
    double* xC = P.y + P.nflat;   // cross solution scratch (ncross entries)
    if (E.nfaces > 0) {
        face(xC, y, 0);
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
        face(xC, x, 1);
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

// Rayleigh-Ritz Gram products G[i][jz] = W_i . Z_jz with Z = [LW_0..LW_{k-1} | MW_0..MW_{k-1} | rf]:
// per block a tile of TR rows of all 3k+1 vectors is staged in shared memory (each vector read
// once); one output per thread; per-block partials reduced in block order by the last block.
constexpr int TR = 64;
constexpr int RR_TASKS = KMAX * (2 * KMAX + 1);
__global__ void __launch_bounds__(512) k_mdot_rr(PrecDev P, const PcgState* s) {
    if (s && s->done) return;
    __shared__ double tile[(3 * KMAX + 1) * (TR + 1)];
    __shared__ bool last;
    const int c = blockIdx.y;
    const LzState& z = P.lz[c];
    if (!z.active) return;
    const int k = z.kc, nz = 2 * k + 1, nv = k + nz, nt = k * nz;
    const int64_t lo = P.comp_off[c], hi = P.comp_off[c + 1];
    const int tid = threadIdx.x;
    double acc0 = 0.0, acc1 = 0.0;
    for (int64_t r0 = lo + int64_t(blockIdx.x) * TR; r0 < hi; r0 += int64_t(gridDim.x) * TR) {
        for (int t = tid; t < nv * TR; t += blockDim.x) {
            const int v = t / TR, rr = t - v * TR;
            const int64_t r = r0 + rr;
            double val = 0.0;
            if (r < hi) {
                if (v < k) val = P.W[size_t(v) * P.nflat + r];
                else if (v < 2 * k) val = P.LW[size_t(v - k) * P.nflat + r];
                else if (v < 3 * k) val = P.MW[size_t(v - 2 * k) * P.nflat + r];
                else val = P.rf[r];
            }
            tile[v * (TR + 1) + rr] = val;
        }
        __syncthreads();
        for (int t = tid, h = 0; t < nt; t += blockDim.x, ++h) {
            const int i = t / nz, jz = t - i * nz;
            const double* a = tile + i * (TR + 1);
            const double* b = tile + (k + jz) * (TR + 1);
            double acc = 0.0;
#pragma unroll 8
            for (int rr = 0; rr < TR; ++rr) acc += a[rr] * b[rr];
            if (h == 0) acc0 += acc;
            else acc1 += acc;
        }
        __syncthreads();
    }
    const int nb = gridDim.x;
    const size_t base = size_t(8 + MAXC * KMAX + c * RR_TASKS);
    for (int t = tid, h = 0; t < nt; t += blockDim.x, ++h) P.part[(base + t) * nb + blockIdx.x] = h == 0 ? acc0 : acc1;
    __threadfence();
    __syncthreads();
    if (tid == 0) last = (atomicAdd(P.counter + base, 1u) == unsigned(nb - 1));
    __syncthreads();
    if (!last) return;
    __threadfence();
    LzState& zz = P.lz[c];
    for (int t = tid; t < nt; t += blockDim.x) {
        double sum = 0.0;
        for (int bx = 0; bx < nb; ++bx) sum += *((volatile double*)&P.part[(base + t) * nb + bx]);
        const int i = t / nz, jz = t - i * nz;
        if (jz < k) zz.A[i * KMAX + jz] = sum;
        else if (jz < 2 * k) zz.B[i * KMAX + (jz - k)] = sum;
        else zz.wr[i] = sum;
    }
    if (tid == 0) P.counter[base] = 0u;
}

// Small generalized symmetric eigenproblem A y = theta B y per component, one warp each:
// B = R R^T (Cholesky), C = R^-1 A R^-T, parallel (round-robin) Jacobi C = V Theta V^T,
// Y = R^-T V, coef = Y f(Theta) Y^T wr  (R9; SPEC.md:243-251 dense_sym_gen_eig).
__global__ void k_lz_eig(PrecDev P, PcgState* s) {
    if (s && s->done) return;
    constexpr int LDK = KMAX + 1;
    __shared__ double sm[MAXC][4][KMAX * LDK];
    __shared__ double rot[MAXC][2][KMAX / 2];
    __shared__ int rpq[MAXC][2][KMAX / 2];
    __shared__ double fe[MAXC][KMAX], ge[MAXC][KMAX];
    const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (c >= P.ncomp) return;
    LzState& z = P.lz[c];
    if (lane < KMAX) z.coef[lane] = 0.0;
    if (!z.active) return;
    const int n = z.kc;
    double* R = sm[c][0];
    double* C = sm[c][1];
    double* V = sm[c][2];
    double* X = sm[c][3];
    auto fail = [&]() {
        if (lane == 0) {
            z.status = DE_EBREAKDOWN;
            if (s) {
                s->status = DE_EBREAKDOWN;
                s->done = 1;
            }
        }
    };
    for (int idx = lane; idx < n * n; idx += 32) {
        const int i = idx / n, j = idx - i * n;
        C[i * LDK + j] = 0.5 * (z.A[i * KMAX + j] + z.A[j * KMAX + i]);
        R[i * LDK + j] = 0.5 * (z.B[i * KMAX + j] + z.B[j * KMAX + i]);
        V[i * LDK + j] = (i == j) ? 1.0 : 0.0;
    }
    __syncwarp();
    for (int j = 0; j < n; ++j) {                          // right-looking Cholesky, lower in R
        const double d = R[j * LDK + j];
        if (!(d > 0.0)) {
            fail();
            return;
        }
        const double l = sqrt(d);
        __syncwarp();
        if (lane == 0) R[j * LDK + j] = l;
        if (lane > j && lane < n) R[lane * LDK + j] /= l;
        __syncwarp();
        for (int idx = lane; idx < (n - j - 1) * (n - j - 1); idx += 32) {
            const int i = j + 1 + idx / (n - j - 1), kk = j + 1 + idx % (n - j - 1);
            if (kk <= i) R[i * LDK + kk] -= R[i * LDK + j] * R[kk * LDK + j];
        }
        __syncwarp();
    }
    if (lane < n) {                                         // X = R^-1 C (lane = column)
        for (int i = 0; i < n; ++i) {
            double t = C[i * LDK + lane];
            for (int kk = 0; kk < i; ++kk) t -= R[i * LDK + kk] * X[kk * LDK + lane];
            X[i * LDK + lane] = t / R[i * LDK + i];
        }
    }
    __syncwarp();
    if (lane < n) {                                         // C = X R^-T (lane = row)
        for (int i = 0; i < n; ++i) {
            double t = X[lane * LDK + i];
            for (int kk = 0; kk < i; ++kk) t -= C[lane * LDK + kk] * R[i * LDK + kk];
            C[lane * LDK + i] = t / R[i * LDK + i];
        }
    }
    __syncwarp();
    for (int idx = lane; idx < n * n; idx += 32) {          // symmetrise (read pairs once)
        const int i = idx / n, j = idx - i * n;
        if (j > i) {
            const double m = 0.5 * (C[i * LDK + j] + C[j * LDK + i]);
            C[i * LDK + j] = m;
            C[j * LDK + i] = m;
        }
    }
    __syncwarp();
    const int m = (n + 1) & ~1, npair = m / 2;
    for (int sweep = 0; sweep < 30 && n > 1; ++sweep) {
        double off = 0.0, dia = 0.0;
        if (lane < n)
            for (int j = 0; j < n; ++j) {
                const double v = C[lane * LDK + j];
                if (j == lane) dia += v * v;
                else off += v * v;
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            off += __shfl_xor_sync(0xffffffffu, off, o);
            dia += __shfl_xor_sync(0xffffffffu, dia, o);
        }
        if (off <= 1e-30 * dia) break;
        int rotated = 0;
        for (int rnd = 0; rnd < m - 1; ++rnd) {
            if (lane < npair) {                             // round-robin pairs (circle method)
                int p, q;
                if (lane == 0) {
                    p = m - 1;
                    q = rnd;
                } else {
                    p = (rnd + lane) % (m - 1);
                    q = (rnd - lane + (m - 1)) % (m - 1);
                }
                if (p > q) {
                    const int t = p;
                    p = q;
                    q = t;
                }
                double cs = 1.0, sn = 0.0;
                if (q < n) {
                    const double apq = C[p * LDK + q];
                    const double app = C[p * LDK + p], aqq = C[q * LDK + q];
                    (void)app;
                    (void)aqq;
                    if (fabs(apq) > 1e-15 * sqrt(dia) && fabs(apq) > 1e-300) {   // else negligible vs ||C||
                        rotated = 1;
                        const double tau = (C[q * LDK + q] - C[p * LDK + p]) / (2.0 * apq);
                        const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        cs = 1.0 / sqrt(1.0 + t * t);
                        sn = t * cs;
                    }
                }
                rot[c][0][lane] = cs;
                rot[c][1][lane] = sn;
                rpq[c][0][lane] = p;
                rpq[c][1][lane] = q;
            }
            __syncwarp();
            if (lane < n)                                   // C <- C J (columns), V <- V J
                for (int t = 0; t < npair; ++t) {
                    const int p = rpq[c][0][t], q = rpq[c][1][t];
                    if (q >= n) continue;
                    const double cs = rot[c][0][t], sn = rot[c][1][t];
                    const double a = C[lane * LDK + p], b = C[lane * LDK + q];
                    C[lane * LDK + p] = cs * a - sn * b;
                    C[lane * LDK + q] = sn * a + cs * b;
                    const double va = V[lane * LDK + p], vb = V[lane * LDK + q];
                    V[lane * LDK + p] = cs * va - sn * vb;
                    V[lane * LDK + q] = sn * va + cs * vb;
                }
            __syncwarp();
            if (lane < n)                                   // C <- J^T C (rows)
                for (int t = 0; t < npair; ++t) {
                    const int p = rpq[c][0][t], q = rpq[c][1][t];
                    if (q >= n) continue;
                    const double cs = rot[c][0][t], sn = rot[c][1][t];
                    const double a = C[p * LDK + lane], b = C[q * LDK + lane];
                    C[p * LDK + lane] = cs * a - sn * b;
                    C[q * LDK + lane] = sn * a + cs * b;
                }
            __syncwarp();
        }
        if (!__any_sync(0xffffffffu, rotated)) break;   // every pair below threshold: converged
    }
    const bool sing = P.singular[c] != 0;
    int bad = 0;
    if (lane < n) {
        const double th = C[lane * LDK + lane];
        z.theta_ritz[lane] = th;
        if (!sing && !(th > 0.0)) bad = 1;
        fe[c][lane] = sing ? 1.0 / (1.0 + pow(fmax(th, 0.0), 1.0 - P.theta)) : pow(th, P.theta - 1.0);
        for (int i = n - 1; i >= 0; --i) {                  // Y(:,e) = R^-T V(:,e), lane = e
            double t = V[i * LDK + lane];
            for (int kk = i + 1; kk < n; ++kk) t -= R[kk * LDK + i] * X[kk * LDK + lane];
            X[i * LDK + lane] = t / R[i * LDK + i];
        }
        double t = 0.0;
        for (int i = 0; i < n; ++i) t += X[i * LDK + lane] * z.wr[i];
        ge[c][lane] = fe[c][lane] * t;
    }
    if (__any_sync(0xffffffffu, bad)) {
        fail();
        return;
    }
    __syncwarp();
    if (lane < n) {
        double t = 0.0;
        for (int e = 0; e < n; ++e) t += X[lane * LDK + e] * ge[c][e];
        z.coef[lane] = t;
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
        if (P.inner_f) face_pcg_solve(P, P.v, P.w, s, st, &nl);                   // w ~ K^-1 M q_j (mode F)
        else elim_solve(P, P.eK, P.v, P.w, s, st, &nl);                            // w = K^-1 M q_j
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
    k_mdot_rr<<<dim3(nb, P.ncomp), 512, 0, st>>>(P, s); ++nl;
    k_lz_eig<<<1, 32 * P.ncomp, 0, st>>>(P, const_cast<PcgState*>(s)); ++nl;
    k_lz_combine<<<eb, 256, 0, st>>>(P, z, s); ++nl;
    if (nlaunch) *nlaunch = nl;
}

void prec_prepare(const PrecDev& P) {
    int mx = 0;
    for (const ElimDev* E : {&P.eK, &P.eM}) {
        const int per_warp = 3 * (E->maxface & 0xffff) + (E->maxface >> 16);
        mx = std::max(mx, face_warps_per_block(per_warp) * per_warp * 8);
    }
    if (mx > 48 * 1024) raise_dyn_smem(reinterpret_cast<const void*>(k_face_solve), size_t(mx));
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
