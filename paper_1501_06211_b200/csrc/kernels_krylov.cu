// kernels_krylov.cu — SURVEY.md §8(a) rows C3 (interface assembly q = sum_s R_s^T q_s) and C4
// (PCG vector updates and dot products), R11:
//   alpha = (r.z)/(p.q); x += alpha p; r -= alpha q; stop if ||r|| <= rtol ||f_free||;
//   beta = (r'.z')/(r.z) (Fletcher-Reeves) or z'.(r'-r)/(r.z) (Polak-Ribiere); p = z + beta p.
// Scalars live on the device (PcgState); each reduction is a fixed-shape two-level tree (block
// partials, then the last block to finish sums the partials in index order), so results are
// bitwise reproducible. Every kernel returns immediately once state->done is set, which lets the
// host launch several captured iterations between convergence polls.
#include "de_internal.h"

namespace de {

constexpr int RB = 256;   // threads per reduction block

__device__ __forceinline__ double block_sum(double v, double* sh) {
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
    return r;   // valid in thread 0
}

// Writes the block partial(s); returns true in thread 0 of the last block, with the totals in tot[].
template <int ND>
__device__ __forceinline__ bool grid_reduce(const double (&v)[ND], double (&tot)[ND], RedBuf rb) {
    __shared__ double sh[32];
    __shared__ bool last;
    double bs[ND];
#pragma unroll
    for (int i = 0; i < ND; ++i) bs[i] = block_sum(v[i], sh);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < ND; ++i) rb.part[blockIdx.x * ND + i] = bs[i];
        __threadfence();
        const unsigned int ticket = atomicAdd(rb.counter, 1u);
        last = (ticket == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return false;
    __threadfence();
    double acc[ND];
#pragma unroll
    for (int i = 0; i < ND; ++i) acc[i] = 0.0;
    for (int b = threadIdx.x; b < int(gridDim.x); b += blockDim.x)
#pragma unroll
        for (int i = 0; i < ND; ++i) acc[i] += *((volatile double*)&rb.part[b * ND + i]);
#pragma unroll
    for (int i = 0; i < ND; ++i) tot[i] = block_sum(acc[i], sh);
    if (threadIdx.x == 0) *rb.counter = 0u;
    return threadIdx.x == 0;
}

static int red_blocks(int64_t n, const RedBuf& rb) {
    return int(std::max<int64_t>(1, std::min<int64_t>((n + RB - 1) / RB, rb.nblk)));
}

__global__ void k_gather(const int32_t* __restrict__ gptr, const int32_t* __restrict__ gsrc,
                         const double* __restrict__ qloc, const double* __restrict__ add,
                         double* __restrict__ q, int64_t nG, const PcgState* s) {
    if (s != nullptr && s->done) return;
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < nG; g += int64_t(gridDim.x) * blockDim.x) {
        double acc = add ? add[g] : 0.0;
        for (int k = gptr[g]; k < gptr[g + 1]; ++k) acc += qloc[gsrc[k]];
        q[g] = acc;
    }
}

void launch_gather(const int32_t* gptr, const int32_t* gsrc, const double* qloc, const double* add,
                   double* q, int64_t nG, const PcgState* s, cudaStream_t st) {
    const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((nG + 255) / 256, 148 * 8)));
    k_gather<<<blocks, 256, 0, st>>>(gptr, gsrc, qloc, add, q, nG, s);
}

// p.q  -> alpha = rz / pq  (breakdown if pq <= 0)
__global__ void k_pcg_pq(const double* __restrict__ p, const double* __restrict__ q, int64_t n, RedBuf rb,
                         PcgState* s) {
    if (s->done) return;
    double v[1] = {0.0}, tot[1];
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        v[0] += p[i] * q[i];
    if (grid_reduce<1>(v, tot, rb)) {
        s->pq = tot[0];
        if (!(tot[0] > 0.0)) {
            s->status = DE_EBREAKDOWN;
            s->done = 1;
        } else {
            s->alpha = s->rz / tot[0];
        }
    }
}

void launch_pcg_pq(const double* p, const double* q, int64_t n, RedBuf rb, PcgState* s, cudaStream_t st) {
    k_pcg_pq<<<red_blocks(n, rb), RB, 0, st>>>(p, q, n, rb, s);
}

// single rank: q = sum of the local contributions (k_gather) and p.q in one pass (k_pcg_pq's reduction and tail)
__global__ void k_gather_pq(const int32_t* __restrict__ gptr, const int32_t* __restrict__ gsrc,
                            const double* __restrict__ qloc, const double* __restrict__ p, double* __restrict__ q,
                            int64_t n, RedBuf rb, PcgState* s) {
    if (s->done) return;
    double v[1] = {0.0}, tot[1];
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < n; g += int64_t(gridDim.x) * blockDim.x) {
        double acc = 0.0;
        for (int k = gptr[g]; k < gptr[g + 1]; ++k) acc += qloc[gsrc[k]];
        q[g] = acc;
        v[0] += p[g] * acc;
    }
    if (grid_reduce<1>(v, tot, rb)) {
        s->pq = tot[0];
        if (!(tot[0] > 0.0)) {
            s->status = DE_EBREAKDOWN;
            s->done = 1;
        } else {
            s->alpha = s->rz / tot[0];
        }
    }
}

void launch_gather_pq(const int32_t* gptr, const int32_t* gsrc, const double* qloc, const double* p, double* q,
                      int64_t n, RedBuf rb, PcgState* s, cudaStream_t st) {
    k_gather_pq<<<red_blocks(n, rb), RB, 0, st>>>(gptr, gsrc, qloc, p, q, n, rb, s);
}

// x += alpha p; r -= alpha q; ||r||^2 -> convergence / iteration cap
__global__ void k_pcg_update_xr(double* __restrict__ x, double* __restrict__ r, double* __restrict__ r_old,
                                const double* __restrict__ p, const double* __restrict__ q, int64_t n,
                                RedBuf rb, PcgState* s) {
    if (s->done) return;
    const double al = s->alpha;
    double v[1] = {0.0}, tot[1];
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        x[i] += al * p[i];
        const double ri = r[i];
        if (r_old) r_old[i] = ri;
        const double rn = ri - al * q[i];
        r[i] = rn;
        v[0] += rn * rn;
    }
    if (grid_reduce<1>(v, tot, rb)) {
        s->rr = tot[0];
        s->it += 1;
        if (tot[0] <= s->tol2) s->done = 1;
        else if (s->it >= s->maxit) {
            s->done = 1;
            s->status = DE_ENOCONV;
        } else if (!(tot[0] == tot[0])) {
            s->done = 1;
            s->status = DE_EBREAKDOWN;
        }
    }
}

void launch_pcg_update_xr(double* x, double* r, double* r_old, const double* p, const double* q, int64_t n,
                          RedBuf rb, PcgState* s, cudaStream_t st) {
    k_pcg_update_xr<<<red_blocks(n, rb), RB, 0, st>>>(x, r, r_old, p, q, n, rb, s);
}

// r.z (and z.r_old for Polak-Ribiere) -> beta, rz
__global__ void k_pcg_rz(const double* __restrict__ r, const double* __restrict__ z, const double* __restrict__ r_old,
                         int64_t n, int pr, RedBuf rb, PcgState* s) {
    if (s->done) return;
    double v[2] = {0.0, 0.0}, tot[2];
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        v[0] += r[i] * z[i];
        if (pr) v[1] += z[i] * r_old[i];
    }
    if (grid_reduce<2>(v, tot, rb)) {
        const double rz_new = tot[0];
        s->beta = pr ? (rz_new - tot[1]) / s->rz : rz_new / s->rz;
        s->rz = rz_new;
    }
}

void launch_pcg_rz(const double* r, const double* z, const double* r_old, int64_t n, int beta_pr, RedBuf rb,
                   PcgState* s, cudaStream_t st) {
    k_pcg_rz<<<red_blocks(n, rb), RB, 0, st>>>(r, z, r_old, n, beta_pr, rb, s);
}

__global__ void k_pcg_update_p(double* __restrict__ p, const double* __restrict__ z, int64_t n, PcgState* s) {
    if (s->done) return;
    const double b = s->beta;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        p[i] = z[i] + b * p[i];
}

void launch_pcg_update_p(double* p, const double* z, int64_t n, PcgState* s, cudaStream_t st) {
    const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)));
    k_pcg_update_p<<<blocks, 256, 0, st>>>(p, z, n, s);
}

// mode 0: r = g (x0 = 0);  mode 1: r = g - Sx;  then rr = r.r; done if rr <= tol2
// mode 2: p = z; rz = r.z
__global__ void k_pcg_init(double* __restrict__ r, double* __restrict__ p, const double* __restrict__ z,
                           const double* __restrict__ g, const double* __restrict__ Sx, int64_t n, int mode,
                           RedBuf rb, PcgState* s) {
    double v[1] = {0.0}, tot[1];
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        if (mode == 2) {
            p[i] = z[i];
            v[0] += r[i] * z[i];
        } else {
            const double ri = mode == 1 ? g[i] - Sx[i] : g[i];
            r[i] = ri;
            v[0] += ri * ri;
        }
    }
    if (grid_reduce<1>(v, tot, rb)) {
        if (mode == 2) {
            s->rz = tot[0];
        } else {
            s->rr = tot[0];
            s->done = tot[0] <= s->tol2 ? 1 : 0;
        }
    }
}

void launch_pcg_init(double* r, double* p, const double* z, const double* g, const double* Sx, int64_t n,
                     int mode, RedBuf rb, PcgState* s, cudaStream_t st) {
    k_pcg_init<<<red_blocks(n, rb), RB, 0, st>>>(r, p, z, g, Sx, n, mode, rb, s);
}

__global__ void k_norm2(const double* __restrict__ v_, int64_t n, RedBuf rb, double* out) {
    double v[1] = {0.0}, tot[1];
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        v[0] += v_[i] * v_[i];
    if (grid_reduce<1>(v, tot, rb)) *out = tot[0];
}

void launch_norm2(const double* v, int64_t n, RedBuf rb, double* out, cudaStream_t st) {
    k_norm2<<<red_blocks(n, rb), RB, 0, st>>>(v, n, rb, out);
}

// ---------------------------------------------------------------- full-system FGMRES (NEXT(4)) helpers
// out[i] = V_i . w for i < nv (nv <= FG_ND), V_i = V + i * ld; one fixed-order reduction (rb.part >= nblk*FG_ND)
__global__ void k_multidot(const double* __restrict__ V, int64_t ld, int nv, const double* __restrict__ w, int64_t n,
                           RedBuf rb, double* __restrict__ out) {
    double v[FG_ND], tot[FG_ND];
#pragma unroll
    for (int i = 0; i < FG_ND; ++i) v[i] = 0.0;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const double wk = w[k];
#pragma unroll
        for (int i = 0; i < FG_ND; ++i)
            if (i < nv) v[i] = fma(V[i * ld + k], wk, v[i]);
    }
    if (grid_reduce<FG_ND>(v, tot, rb))
        for (int i = 0; i < nv; ++i) out[i] = tot[i];
}

// w += sign * sum_{i < nv} coef[i] V_i (coef on the device)
__global__ void k_multi_axpy(double* __restrict__ w, const double* __restrict__ V, int64_t ld, int nv,
                             const double* __restrict__ coef, double sign, int64_t n) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        double acc = 0.0;
        for (int i = 0; i < nv; ++i) acc = fma(coef[i], V[i * ld + k], acc);
        w[k] = fma(sign, acc, w[k]);
    }
}

// dst = src / sqrt(*sq) (sq = squared norm on the device; dst = 0 when it is 0)
__global__ void k_scale_invnorm(double* __restrict__ dst, const double* __restrict__ src, const double* sq, int64_t n) {
    const double s = *sq > 0.0 ? 1.0 / sqrt(*sq) : 0.0;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x)
        dst[k] = src[k] * s;
}

void launch_multidot(const double* V, int64_t ld, int nv, const double* w, int64_t n, RedBuf rb, double* out,
                     cudaStream_t st) {
    k_multidot<<<red_blocks(n, rb), RB, 0, st>>>(V, ld, nv, w, n, rb, out);
}
void launch_multi_axpy(double* w, const double* V, int64_t ld, int nv, const double* coef, double sign, int64_t n,
                       cudaStream_t st) {
    k_multi_axpy<<<int(std::min<int64_t>((n + 255) / 256, 148 * 8)), 256, 0, st>>>(w, V, ld, nv, coef, sign, n);
}
void launch_scale_invnorm(double* dst, const double* src, const double* sq, int64_t n, cudaStream_t st) {
    k_scale_invnorm<<<int(std::min<int64_t>((n + 255) / 256, 148 * 8)), 256, 0, st>>>(dst, src, sq, n);
}

__global__ void k_copy(double* __restrict__ dst, const double* __restrict__ src, int64_t n, const PcgState* s) {
    if (s != nullptr && s->done) return;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        dst[i] = src[i];
}

void launch_copy(double* dst, const double* src, int64_t n, const PcgState* s, cudaStream_t st) {
    const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)));
    k_copy<<<blocks, 256, 0, st>>>(dst, src, n, s);
}

// buf = sum_{r < n} slots[r] in rank order (the loopback all-reduce: the same fixed order on every rank)
__global__ void k_sum_slots(double* __restrict__ buf, const double* __restrict__ slots, int n, size_t cap,
                            int64_t len) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < len; i += int64_t(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < n; ++r) s += slots[size_t(r) * cap + i];
        buf[i] = s;
    }
}

void launch_sum_slots(double* buf, const double* slots, int n, size_t cap, int64_t len, cudaStream_t st) {
    const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((len + 255) / 256, 148 * 8)));
    k_sum_slots<<<blocks, 256, 0, st>>>(buf, slots, n, cap, len);
}

__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ x, double a, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        y[i] += a * x[i];
}

void launch_axpy(double* y, const double* x, double a, int64_t n, cudaStream_t st) {
    const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)));
    k_axpy<<<blocks, 256, 0, st>>>(y, x, a, n);
}

__global__ void k_scatter_gamma(const int32_t* __restrict__ gd, const double* __restrict__ uG, double* __restrict__ u,
                                int64_t nG) {
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < nG; g += int64_t(gridDim.x) * blockDim.x)
        u[gd[g]] = uG[g];
}

void launch_scatter_gamma(const int32_t* gamma_dofs, const double* uG, double* u, int64_t nG, cudaStream_t st) {
    if (nG == 0) return;
    const int blocks = int(std::min<int64_t>((nG + 255) / 256, 148 * 8));
    k_scatter_gamma<<<blocks, 256, 0, st>>>(gamma_dofs, uG, u, nG);
}

__global__ void k_gather_gamma(const int32_t* __restrict__ gd, const double* __restrict__ f, double* __restrict__ fG,
                               int64_t nG) {
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < nG; g += int64_t(gridDim.x) * blockDim.x)
        fG[g] = f[gd[g]];
}

void launch_gather_gamma(const int32_t* gamma_dofs, const double* f, double* fG, int64_t nG, cudaStream_t st) {
    if (nG == 0) return;
    const int blocks = int(std::min<int64_t>((nG + 255) / 256, 148 * 8));
    k_gather_gamma<<<blocks, 256, 0, st>>>(gamma_dofs, f, fG, nG);
}

__global__ void k_zero_dirichlet(const int8_t* __restrict__ cls, double* __restrict__ u, int64_t ndof) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < ndof; i += int64_t(gridDim.x) * blockDim.x)
        if (cls[i] == 2) u[i] = 0.0;
}

void launch_zero_dirichlet(const int8_t* cls, double* u, int64_t ndof, cudaStream_t st) {
    const int blocks = int(std::min<int64_t>((ndof + 255) / 256, 148 * 8));
    k_zero_dirichlet<<<blocks, 256, 0, st>>>(cls, u, ndof);
}

}  // namespace de
