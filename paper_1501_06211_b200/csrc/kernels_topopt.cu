// kernels_topopt.cu — SURVEY.md §8(f) NEXT(4), second half: the design update of the topology-optimisation
// loop the paper's solver serves (minimum compliance, densities updated between solves).
// The paper states no OC constants; R20 fixes the standard optimality-criteria step:
//   dc_e   = -p rho_e^(p-1) (E0 - Emin) u_e^T KE0 u_e,   c = sum_e E_e u_e^T KE0 u_e
//   rho_e' = clip(rho_e (max(-dc_e, 0) / lambda)^eta, max(rho_min, rho_e - move), min(1, rho_e + move))
//   lambda: bisection on [0, 1e9 max_e(-dc_e)] until l2 - l1 <= tol (l1 + l2), sum_e rho_e' = V n_elem.
// HBM-bound elementwise work: one thread per element, u gathered through L2 (each node is shared by 2^dim
// elements), block partial sums reduced in a fixed order by one block (deterministic). The bisection keeps
// lambda on the device (OcState), so the whole update is a launch sequence without host round trips.
#include "de_internal.h"

namespace de {

// Own copy of the unit-modulus element stiffness (no relocatable device code across translation units).
__constant__ double c_KE_oc[24 * 24];

void upload_KE0_oc(const double* ke, int nke, cudaStream_t st) {
    cudaMemcpyToSymbolAsync(c_KE_oc, ke, sizeof(double) * nke * nke, 0, cudaMemcpyHostToDevice, st);
}

constexpr int OC_T = 256;

// Block reduction of non-negative values (sum or max); the result is valid in warp 0.
template <typename Op>
__device__ __forceinline__ double block_sum_oc(double v, double* sh, Op op) {
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        v = l < (OC_T >> 5) ? sh[l] : 0.0;   // 0 is the identity of both reductions (all values are >= 0)
        for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    }
    __syncthreads();
    return v;
}

struct SumOp { __device__ double operator()(double a, double b) const { return a + b; } };
struct MaxOp { __device__ double operator()(double a, double b) const { return fmax(a, b); } };

// part[2 b] = sum of E_e en_e over the block's elements, part[2 b + 1] = max of -dc_e.
template <int DIM>
__global__ void __launch_bounds__(OC_T) k_elem_sens(MeshDev m, const double* __restrict__ u,
                                                    const double* __restrict__ rho, const double* __restrict__ Ee,
                                                    double dEdrho_scale, double p, int64_t nelem,
                                                    double* __restrict__ dc, double* __restrict__ part) {
    __shared__ double sh[OC_T / 32];
    constexpr int dim = DIM, nv = 1 << DIM, nke = DIM << DIM;
    double csum = 0.0, gmax = 0.0;
    for (int64_t e = blockIdx.x * int64_t(OC_T) + threadIdx.x; e < nelem; e += int64_t(gridDim.x) * OC_T) {
        const int ex = int(e % m.nel[0]);
        const int64_t r = e / m.nel[0];
        const int ey = int(r % m.nel[1]);
        const int ez = int(r / m.nel[1]);
        double ue[nke];
#pragma unroll
        for (int l = 0; l < nv; ++l) {
            const int64_t node = (ex + (l & 1)) + int64_t(m.nn[0]) *
                                 ((ey + ((l >> 1) & 1)) + int64_t(m.nn[1]) * (ez + ((l >> 2) & 1)));
#pragma unroll
            for (int c = 0; c < dim; ++c) ue[dim * l + c] = u[dim * node + c];
        }
        double en = 0.0;
#pragma unroll
        for (int i = 0; i < nke; ++i) {
            double t = 0.0;
#pragma unroll
            for (int j = 0; j < nke; ++j) t += c_KE_oc[i * nke + j] * ue[j];
            en += ue[i] * t;
        }
        const double rh = rho[e];
        const double d = -p * (p == 1.0 ? 1.0 : pow(rh, p - 1.0)) * dEdrho_scale * en;
        dc[e] = d;
        csum += Ee[e] * en;
        gmax = fmax(gmax, -d);
    }
    csum = block_sum_oc(csum, sh, SumOp());
    gmax = block_sum_oc(gmax, sh, MaxOp());
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = csum;
        part[2 * blockIdx.x + 1] = gmax;
    }
}

// One block: fixed-order reduction of the partials; initialises the bisection state.
__global__ void k_sens_finish(const double* __restrict__ part, int nb, OcState* st) {
    __shared__ double sh[OC_T / 32];
    double s = 0.0, g = 0.0;
    for (int b = threadIdx.x; b < nb; b += OC_T) {
        s += part[2 * b];
        g = fmax(g, part[2 * b + 1]);
    }
    s = block_sum_oc(s, sh, SumOp());
    g = block_sum_oc(g, sh, MaxOp());
    if (threadIdx.x == 0) {
        st->compliance = s;
        st->l1 = 0.0;
        st->l2 = fmax(g, 1e-300) * 1e9;
        st->it = 0;
        st->done = 0;
    }
}

__device__ __forceinline__ double oc_new(double rh, double dce, double lm, double move, double rho_min,
                                         double eta) {
    const double q = fmax(-dce, 0.0) / lm;
    const double b = eta == 0.5 ? sqrt(q) : pow(q, eta);
    return fmin(fmax(rh * b, fmax(rho_min, rh - move)), fmin(1.0, rh + move));
}

// Sum of the trial densities at lambda = (l1 + l2)/2 (block partials); no-op once converged.
__global__ void __launch_bounds__(OC_T) k_oc_sum(const double* __restrict__ rho, const double* __restrict__ dc,
                                                 int64_t n, OcParams prm, const OcState* __restrict__ st,
                                                 double* __restrict__ part) {
    __shared__ double sh[OC_T / 32];
    if (st->done) return;
    const double lm = 0.5 * (st->l1 + st->l2);
    double s = 0.0;
    for (int64_t e = blockIdx.x * int64_t(OC_T) + threadIdx.x; e < n; e += int64_t(gridDim.x) * OC_T)
        s += oc_new(rho[e], dc[e], lm, prm.move, prm.rho_min, prm.eta);
    s = block_sum_oc(s, sh, SumOp());
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_oc_decide(const double* __restrict__ part, int nb, OcParams prm, double target, OcState* st) {
    __shared__ double sh[OC_T / 32];
    if (st->done) return;
    double s = 0.0;
    for (int b = threadIdx.x; b < nb; b += OC_T) s += part[b];
    s = block_sum_oc(s, sh, SumOp());
    if (threadIdx.x == 0) {
        const double lm = 0.5 * (st->l1 + st->l2);
        if (s > target) st->l1 = lm;
        else st->l2 = lm;
        st->it += 1;
        if (st->l2 - st->l1 <= prm.tol * (st->l1 + st->l2) || st->it >= prm.maxit) st->done = 1;
        st->lambda = 0.5 * (st->l1 + st->l2);
    }
}

__global__ void k_oc_apply(const double* __restrict__ rho, const double* __restrict__ dc, int64_t n, OcParams prm,
                           const OcState* __restrict__ st, double* __restrict__ rho_new) {
    const double lm = st->lambda;
    for (int64_t e = blockIdx.x * int64_t(OC_T) + threadIdx.x; e < n; e += int64_t(gridDim.x) * OC_T)
        rho_new[e] = oc_new(rho[e], dc[e], lm, prm.move, prm.rho_min, prm.eta);
}

int oc_blocks(int64_t n) { return int(std::min<int64_t>((n + OC_T - 1) / OC_T, 148 * 8)); }

int launch_sensitivities(const MeshDev& m, const double* u, const double* rho, const double* Ee, double E0,
                         double Emin, double p, int64_t nelem, double* dc, double* part, OcState* st,
                         cudaStream_t s) {
    const int nb = oc_blocks(nelem);
    if (m.dim == 2) k_elem_sens<2><<<nb, OC_T, 0, s>>>(m, u, rho, Ee, E0 - Emin, p, nelem, dc, part);
    else k_elem_sens<3><<<nb, OC_T, 0, s>>>(m, u, rho, Ee, E0 - Emin, p, nelem, dc, part);
    k_sens_finish<<<1, OC_T, 0, s>>>(part, nb, st);
    return 2;
}

int launch_oc_update(const double* rho, const double* dc, int64_t n, const OcParams& prm, double* part,
                     OcState* st, double* rho_new, cudaStream_t s) {
    const int nb = oc_blocks(n);
    const double target = prm.volfrac * double(n);
    for (int i = 0; i < prm.maxit; ++i) {
        k_oc_sum<<<nb, OC_T, 0, s>>>(rho, dc, n, prm, st, part);
        k_oc_decide<<<1, OC_T, 0, s>>>(part, nb, prm, target, st);
    }
    k_oc_apply<<<nb, OC_T, 0, s>>>(rho, dc, n, prm, st, rho_new);
    return 2 * prm.maxit + 1;
}

}  // namespace de
