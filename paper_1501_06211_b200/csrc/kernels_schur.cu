// kernels_schur.cu — SURVEY.md §8(a) rows C1 (condensed rhs), C2 (Schur apply, the headline kernel)
// and C6 (back-substitution): per owned subdomain s
//
//   C2 (SCHUR_APPLY):   x = R_s p;  y = A_IG x;  w = A_II^-1 y;  q_s = A_GG x - A_GI w
//   C1 (SCHUR_CONDENSE): w = A_II^-1 f_I;  q_s = -A_GI w     (g = f_G + sum_s R_s^T q_s)
//   C6 (SCHUR_BACKSUB):  w = A_II^-1 (f_I - A_IG R_s u_G);  u_I = w   (PAPER.md:141,143 combined, :136)
//
// One warp per subdomain (one-warp CTAs, ~14 resident per SM at 2D sizes). The interior solve
// w = L^-T L^-1 y streams the column-band factor twice (forward ascending, backward descending)
// through a ring of shared-memory stages filled by TMA bulk copies (cp.async.bulk + mbarrier
// complete_tx) issued by lane 0; the ring is shared by both sweeps so the backward sweep's first
// stages (the columns the forward sweep read last) are prefetched while the forward sweep finishes
// and come back from L2.
//   forward  (column axpy): y_j = t_j / L_jj; t_{j+k} -= L_{j+k,j} y_j   (window of b+1 rows in smem)
//   backward (blocks of G columns, lane groups own a column): t_j = y_j - sum_{i>block} L_ij x_i,
//            then a G-step chain inside the block.
#include "de_internal.h"

namespace de {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    const long long t0 = clock64();
    while (!ok) {
        if (clock64() - t0 > (1ll << 35)) __trap();   // never hang the GPU on a lost transaction
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

struct Ring {
    uint64_t* bar;
    double* stg;
    int nstage, G, ld, n, nfw;   // nfw = forward stage count (same for backward)
    const double* L;

    // stage T of the unified ring: T < nfw forward stage T, else backward stage T - nfw
    __device__ __forceinline__ void cols(int T, int& c0, int& nc) const {
        if (T < nfw) {
            c0 = T * G;
            nc = min(G, n - c0);
        } else {
            const int u = T - nfw;
            const int hi = n - u * G;
            c0 = max(0, hi - G);
            nc = hi - c0;
        }
    }
    __device__ __forceinline__ void issue(int T) const {   // lane 0 only
        int c0, nc;
        cols(T, c0, nc);
        const int slot = T % nstage;
        const uint32_t bytes = uint32_t(nc) * uint32_t(ld) * 8u;
        mbar_expect_tx(bar + slot, bytes);
        tma_load_1d(stg + size_t(slot) * G * ld, L + size_t(c0) * ld, bytes, bar + slot);
    }
    __device__ __forceinline__ const double* wait(int T) const {
        const int slot = T % nstage;
        mbar_wait(bar + slot, uint32_t((T / nstage) & 1));
        return stg + size_t(slot) * G * ld;
    }
};

template <int G>
__global__ void __launch_bounds__(32) k_schur_local(SchurArgs a, int nstage, int win) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (a.state != nullptr && a.state->done) return;
    const int lane = threadIdx.x;
    const SubDesc d = a.sd[blockIdx.x];
    const int n = d.nI, nG = d.nG, B = a.band_w, ld = a.ld;
    const int mode = a.mode;
    const int wmask = win - 1;

    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    double* stg = reinterpret_cast<double*>(smem + 128);
    double* wn = stg + size_t(nstage) * G * ld;
    double* xl = wn + win;
    double* y = a.scratch + d.ioff;     // forward solution, then w

    Ring ring{bar, stg, nstage, G, ld, n, (n + G - 1) / G, a.band + d.band_off};
    const int ntot = 2 * ring.nfw;
    if (lane == 0) {
        for (int i = 0; i < nstage; ++i) mbar_init(bar + i, 1);
        fence_mbar_init();
        for (int T = 0; T < min(nstage, ntot); ++T) ring.issue(T);
    }
    // gather x_s = R_s p (or u_Gamma) into shared memory
    if (mode != SCHUR_CONDENSE)
        for (int l = lane; l < nG; l += 32) xl[l] = a.xin[a.Rg[d.goff + l]];
    __syncwarp();

    const int32_t* igp = a.igp + d.igp_off;
    const int32_t* idofs = a.idofs + d.ioff;
    auto rhs = [&](int r) -> double {
        double v = (mode == SCHUR_APPLY) ? 0.0 : a.f[idofs[r]];
        if (mode != SCHUR_CONDENSE) {
            double acc = 0.0;
            for (int e = igp[r]; e < igp[r + 1]; ++e) acc += a.ig_val[e] * xl[a.ig_col[e]];
            v = (mode == SCHUR_APPLY) ? acc : v - acc;
        }
        return v;
    };

    // ------------------------------------------------------------------ forward sweep
    for (int r = lane; r <= B && r < n; r += 32) wn[r & wmask] = rhs(r);
    // rows entering at stage t are c0+B+1 .. c0+B+nc; prefetch them one stage ahead
    double pend = 0.0;
    if (lane < G) {
        const int r = B + 1 + lane;
        if (r < n) pend = rhs(r);
    }
    __syncwarp();
    int T = 0;
    for (int t = 0; t < ring.nfw; ++t, ++T) {
        const double* S = ring.wait(T);
        const int c0 = t * G, nc = min(G, n - c0);
        if (lane < nc) {
            const int r = c0 + B + 1 + lane;
            if (r < n) wn[r & wmask] = pend;
        }
        if (lane < G) {
            const int r = c0 + G + B + 1 + lane;
            pend = (r < n) ? rhs(r) : 0.0;
        }
        __syncwarp();
        for (int cc = 0; cc < nc; ++cc) {
            const int j = c0 + cc;
            const double* col = S + cc * ld;
            const double yj = wn[j & wmask] * col[0];
            for (int k = lane + 1; k <= B; k += 32) wn[(j + k) & wmask] -= col[k] * yj;
            if (lane == 0) y[j] = yj;
            __syncwarp();
        }
        if (lane == 0 && T + nstage < ntot) {
            fence_proxy_async();
            ring.issue(T + nstage);
        }
        __syncwarp();
    }
    // ------------------------------------------------------------------ backward sweep
    constexpr int LPC = 32 / G;             // lanes per column in a block
    const int cc_me = lane / LPC, part = lane % LPC;
    double* xw = wn;                        // window of solved x values (rows above the block)
    for (int u = 0; u < ring.nfw; ++u, ++T) {
        const double* S = ring.wait(T);
        const int hi = n - u * G, c_lo = max(0, hi - G), nc = hi - c_lo;
        double tv = 0.0;
        const double* colme = S + cc_me * ld;
        if (cc_me < nc) {
            const int j = c_lo + cc_me;
            for (int dd = (hi - j) + part; dd <= B && j + dd < n; dd += LPC) tv += colme[dd] * xw[(j + dd) & wmask];
        }
#pragma unroll
        for (int o = LPC / 2; o > 0; o >>= 1) tv += __shfl_xor_sync(0xffffffffu, tv, o);
        if (cc_me < nc) tv = y[c_lo + cc_me] - tv;
        for (int cj = nc - 1; cj >= 0; --cj) {
            const double mine = tv * colme[0];
            const double xj = __shfl_sync(0xffffffffu, mine, cj * LPC);
            if (cc_me < cj) tv -= colme[cj - cc_me] * xj;
            if (lane == 0) {
                xw[(c_lo + cj) & wmask] = xj;
                y[c_lo + cj] = xj;
            }
        }
        __syncwarp();
        if (lane == 0 && T + nstage < ntot) {
            fence_proxy_async();
            ring.issue(T + nstage);
        }
        __syncwarp();
    }
    // ------------------------------------------------------------------ outputs
    if (mode == SCHUR_BACKSUB) {
        for (int i = lane; i < n; i += 32) a.u[idofs[i]] = y[i];
        return;
    }
    const int32_t* gxp = a.gxp + d.gxp_off;
    for (int l = lane; l < nG; l += 32) {
        double q = 0.0;
        for (int e = gxp[l]; e < gxp[l + 1]; ++e) {
            const int c = a.gx_col[e];
            if (c >= 0) {
                if (mode == SCHUR_APPLY) q += a.gx_val[e] * xl[c];
            } else {
                q -= a.gx_val[e] * y[-c - 1];
            }
        }
        a.qloc[d.goff + l] = q;
    }
}

int launch_schur_local(const SchurArgs& a, cudaStream_t st) {
    if (a.nsl == 0) return 0;
    const int G = a.band_w <= 127 ? 8 : 4;
    int win = 32;
    while (win < a.band_w + 1 + G + 1) win <<= 1;
    const int nstage = 3;
    const size_t smem = 128 + sizeof(double) * (size_t(nstage) * G * a.ld + win + a.maxG);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    const bool set_attr = (cs == cudaStreamCaptureStatusNone) && smem > 48 * 1024;
    if (G == 8) {
        if (set_attr) cudaFuncSetAttribute(k_schur_local<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        k_schur_local<8><<<a.nsl, 32, smem, st>>>(a, nstage, win);
    } else {
        if (set_attr) cudaFuncSetAttribute(k_schur_local<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        k_schur_local<4><<<a.nsl, 32, smem, st>>>(a, nstage, win);
    }
    return 1;
}

}  // namespace de
