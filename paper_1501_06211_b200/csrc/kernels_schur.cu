// kernels_schur.cu — SURVEY.md §8(a) rows C1 (condensed rhs), C2 (Schur apply, the headline kernel)
// and C6 (back-substitution): per owned subdomain s
//
//   C2 (SCHUR_APPLY):    x = R_s p;  y = A_IG x;  w = A_II^-1 y;  q_s = A_GG x - A_GI w
//   C1 (SCHUR_CONDENSE): w = A_II^-1 f_I;  q_s = -A_GI w     (g = f_G + sum_s R_s^T q_s)
//   C6 (SCHUR_BACKSUB):  w = A_II^-1 (f_I - A_IG R_s u_G);  u_I = w   (PAPER.md:141,143 combined, :136)
//
// One warp per subdomain (one-warp CTAs). A_II = L L^T is stored twice in column-band form: L itself
// and M = P L^T P (P = index reversal; column j' of M is row n-1-j' of L, reversed). Both triangular
// solves are then the same forward column-axpy sweep
//      y_j = t_j / L_jj ;  t_{j+k} -= L_{j+k,j} y_j   (k = 1..b)
// run on L (y = L^-1 rhs) and on M (P w = M^-1 P y). The b+1 active rows live in REGISTERS: lane l
// holds rows r = l (mod 32) in NS slots; the owner of row j broadcasts y_j with one shuffle, so the
// dependency chain per row is SHFL + DMUL + DFMA. Columns stream through a ring of shared-memory stages
// filled by TMA bulk copies (cp.async.bulk + mbarrier complete_tx) issued by lane 0; the ring runs
// over L then M, so M's first stages are in flight while the L sweep finishes.
#include "de_internal.h"

#include <cstdlib>

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

// Unified ring over 2*nst stages: stage T < nst streams columns [T*G, ...) of L, stage T >= nst the
// same columns of M.
struct Ring {
    uint64_t* bar;
    double* stg;
    int nstage, G, ld, n, nst;
    const double* L;
    const double* M;
    __device__ __forceinline__ void issue(int T) const {   // lane 0 only
        const int t = T < nst ? T : T - nst;
        const int c0 = t * G, nc = min(G, n - c0);
        const int slot = T % nstage;
        const uint32_t bytes = uint32_t(nc) * uint32_t(ld) * 8u;
        mbar_expect_tx(bar + slot, bytes);
        tma_load_1d(stg + size_t(slot) * G * ld, (T < nst ? L : M) + size_t(c0) * ld, bytes, bar + slot);
    }
    __device__ __forceinline__ const double* wait(int T) const {
        const int slot = T % nstage;
        mbar_wait(bar + slot, uint32_t((T / nstage) & 1));
        return stg + size_t(slot) * G * ld;
    }
};

// One forward column sweep over the ring's current matrix. `src` holds the dense right-hand side
// (row r at src[r]); `dst` receives the solution (row j at dst[j], or dst[n-1-j] when reversed).
// src and dst may alias: row j is written only after every row <= j + 32*NS has been read.
// Entering rows and outputs move in coalesced 32-row batches (lane l owns rows = l mod 32).
template <int G, int NS>
__device__ __forceinline__ void sweep(const Ring& ring, const double* src, double* dst, bool reversed, int& T,
                                      int lane, int B, int n) {
    // reversed: rhs row r is src[n-1-r] and solution row j goes to dst[n-1-j] (the M = P L^T P sweep)
    const int ld = ring.ld;
    double v[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const int r = lane + 32 * s;
        v[s] = r < n ? src[reversed ? n - 1 - r : r] : 0.0;
    }
    double pend = 0.0, outv = 0.0;
    for (int t = 0; t < ring.nst; ++t, ++T) {
        const double* S = ring.wait(T);
        const int c0 = t * G, nc = min(G, n - c0);
#pragma unroll
        for (int cc = 0; cc < G; ++cc) {
            if (cc < nc) {
                const int j = c0 + cc;
                const int o = j & 31;
                if (o == 0) {   // new 32-row block: prefetch this block's entering rows (coalesced)
                    const int r = j + lane + 32 * NS;
                    pend = r < n ? src[reversed ? n - 1 - r : r] : 0.0;
                }
                const double* col = S + cc * ld;
                const int k0 = (lane - j) & 31;
                double cv[NS];
#pragma unroll
                for (int s = 0; s < NS; ++s) {
                    const int k = k0 + 32 * s;
                    cv[s] = (k <= B && (s > 0 || k0 != 0)) ? col[k] : 0.0;
                }
                const double yj = __shfl_sync(0xffffffffu, v[0], o) * col[0];
#pragma unroll
                for (int s = 0; s < NS; ++s) v[s] = fma(-cv[s], yj, v[s]);
                if (lane == o) {
                    outv = yj;
#pragma unroll
                    for (int s = 0; s < NS - 1; ++s) v[s] = v[s + 1];
                    v[NS - 1] = pend;
                }
                if (o == 31 || j == n - 1) {   // block complete: coalesced store of 32 outputs
                    const int r = j - o + lane;
                    if (lane <= o) dst[reversed ? n - 1 - r : r] = outv;
                }
            }
        }
        __syncwarp();
        if (lane == 0 && T + ring.nstage < 2 * ring.nst) {
            fence_proxy_async();
            ring.issue(T + ring.nstage);
        }
    }
}

template <int G, int NS>
__global__ void __launch_bounds__(32) k_schur_local(SchurArgs a, int nstage) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (a.state != nullptr && a.state->done) return;
    const int lane = threadIdx.x;
    // SCHUR_COLUMNS: warp (sl, t) forms column t of S_sl from x = e_t
    const bool cols = a.mode == SCHUR_COLUMNS;
    const int sl = cols ? a.col_s0 + int(blockIdx.x) / a.maxG : int(blockIdx.x);
    const int tcol = cols ? int(blockIdx.x) % a.maxG : 0;
    const SubDesc d = a.sd[sl];
    if (cols && tcol >= d.nG) return;
    const int n = d.nI, nG = d.nG, B = a.band_w, ld = a.ld;
    const int mode = cols ? SCHUR_APPLY : a.mode;

    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    double* stg = reinterpret_cast<double*>(smem + 128);
    double* xl = stg + size_t(nstage) * G * ld;

    const double* Lb = a.band + d.band_off;
    Ring ring{bar, stg, nstage, G, ld, n, (n + G - 1) / G, Lb, Lb + size_t(n) * ld};
    if (lane == 0) {
        for (int i = 0; i < nstage; ++i) mbar_init(bar + i, 1);
        fence_mbar_init();
        for (int T = 0; T < min(nstage, 2 * ring.nst); ++T) ring.issue(T);
    }
    if (cols)
        for (int l = lane; l < nG; l += 32) xl[l] = (l == tcol) ? 1.0 : 0.0;
    else if (mode != SCHUR_CONDENSE)
        for (int l = lane; l < nG; l += 32) xl[l] = a.xin[a.Rg[d.goff + l]];
    __syncwarp();
    const int32_t* igp = a.igp + d.igp_off;
    const int32_t* idofs = a.idofs + d.ioff;
    double* y = cols ? a.colscratch + size_t(blockIdx.x) * a.max_nI : a.scratch + d.ioff;
    for (int r = lane; r < n; r += 32) {          // dense interior right-hand side
        double v = (mode == SCHUR_APPLY) ? 0.0 : a.f[idofs[r]];
        if (mode != SCHUR_CONDENSE) {
            double acc = 0.0;
            for (int e = igp[r]; e < igp[r + 1]; ++e) acc += a.ig_val[e] * xl[a.ig_col[e]];
            v = (mode == SCHUR_APPLY) ? acc : v - acc;
        }
        y[r] = v;
    }
    __syncwarp();
    int T = 0;
    sweep<G, NS>(ring, y, y, false, T, lane, B, n);   // y = L^-1 rhs
    __syncwarp();
    sweep<G, NS>(ring, y, y, true, T, lane, B, n);    // w = L^-T y  (M^-1 on reversed vectors)
    __syncwarp();
    const double* w = y;
    if (mode == SCHUR_BACKSUB) {
        for (int i = lane; i < n; i += 32) a.u[idofs[i]] = w[i];
        return;
    }
    const int32_t* gxp = a.gxp + d.gxp_off;
    for (int l = lane; l < nG; l += 32) {
        double q = 0.0;
        for (int e = gxp[l]; e < gxp[l + 1]; ++e) {
            const int cidx = a.gx_col[e];
            if (cidx >= 0) {
                if (mode == SCHUR_APPLY) q += a.gx_val[e] * xl[cidx];
            } else {
                q -= a.gx_val[e] * w[-cidx - 1];
            }
        }
        if (cols && l / STS >= tcol / STS) a.sexp[d.sexp_off + sexp_packed_index(l, tcol)] = q;   // S_s[l][tcol]
        else a.qloc[d.goff + l] = q;
    }
}

// q_s = S_s x_s from the packed lower tiles (STS x STS, see de_internal.h): every tile is read once and used twice
// (T x_J for its row block, T^T x_I for its column block), so only half the dense bytes stream from HBM.
// Warp w owns tile rows dealt in zig-zag order (0, nt-1, 1, nt-2, ...) for balance; lane l holds rows h + 2k
// (h = l / 16, k < 8) and column l % 16 of a tile. Per-warp partial vectors are summed in a fixed order.
constexpr int SE_T = 256, SE_W = SE_T / 32, SE_U = 4;
__global__ void __launch_bounds__(SE_T) k_schur_explicit(const SubDesc* __restrict__ sd, const double* __restrict__ sexp,
                                                         const int32_t* __restrict__ Rg, const double* __restrict__ xin,
                                                         double* __restrict__ qloc, const PcgState* s) {
    if (s != nullptr && s->done) return;
    extern __shared__ double se_sm[];
    const SubDesc d = sd[blockIdx.x];
    const int nG = d.nG, nt = (nG + STS - 1) / STS, np = nt * STS, tid = threadIdx.x;
    const int lane = tid & 31, w = tid >> 5, h = lane >> 4, j = lane & 15;
    double* xs = se_sm;            // [np], zero past nG
    double* yw = se_sm + np;       // [SE_W][np]
    for (int l = tid; l < np; l += SE_T) xs[l] = l < nG ? xin[Rg[d.goff + l]] : 0.0;
    for (int l = tid; l < SE_W * np; l += SE_T) yw[l] = 0.0;
    __syncthreads();
    const double* S = sexp + d.sexp_off;
    double* y = yw + w * np;
    for (int m = w; m < nt; m += SE_W) {
        const int I = (m & 1) ? nt - 1 - m / 2 : m / 2;
        const double* Trow = S + int64_t(I) * (I + 1) / 2 * (STS * STS);
        double xi[STS / 2], acc[STS / 2];
#pragma unroll
        for (int k = 0; k < STS / 2; ++k) {
            xi[k] = xs[I * STS + h + 2 * k];
            acc[k] = 0.0;
        }
        for (int J0 = 0; J0 <= I; J0 += SE_U) {   // SE_U tiles per step: 8 SE_U loads per lane in flight
            double tv[SE_U][STS / 2];
#pragma unroll
            for (int u = 0; u < SE_U; ++u) {
                const double* T = Trow + (J0 + u) * (STS * STS);
#pragma unroll
                for (int k = 0; k < STS / 2; ++k) tv[u][k] = J0 + u <= I ? __ldcs(T + (h + 2 * k) * STS + j) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < SE_U; ++u) {
                const int J = J0 + u;
                if (J > I) break;
                const double xj = xs[J * STS + j];
                double tt = 0.0;
#pragma unroll
                for (int k = 0; k < STS / 2; ++k) {
                    acc[k] = fma(tv[u][k], xj, acc[k]);
                    tt = fma(tv[u][k], xi[k], tt);
                }
                if (J < I) {   // T^T x_I -> rows of block J
                    tt += __shfl_xor_sync(0xffffffffu, tt, 16);
                    if (h == 0) y[J * STS + j] += tt;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < STS / 2; ++k)
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
        if (j == 0)
#pragma unroll
            for (int k = 0; k < STS / 2; ++k) y[I * STS + h + 2 * k] += acc[k];
        __syncwarp();
    }
    __syncthreads();
    for (int l = tid; l < nG; l += SE_T) {
        double q = 0.0;
#pragma unroll
        for (int ww = 0; ww < SE_W; ++ww) q += yw[ww * np + l];
        qloc[d.goff + l] = q;
    }
}

void launch_schur_explicit(const SubDesc* sd, int nsl, const double* sexp, const int32_t* Rg, const double* xin,
                           double* qloc, int maxG, const PcgState* s, cudaStream_t st) {
    if (nsl == 0) return;
    const int np = (maxG + STS - 1) / STS * STS;
    const size_t smem = size_t(1 + SE_W) * np * sizeof(double);
    k_schur_explicit<<<nsl, SE_T, smem, st>>>(sd, sexp, Rg, xin, qloc, s);
}

// once per context, outside any graph capture
void prepare_schur_explicit(int maxG) {
    const int np = (maxG + STS - 1) / STS * STS;
    raise_dyn_smem(reinterpret_cast<const void*>(k_schur_explicit), size_t(1 + SE_W) * np * sizeof(double));
}

// ------------------------------------------------------------------ explicit S_s formation, R columns per warp
// The forward column sweep of sweep() for R right-hand sides at once: every factor column loaded from the
// TMA stage feeds R independent chains (ILP across columns, R-fold less factor traffic per column).
// yb holds the R right-hand sides row-major ([row][k]); solutions overwrite them (same aliasing rule).
template <int G, int NS, int R>
__device__ __forceinline__ void sweep_multi(const Ring& ring, double* yb, bool reversed, int& T, int lane, int B, int n) {
    const int ld = ring.ld;
    auto at = [&](int r) { return size_t(reversed ? n - 1 - r : r) * R; };
    double v[R][NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const int r = lane + 32 * s;
#pragma unroll
        for (int k = 0; k < R; ++k) v[k][s] = r < n ? yb[at(r) + k] : 0.0;
    }
    double pend[R], outv[R];
#pragma unroll
    for (int k = 0; k < R; ++k) pend[k] = outv[k] = 0.0;
    for (int t = 0; t < ring.nst; ++t, ++T) {
        const double* S = ring.wait(T);
        const int c0 = t * G, nc = min(G, n - c0);
#pragma unroll
        for (int cc = 0; cc < G; ++cc) {
            if (cc < nc) {
                const int j = c0 + cc;
                const int o = j & 31;
                if (o == 0) {
                    const int r = j + lane + 32 * NS;
#pragma unroll
                    for (int k = 0; k < R; ++k) pend[k] = r < n ? yb[at(r) + k] : 0.0;
                }
                const double* col = S + cc * ld;
                const int k0 = (lane - j) & 31;
                double cv[NS];
#pragma unroll
                for (int s = 0; s < NS; ++s) {
                    const int kk = k0 + 32 * s;
                    cv[s] = (kk <= B && (s > 0 || k0 != 0)) ? col[kk] : 0.0;
                }
                const double inv = col[0];
                double yj[R];
#pragma unroll
                for (int k = 0; k < R; ++k) yj[k] = __shfl_sync(0xffffffffu, v[k][0], o) * inv;
#pragma unroll
                for (int k = 0; k < R; ++k)
#pragma unroll
                    for (int s = 0; s < NS; ++s) v[k][s] = fma(-cv[s], yj[k], v[k][s]);
                if (lane == o) {
#pragma unroll
                    for (int k = 0; k < R; ++k) {
                        outv[k] = yj[k];
#pragma unroll
                        for (int s = 0; s < NS - 1; ++s) v[k][s] = v[k][s + 1];
                        v[k][NS - 1] = pend[k];
                    }
                }
                if (o == 31 || j == n - 1) {
                    const int r = j - o + lane;
                    if (lane <= o)
#pragma unroll
                        for (int k = 0; k < R; ++k) yb[at(r) + k] = outv[k];
                }
            }
        }
        __syncwarp();
        if (lane == 0 && T + ring.nstage < 2 * ring.nst) {
            fence_proxy_async();
            ring.issue(T + ring.nstage);
        }
    }
}

// Columns t0..t0+R-1 of S_s = A_GG - A_GI A_II^-1 A_IG (x = e_t), one warp per (subdomain, column group).
template <int G, int NS, int R>
__global__ void __launch_bounds__(32) k_schur_cols(SchurArgs a, int nstage) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x;
    const int wps = (a.maxG + R - 1) / R;
    const int sl = a.col_s0 + int(blockIdx.x) / wps, t0 = (int(blockIdx.x) % wps) * R;
    const SubDesc d = a.sd[sl];
    if (t0 >= d.nG) return;
    const int n = d.nI, nG = d.nG, B = a.band_w, ld = a.ld;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    double* stg = reinterpret_cast<double*>(smem + 128);
    const double* Lb = a.band + d.band_off;
    Ring ring{bar, stg, nstage, G, ld, n, (n + G - 1) / G, Lb, Lb + size_t(n) * ld};
    if (lane == 0) {
        for (int i = 0; i < nstage; ++i) mbar_init(bar + i, 1);
        fence_mbar_init();
        for (int T = 0; T < min(nstage, 2 * ring.nst); ++T) ring.issue(T);
    }
    const int32_t* igp = a.igp + d.igp_off;
    double* yb = a.colscratch + size_t(blockIdx.x) * size_t(a.max_nI) * R;
    for (int r = lane; r < n; r += 32) {                  // rhs columns t0..t0+R-1 of A_IG
        double acc[R];
#pragma unroll
        for (int k = 0; k < R; ++k) acc[k] = 0.0;
        for (int e = igp[r]; e < igp[r + 1]; ++e) {
            const int cidx = a.ig_col[e] - t0;
#pragma unroll
            for (int k = 0; k < R; ++k)
                if (cidx == k) acc[k] += a.ig_val[e];
        }
#pragma unroll
        for (int k = 0; k < R; ++k) yb[size_t(r) * R + k] = acc[k];
    }
    __syncwarp();
    int T = 0;
    sweep_multi<G, NS, R>(ring, yb, false, T, lane, B, n);
    __syncwarp();
    sweep_multi<G, NS, R>(ring, yb, true, T, lane, B, n);
    __syncwarp();
    const int32_t* gxp = a.gxp + d.gxp_off;
    for (int l = lane; l < nG; l += 32) {
        double q[R];
#pragma unroll
        for (int k = 0; k < R; ++k) q[k] = 0.0;
        for (int e = gxp[l]; e < gxp[l + 1]; ++e) {
            const int cidx = a.gx_col[e];
            const double val = a.gx_val[e];
            if (cidx >= 0) {
#pragma unroll
                for (int k = 0; k < R; ++k)
                    if (cidx == t0 + k) q[k] += val;
            } else {
#pragma unroll
                for (int k = 0; k < R; ++k) q[k] -= val * yb[size_t(-cidx - 1) * R + k];
            }
        }
#pragma unroll
        for (int k = 0; k < R; ++k)   // S_s[l][t0+k] into the packed lower tiles
            if (t0 + k < nG && l / STS >= (t0 + k) / STS) a.sexp[d.sexp_off + sexp_packed_index(l, t0 + k)] = q[k];
    }
}

// ---------------------------------------------------------------- S_s formation, thread per column
// Columns of S_s = A_GG - A_GI A_II^-1 A_IG (x = e_t), one CTA per subdomain, thread t <-> column t.
// Both triangular solves are the same recurrence over r = 0..n-1 on a stream of factor columns taken in
// decreasing order, z_r = (rhs_r - sum_{k=1..B} F[c][k] z_{r-k}) F[c][0], c = n-1-r: the forward L solve reads
// the M = P L^T P copy (its column n-1-r is row r of L) and the backward L^T solve reads L (rhs = y reversed).
// The last SF_W values z_{r-1..r-B} of a thread live in registers: the row loop is unrolled by SF_W, so every
// window index is a compile-time constant. Factor columns are shared by the CTA through a two-half shared
// ring filled by cp.async SF_CB rows ahead.
constexpr int SF_T = FORM_THREADS;   // threads = columns per pass
constexpr int SF_W = 68;     // register window (>= B + 1; 2D 32x32 subdomains: B = 65..67)
constexpr int SF_CB = 16;    // rows per ring half
constexpr int SF_U = 8;      // rows per unrolled block of the recurrence

__device__ __forceinline__ void sf_cp16(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}

// rows r0 .. r0+SF_CB-1 (factor columns n-1-r) into ring half (r0 / SF_CB) & 1
__device__ __forceinline__ void sf_issue(const double* __restrict__ F, int n, int ld, int r0, double* ring) {
    double* dst = ring + size_t((r0 / SF_CB) & 1) * SF_CB * ld;
    const int chunks = ld / 2;
    for (int q = threadIdx.x; q < SF_CB * chunks; q += blockDim.x) {
        const int cc = q / chunks, off = (q - cc * chunks) * 2, r = r0 + cc;
        if (r < n) sf_cp16(dst + cc * ld + off, F + size_t(n - 1 - r) * ld + off);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// One solve over the factor stream (see above): rhs(r) gives the right-hand side of row r and out(r, z) takes
// its solution. PF > 0: rhs(r) is a global load, issued PF rows ahead into a register ring (static indices,
// SF_W % PF == 0); it enters after the window terms either way, so its latency overlaps them.
template <int PF, class Rhs, class Out>
__device__ __forceinline__ void sf_sweep(const double* __restrict__ F, int n, int ld, int B, double* ring, Rhs rhs,
                                         Out out) {
    // rows in unrolled blocks of SF_U: z[j] holds the solution of row r0-1-j (0 before row 0), the block's own
    // rows go to nz[]; after the block the window shifts by SF_U (a fully unrolled 68-row body would not fit the
    // instruction cache)
    static_assert(PF == 0 || PF == SF_U, "prefetch ring = block");
    double z[SF_W], pf[SF_U];
#pragma unroll
    for (int q = 0; q < SF_W; ++q) z[q] = 0.0;
#pragma unroll
    for (int q = 0; q < SF_U; ++q) pf[q] = (PF > 0 && q < n) ? rhs(q) : 0.0;
    __syncthreads();   // ring free (previous sweep done)
    sf_issue(F, n, ld, 0, ring);
    for (int r0 = 0; r0 < n; r0 += SF_U) {
        double nz[SF_U];
#pragma unroll
        for (int q = 0; q < SF_U; ++q) {
            const int r = r0 + q;
            nz[q] = 0.0;
            if (r < n) {
                if ((r % SF_CB) == 0) {   // this half has landed; start the next one (the other half is free)
                    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
                    __syncthreads();
                    if (r + SF_CB < n) sf_issue(F, n, ld, r + SF_CB, ring);
                }
                const double* col = ring + (size_t((r / SF_CB) & 1) * SF_CB + (r % SF_CB)) * ld;
                double b;
                if constexpr (PF > 0) {
                    b = pf[q];
                    pf[q] = r + PF < n ? rhs(r + PF) : 0.0;
                } else {
                    b = rhs(r);
                }
                double acc[4] = {0.0, 0.0, 0.0, 0.0};
                // (16-byte coefficient loads -- double2 or explicit ld.shared.v2.f64, 544 LDS.128 instead of 1208 LDS.64
                // in the SASS -- measured SLOWER on c5: refactorisation 60.7 -> 86.7 / 90.2 ms)
#pragma unroll
                for (int k = SF_W - 1; k >= 1; --k)   // oldest rows first: the newest terms close the row
                    if (k <= B) acc[k & 3] = fma(-col[k], k <= q ? nz[q - k] : z[k - q - 1], acc[k & 3]);
                const double zr = (b + ((acc[0] + acc[1]) + (acc[2] + acc[3]))) * col[0];
                nz[q] = zr;
                out(r, zr);
            }
        }
#pragma unroll
        for (int j = SF_W - 1; j >= SF_U; --j) z[j] = z[j - SF_U];
#pragma unroll
        for (int q = 0; q < SF_U; ++q) z[SF_U - 1 - q] = nz[q];
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

__global__ void __launch_bounds__(SF_T, 1) k_schur_form(SchurArgs a) {
    extern __shared__ __align__(16) double ring[];   // [2][SF_CB][ld], then the staged A_IG rows
    const int sl = a.col_s0 + int(blockIdx.x);
    const SubDesc d = a.sd[sl];
    const int n = d.nI, nG = d.nG, B = a.band_w, ld = a.ld, tid = threadIdx.x;
    const double* Lb = a.band + d.band_off;
    const double* Mb = Lb + size_t(n) * ld;
    const int32_t* igp = a.igp + d.igp_off;
    const int32_t* gxp = a.gxp + d.gxp_off;
    double* ys = a.colscratch + size_t(blockIdx.x) * size_t(a.max_nI) * SF_T;   // [row][SF_T]
    // A_IG rows of this subdomain in shared memory (values, columns, row pointers rebased to 0)
    double* s_val = ring + size_t(2) * SF_CB * ld;
    int* s_col = reinterpret_cast<int*>(s_val + a.max_ig);
    int* s_ptr = s_col + a.max_ig;
    const int e0 = igp[0], ne = igp[n] - e0;
    for (int e = tid; e < ne; e += SF_T) {
        s_val[e] = a.ig_val[e0 + e];
        s_col[e] = a.ig_col[e0 + e];
    }
    for (int r = tid; r <= n; r += SF_T) s_ptr[r] = igp[r] - e0;
    __syncthreads();
    for (int t0 = 0; t0 < nG; t0 += SF_T) {
        const int t = t0 + tid;
        // forward: L y = A_IG e_t (rows of L = columns of M, reversed)
        sf_sweep<0>(Mb, n, ld, B, ring,
                    [&](int r) {
                        double v = 0.0;
                        for (int e = s_ptr[r]; e < s_ptr[r + 1]; ++e)
                            if (s_col[e] == t) v += s_val[e];
                        return v;
                    },
                    [&](int r, double zr) { ys[size_t(r) * SF_T + tid] = zr; });
        // backward: L^T x = y, row order reversed, in place (a row's rhs is read PF rows before it is overwritten)
        sf_sweep<SF_U>(Lb, n, ld, B, ring, [&](int r) { return ys[size_t(n - 1 - r) * SF_T + tid]; },
                     [&](int r, double zr) { ys[size_t(n - 1 - r) * SF_T + tid] = zr; });
        // S_s[l][t] = A_GG[l][t] - A_GI[l][:] x; stored at (row t, column l) by symmetry (coalesced)
        if (t < nG)
            for (int l = 0; l < nG; ++l) {
                double q = 0.0;
                for (int e = gxp[l]; e < gxp[l + 1]; ++e) {
                    const int cidx = a.gx_col[e];
                    const double val = a.gx_val[e];
                    if (cidx >= 0) q += (cidx == t) ? val : 0.0;
                    else q -= val * ys[size_t(-cidx - 1) * SF_T + tid];
                }
                if (l / STS >= t / STS) a.sexp[d.sexp_off + sexp_packed_index(l, t)] = q;   // S_s[l][t]
            }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- wide bands (3D): blocked solves
// One CTA per subdomain for APPLY / CONDENSE / BACKSUB when b+1 exceeds the register window of the warp
// sweep: L is streamed in BK_P-column panels (two-stage TMA ring, one bulk copy per panel). Forward L y = rhs:
// one warp solves the panel's diagonal block (lane = row, one shuffle per column), then the CTA updates the
// <= b rows below it. Backward L^T x = y reads the same L panels in descending order: the CTA forms each panel
// column's dot product with the solved x below the panel, then one warp solves the diagonal block. The chain
// per row is one shuffle + FMA instead of a full band row, and the M copy is not read.
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// Inverses of the BLK_D x BLK_D diagonal blocks of every local factor (one warp per block, lane c = column c of the
// inverse by forward substitution): the blocked sweeps below apply them as small dense products, so no 16-step
// shuffle chain sits between a panel's arrival and its trailing update.
template <int BLK_D>
__global__ void __launch_bounds__(256) k_blk_diag_inv(const SubDesc* sd, int nsl, const double* __restrict__ band, int ld,
                                                      double* __restrict__ dinv, int np_max) {
    const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int sl = gwarp / np_max, p = gwarp - sl * np_max;
    if (sl >= nsl) return;
    const SubDesc d = sd[sl];
    const int n = d.nI, j0 = p * BLK_D;
    double* out = dinv + (size_t(sl) * np_max + p) * BLK_D * BLK_D;
    if (j0 >= n) return;
    const int nc = min(BLK_D, n - j0);
    const double* Lb = band + d.band_off;
    if (lane >= BLK_D) return;
    double x[BLK_D];
    const int c = lane;
#pragma unroll
    for (int i = 0; i < BLK_D; ++i) {
        double v = 0.0;
        if (c < nc && i < nc) {
            if (i == c) {
                v = Lb[size_t(j0 + c) * ld];              // slot 0 holds 1 / L_cc
            } else if (i > c) {
                double sacc = 0.0;
#pragma unroll
                for (int k = 0; k < BLK_D; ++k)
                    if (k >= c && k < i) sacc = fma(Lb[size_t(j0 + k) * ld + (i - k)], x[k], sacc);
                v = -sacc * Lb[size_t(j0 + i) * ld];
            }
        } else if (i == c) {
            v = 1.0;                                       // identity padding of the last block
        }
        x[i] = v;
    }
#pragma unroll
    for (int i = 0; i < BLK_D; ++i) out[i * BLK_D + c] = x[i];
}

void launch_blk_diag_inv(const SubDesc* sd, int nsl, const double* band, int ld, double* dinv, int dinv_np, int bs,
                         cudaStream_t st) {
    const long long warps = (long long)nsl * dinv_np;
    if (warps <= 0) return;
    const unsigned grid = unsigned((warps + 7) / 8);
    if (bs == 16) k_blk_diag_inv<16><<<grid, 256, 0, st>>>(sd, nsl, band, ld, dinv, dinv_np);
    else if (bs == 12) k_blk_diag_inv<12><<<grid, 256, 0, st>>>(sd, nsl, band, ld, dinv, dinv_np);
    else if (bs == 8) k_blk_diag_inv<8><<<grid, 256, 0, st>>>(sd, nsl, band, ld, dinv, dinv_np);
    else k_blk_diag_inv<4><<<grid, 256, 0, st>>>(sd, nsl, band, ld, dinv, dinv_np);
}

constexpr int BK_T = 256;   // threads; BK_P panel columns, BK_S ring stages (template: tuned per band width)
// BK_TH: the last BK_TH columns of every panel are loaded by the CTA's threads (16-byte cp.async, completion tracked by the
// panel's mbarrier) beside the bulk copy of the first BK_P - BK_TH: a second stream per SM.
template <int BK_P, int BK_S, int BK_TH = 0>
__global__ void __launch_bounds__(BK_T, 1) k_schur_blk(SchurArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (a.state != nullptr && a.state->done) return;
    const unsigned FULL = 0xffffffffu;
    const SubDesc d = a.sd[blockIdx.x];
    const int n = d.nI, nG = d.nG, B = a.band_w, ld = a.ld, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int mode = a.mode;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    double* pan = reinterpret_cast<double*>(smem + 128);   // [BK_S][BK_P][ld]
    double* dblk = pan + BK_S * BK_P * ld;                 // [BK_S][BK_P][BK_P] inverse diagonal blocks (use_dinv)
    double* v = dblk + BK_S * BK_P * BK_P;               // [n]: rhs, then y, then x
    const bool use_dinv = a.dinv != nullptr && a.dinv_bs == BK_P;
    const double* dsrc = use_dinv ? a.dinv + size_t(blockIdx.x) * a.dinv_np * BK_P * BK_P : nullptr;
    // [nG] gathered interface values: behind v, or (ring of three or more stages: no room for both) in the LAST ring
    // stage, which the prologue and the epilogue use while no panel lives there
    constexpr bool XL_IN_RING = BK_S >= 3;
    double* xl = XL_IN_RING ? pan + size_t(BK_S - 1) * BK_P * ld : v + a.max_nI;
    const double* Lb = a.band + d.band_off;
    const int np = (n + BK_P - 1) / BK_P;
    auto panel_of = [&](int q) { return q < np ? q : 2 * np - 1 - q; };   // forward ascending, backward descending
    auto issue = [&](int q) {   // thread 0: the bulk copies of panel q (its first BK_P - BK_TH columns) and of its diagonal block
        const int p = panel_of(q), c0 = p * BK_P, nc = min(BK_P - BK_TH, n - c0);
        const uint32_t bytes = uint32_t(nc) * uint32_t(ld) * 8u;
        const uint32_t dbytes = use_dinv ? uint32_t(BK_P * BK_P * 8) : 0u;
        mbar_expect_tx(bar + (q % BK_S), bytes + dbytes);
        tma_load_1d(pan + size_t(q % BK_S) * BK_P * ld, Lb + size_t(c0) * ld, bytes, bar + (q % BK_S));
        if (use_dinv)
            tma_load_1d(dblk + size_t(q % BK_S) * BK_P * BK_P, dsrc + size_t(p) * BK_P * BK_P, dbytes, bar + (q % BK_S));
    };
    auto issue_threads = [&](int q) {   // every thread: its share of the panel's last BK_TH columns, then one arrival
        if constexpr (BK_TH > 0) {
            const int p = panel_of(q), c0 = p * BK_P + (BK_P - BK_TH), nc = max(0, min(BK_TH, n - c0));
            const int chunks = nc * ld / 2;   // 16-byte chunks (ld is even)
            const double* src = Lb + size_t(c0) * ld;
            double* dst = pan + size_t(q % BK_S) * BK_P * ld + size_t(BK_P - BK_TH) * ld;
            for (int i = tid; i < chunks; i += BK_T) {
                const unsigned sa = smem_u32(dst + 2 * i);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src + 2 * i) : "memory");
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar + (q % BK_S))) : "memory");
        }
    };
    if (tid == 0) {
        for (int i = 0; i < BK_S; ++i) mbar_init(bar + i, 1 + (BK_TH > 0 ? BK_T : 0));
        fence_mbar_init();
    }
    if (BK_TH > 0) __syncthreads();   // the barriers exist before any thread arrives on them
    for (int q = 0; q < min(BK_S - (XL_IN_RING ? 1 : 0), 2 * np); ++q) {
        if (tid == 0) issue(q);
        issue_threads(q);
    }
    if (mode != SCHUR_CONDENSE)
        for (int l = tid; l < nG; l += BK_T) xl[l] = a.xin[a.Rg[d.goff + l]];
    __syncthreads();
    const int32_t* igp = a.igp + d.igp_off;
    const int32_t* idofs = a.idofs + d.ioff;
    for (int r = tid; r < n; r += BK_T) {          // dense interior right-hand side
        double val = (mode == SCHUR_APPLY) ? 0.0 : a.f[idofs[r]];
        if (mode != SCHUR_CONDENSE) {
            double acc = 0.0;
            for (int e = igp[r]; e < igp[r + 1]; ++e) acc += a.ig_val[e] * xl[a.ig_col[e]];
            val = (mode == SCHUR_APPLY) ? acc : val - acc;
        }
        v[r] = val;
    }
    __syncthreads();
    if (XL_IN_RING && BK_S - 1 < 2 * np) {   // the last stage is free of xl now
        if (tid == 0) issue(BK_S - 1);
        issue_threads(BK_S - 1);
    }
    for (int q = 0; q < 2 * np; ++q) {
        mbar_wait(bar + (q % BK_S), uint32_t((q / BK_S) & 1));
        const double* P = pan + size_t(q % BK_S) * BK_P * ld;
        const int p = panel_of(q), j0 = p * BK_P, nc = min(BK_P, n - j0);
        if (q < np) {   // forward: diagonal block, then the rows below
            if (wid == 0 && use_dinv) {   // y_blk = L_jj^-1 v_blk: 16 independent row products, no chain
                const double* D = dblk + size_t(q % BK_S) * BK_P * BK_P;
                double acc = 0.0;
                if (lane < nc) {
#pragma unroll
                    for (int jj = 0; jj < BK_P; ++jj)
                        if (jj <= lane) acc = fma(D[lane * BK_P + jj], v[j0 + jj], acc);
                }
                __syncwarp();
                if (lane < nc) v[j0 + lane] = acc;
            } else if (wid == 0) {   // unrolled: every coefficient load is off the shuffle-FMA chain
                double vr = lane < nc ? v[j0 + lane] : 0.0;
                double cf[BK_P], dg[BK_P];
#pragma unroll
                for (int jj = 0; jj < BK_P; ++jj) {
                    cf[jj] = (jj < nc && lane > jj && lane < nc) ? P[jj * ld + (lane - jj)] : 0.0;
                    dg[jj] = jj < nc ? P[jj * ld] : 0.0;   // slot 0 holds 1 / L_jj
                }
#pragma unroll
                for (int jj = 0; jj < BK_P; ++jj) {
                    const double yj = __shfl_sync(FULL, vr, jj) * dg[jj];
                    vr = lane == jj ? yj : fma(-cf[jj], yj, vr);
                }
                if (lane < nc) v[j0 + lane] = vr;
            }
            __syncthreads();
            const int ihi = min(n, j0 + nc + B);
            for (int i = j0 + nc + tid; i < ihi; i += BK_T) {
                double acc = 0.0;
#pragma unroll
                for (int jj = 0; jj < BK_P; ++jj) {
                    const int k = i - (j0 + jj);
                    if (jj < nc && k <= B) acc = fma(P[jj * ld + k], v[j0 + jj], acc);
                }
                v[i] -= acc;
            }
        } else {        // backward: dots with the solved rows below, then the diagonal block
            for (int jj = wid; jj < nc; jj += BK_T / 32) {
                const int j = j0 + jj;
                double acc = 0.0;
                for (int k = (j0 + nc - j) + lane; k <= B && j + k < n; k += 32) acc = fma(P[jj * ld + k], v[j + k], acc);
                acc = warp_sum_d(acc);
                if (lane == 0) v[j] -= acc;
            }
            __syncthreads();
            if (wid == 0 && use_dinv) {   // x_blk = L_jj^-T t_blk
                const double* D = dblk + size_t(q % BK_S) * BK_P * BK_P;
                double acc = 0.0;
                if (lane < nc) {
#pragma unroll
                    for (int jj = 0; jj < BK_P; ++jj)
                        if (jj >= lane && jj < nc) acc = fma(D[jj * BK_P + lane], v[j0 + jj], acc);
                }
                __syncwarp();
                if (lane < nc) v[j0 + lane] = acc;
            } else if (wid == 0) {
                double tr = lane < nc ? v[j0 + lane] : 0.0;
                double cf[BK_P], dg[BK_P];
#pragma unroll
                for (int jj = 0; jj < BK_P; ++jj) {
                    cf[jj] = (jj < nc && lane < jj) ? P[lane * ld + (jj - lane)] : 0.0;
                    dg[jj] = jj < nc ? P[jj * ld] : 0.0;
                }
#pragma unroll
                for (int jj = BK_P - 1; jj >= 0; --jj) {
                    const double xj = __shfl_sync(FULL, tr, jj) * dg[jj];
                    tr = lane == jj ? xj : fma(-cf[jj], xj, tr);
                }
                if (lane < nc) v[j0 + lane] = tr;
            }
        }
        __syncthreads();
        if (q + BK_S < 2 * np) {   // every reader is past this panel
            if (tid == 0) issue(q + BK_S);
            issue_threads(q + BK_S);
        }
    }
    if (mode == SCHUR_BACKSUB) {
        for (int i = tid; i < n; i += BK_T) a.u[idofs[i]] = v[i];
        return;
    }
    if (XL_IN_RING && mode == SCHUR_APPLY) {   // every panel is consumed: the ring holds xl again for A_GG x
        for (int l = tid; l < nG; l += BK_T) xl[l] = a.xin[a.Rg[d.goff + l]];
        __syncthreads();
    }
    const int32_t* gxp = a.gxp + d.gxp_off;
    for (int l = tid; l < nG; l += BK_T) {
        double qv = 0.0;
        for (int e = gxp[l]; e < gxp[l + 1]; ++e) {
            const int cidx = a.gx_col[e];
            if (cidx >= 0) {
                if (mode == SCHUR_APPLY) qv += a.gx_val[e] * xl[cidx];
            } else {
                qv -= a.gx_val[e] * v[-cidx - 1];
            }
        }
        a.qloc[d.goff + l] = qv;
    }
}

// panel width / ring depth of k_schur_blk (env DE_BLK_VARIANT: 0 = 16 x 2 (default), 1 = 8 x 4, 2 = 12 x 3, 3 = 8 x 5,
// 4 = 4 x 8). Measured on c4 (ld = 474): 1.33 / 1.54 / 1.54 / 1.64 / 2.31 ms per apply -- the time is ~0.6 us of fixed
// per-panel work (diagonal-block chain, barriers) plus ~0.09 us per column of streaming, so narrower panels lose.
typedef void (*blk_fn)(SchurArgs);
struct BlkVariant {
    blk_fn fn;
    size_t smem;
    int panel;
};
static BlkVariant blk_variant(int ld, int max_nI, int maxG, bool set_attr) {
    static const int PS[8][2] = {{16, 2}, {8, 4}, {12, 3}, {8, 5}, {4, 8}, {16, 3}, {16, 2}, {16, 3}};
    static const blk_fn FN[8] = {k_schur_blk<16, 2>, k_schur_blk<8, 4>, k_schur_blk<12, 3>, k_schur_blk<8, 5>, k_schur_blk<4, 8>,
                                 k_schur_blk<16, 3>, k_schur_blk<16, 2, 8>, k_schur_blk<16, 3, 8>};   // 6, 7: half of every panel by cp.async
    int v = 0;
    if (const char* e = getenv("DE_BLK_VARIANT")) v = std::max(0, std::min(7, atoi(e)));
    auto need = [&](int k) {   // rings of >= 3 stages keep xl in their last stage (no maxG term)
        return 128 + sizeof(double) * (size_t(PS[k][1]) * (PS[k][0] * ld + PS[k][0] * PS[k][0]) + max_nI + (PS[k][1] >= 3 ? 0 : maxG));
    };
    if (need(v) > 227 * 1024 || (PS[v][1] >= 3 && maxG > PS[v][0] * ld)) v = 0;
    BlkVariant r{FN[v], need(v), PS[v][0]};
    if (set_attr) raise_dyn_smem(reinterpret_cast<const void*>(r.fn), r.smem);
    return r;
}

// panel width of the variant in use (= block size of the inverse diagonal blocks)
int schur_blk_panel_width(int ld, int max_nI, int maxG) { return blk_variant(ld, max_nI, maxG, false).panel; }

// once per context, outside any graph capture
void prepare_schur_blk(int ld, int band_w, int max_nI, int maxG) {
    if ((band_w + 1 + 31) / 32 <= 4) return;
    blk_variant(ld, max_nI, maxG, true);
}

constexpr int COL_R = 8;

template <int G, int NS>
static void launch_cols(const SchurArgs& a, int nstage, size_t smem, cudaStream_t st) {
    raise_dyn_smem(reinterpret_cast<const void*>(k_schur_cols<G, NS, COL_R>), smem);
    const unsigned wps = unsigned((a.maxG + COL_R - 1) / COL_R);
    k_schur_cols<G, NS, COL_R><<<unsigned(a.nsl) * wps, 32, smem, st>>>(a, nstage);
}

template <int G, int NS>
static void launch_t(const SchurArgs& a, int nstage, size_t smem, cudaStream_t st) {
    if constexpr (NS <= 4) {
        if (a.mode == SCHUR_COLUMNS) {   // multi-RHS formation (2D bands)
            launch_cols<G, NS>(a, nstage, smem, st);
            return;
        }
    }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusNone) {
        raise_dyn_smem(reinterpret_cast<const void*>(k_schur_local<G, NS>), smem);
        cudaFuncSetAttribute(k_schur_local<G, NS>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
    }
    const unsigned grid = a.mode == SCHUR_COLUMNS ? unsigned(a.nsl) * unsigned(a.maxG) : unsigned(a.nsl);
    k_schur_local<G, NS><<<grid, 32, smem, st>>>(a, nstage);
}

int launch_schur_local(const SchurArgs& a, cudaStream_t st) {
    if (a.nsl == 0) return 0;
    if (a.mode != SCHUR_COLUMNS && (a.band_w + 1 + 31) / 32 > 4 && !getenv("DE_SCHUR_WARP")) {   // wide bands
        const BlkVariant bv = blk_variant(a.ld, a.max_nI, a.maxG, false);
        bv.fn<<<unsigned(a.nsl), BK_T, bv.smem, st>>>(a);
        return 1;
    }
    if (a.mode == SCHUR_COLUMNS && a.band_w + 1 <= SF_W && a.ld % 2 == 0 && !getenv("DE_FORM_WARP") &&
        size_t(2) * SF_CB * a.ld * 8 + size_t(a.max_ig) * 12 + size_t(a.max_nI + 1) * 4 <= 200 * 1024) {
        const size_t smem = size_t(2) * SF_CB * a.ld * sizeof(double) + size_t(a.max_ig) * 12 + size_t(a.max_nI + 1) * 4;
        raise_dyn_smem(reinterpret_cast<const void*>(k_schur_form), smem);
        k_schur_form<<<unsigned(a.nsl), SF_T, smem, st>>>(a);
        return 1;
    }
    const int need = (a.band_w + 1 + 31) / 32;   // register slots per lane covering b+1 rows
    const int G = 4, nstage = 4;
    const size_t smem = 128 + sizeof(double) * (size_t(nstage) * G * a.ld + a.maxG);
    if (need <= 1) launch_t<4, 1>(a, nstage, smem, st);
    else if (need <= 2) launch_t<4, 2>(a, nstage, smem, st);
    else if (need <= 3) launch_t<4, 3>(a, nstage, smem, st);
    else if (need <= 4) launch_t<4, 4>(a, nstage, smem, st);
    else if (need <= 8) launch_t<4, 8>(a, nstage, smem, st);
    else if (need <= 12) launch_t<4, 12>(a, nstage, smem, st);
    else if (need <= 16) launch_t<4, 16>(a, nstage, smem, st);
    else if (need <= 20) launch_t<4, 20>(a, nstage, smem, st);
    else return -1;
    return 1;
}

}  // namespace de
