// kernels_fem.cu — SURVEY.md §8(a) rows B1 (SIMP element blocks) and B2 (batched band Cholesky),
// plus the matrix-free true-residual check K u - f (C6).
//
// B1: E_e = Emin + rho_e^p (E0 - Emin) (R1; PAPER.md:286 for p = 1), and every entry of
//     A_II,s (lower band, local lexicographic order), A_IG,s and A_GG,s (ring) is
//     sum_{elements e of s containing both nodes} E_e * KE0[la,ca][lb,cb]  — node-pair centric, in a fixed
//     element order, atomic-free and deterministic.
// B2: A_II,s = L L^T by right-looking band Cholesky ("O(k^2 n), k is the bandwidth"),
//     written twice: L (column band) and M = P L^T P (column j' of M = row n-1-j' of L, reversed),
//     so both triangular solves of the Schur apply are forward column sweeps;
//     2D bands (b ~ 65) keep the active (b+1)^2 window in shared memory; 3D bands (b ~ 400-500) use
//     32-column panels in shared memory with the trailing rank-32 update in global memory (L2).
//     Storage: column band, ld = b+1 rounded to even, slot 0 = 1/L_jj (the solves multiply).
#include "de_internal.h"

#include <cstdlib>

namespace de {

__constant__ double c_KE[24 * 24];

void upload_KE0(const double* ke, int nke, cudaStream_t st) {
    cudaMemcpyToSymbolAsync(c_KE, ke, sizeof(double) * nke * nke, 0, cudaMemcpyHostToDevice, st);
}

__global__ void k_simp(const double* __restrict__ rho, double* __restrict__ Ee, int64_t n, double E0,
                       double Emin, double p) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const double r = rho[i];
        const double rp = (p == 3.0) ? r * r * r : pow(r, p);
        Ee[i] = Emin + rp * (E0 - Emin);
    }
}

void launch_simp(const double* rho, double* Ee, int64_t nelem, double E0, double Emin, double p,
                 cudaStream_t st) {
    const int blocks = int(std::min<int64_t>((nelem + 255) / 256, 148 * 16));
    k_simp<<<blocks, 256, 0, st>>>(rho, Ee, nelem, E0, Emin, p);
}

// Stiffness coupling between dofs da and db from the elements containing both nodes; if
// s_restrict >= 0 only elements of that subdomain contribute (subassembled A_GG,s).
__device__ __forceinline__ double stiffness_entry(const MeshDev& m, const double* __restrict__ Ee,
                                                  int da, int db, int s_restrict) {
    const int dim = m.dim;
    const int na = da / dim, ca = da - na * dim;
    const int nb = db / dim, cb = db - nb * dim;
    int ia[3], ib[3], lo[3], hi[3];
    int ra = na, rb = nb;
    for (int a = 0; a < 3; ++a) {
        ia[a] = ra % m.nn[a];
        ra /= m.nn[a];
        ib[a] = rb % m.nn[a];
        rb /= m.nn[a];
        if (a < dim) {
            const int d = ia[a] - ib[a];
            if (d > 1 || d < -1) return 0.0;
            lo[a] = max(max(ia[a], ib[a]) - 1, 0);
            hi[a] = min(min(ia[a], ib[a]), m.nel[a] - 1);
            if (lo[a] > hi[a]) return 0.0;
        } else {
            lo[a] = hi[a] = 0;
        }
    }
    double acc = 0.0;
    for (int ez = lo[2]; ez <= hi[2]; ++ez)
        for (int ey = lo[1]; ey <= hi[1]; ++ey)
            for (int ex = lo[0]; ex <= hi[0]; ++ex) {
                if (s_restrict >= 0) {
                    const int s = ex / m.sub[0] + m.ps[0] * (ey / m.sub[1] + m.ps[1] * (ez / m.sub[2]));
                    if (s != s_restrict) continue;
                }
                const int la = (ia[0] - ex) + 2 * (ia[1] - ey) + 4 * (ia[2] - ez);
                const int lb = (ib[0] - ex) + 2 * (ib[1] - ey) + 4 * (ib[2] - ez);
                const int64_t e = ex + int64_t(m.nel[0]) * (ey + int64_t(m.nel[1]) * ez);
                acc += Ee[e] * c_KE[(dim * la + ca) * m.nke + dim * lb + cb];
            }
    return acc;
}

__global__ void k_assemble_band(MeshDev m, const SubDesc* __restrict__ sd, const int32_t* __restrict__ idofs,
                                const double* __restrict__ Ee, double* __restrict__ band, int ld, int bw) {
    const SubDesc d = sd[blockIdx.y];
    const int64_t total = int64_t(d.nI) * ld;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
        const int j = int(t / ld), k = int(t - int64_t(j) * ld);
        const int r = j + k;
        double v = 0.0;
        if (k <= bw && r < d.nI) v = stiffness_entry(m, Ee, idofs[d.ioff + r], idofs[d.ioff + j], -1);
        band[d.band_off + t] = v;
        band[d.band_off + total + t] = 0.0;   // M copy (filled by the factorisation; zero padding)
    }
}

void launch_assemble_band(const MeshDev& m, const SubDesc* sd, int nsl, const int32_t* idofs,
                          const double* Ee, double* band, int ld, int band_w, int max_nI,
                          cudaStream_t st) {
    if (nsl == 0) return;
    const int64_t per = int64_t(max_nI) * ld;
    dim3 grid(unsigned(std::min<int64_t>((per + 255) / 256, 64)), nsl);
    k_assemble_band<<<grid, 256, 0, st>>>(m, sd, idofs, Ee, band, ld, band_w);
}

__global__ void k_assemble_pairs(MeshDev m, const int32_t* __restrict__ da, const int32_t* __restrict__ db,
                                 const int32_t* __restrict__ sub, const double* __restrict__ Ee,
                                 double* __restrict__ val, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        val[i] = stiffness_entry(m, Ee, da[i], db[i], sub[i]);
}

void launch_assemble_pairs(const MeshDev& m, const int32_t* da, const int32_t* db,
                           const int32_t* sub_of_entry, const double* Ee, double* val, int64_t n,
                           cudaStream_t st) {
    if (n == 0) return;
    const int blocks = int(std::min<int64_t>((n + 255) / 256, 148 * 16));
    k_assemble_pairs<<<blocks, 256, 0, st>>>(m, da, db, sub_of_entry, Ee, val, n);
}

// ---------------------------------------------------------------- B2: band Cholesky

// 32-column panels factored in shared memory; trailing update in global memory (2D and 3D; measured on c5:
// 16 ms against 39 ms for a column-at-a-time shared-memory window).
constexpr int NBP = 32;
// TU: trailing update 0 = one thread per entry (two shared loads per DFMA), 1 = FP64 tensor cores: every warp forms
// 8 x 8 tiles of the rank-32 update W[r][c] = sum_k L[r][k] L[c][k] with mma.sync.m8n8k4.f64 (row fragments of the
// panel for A, the same panel's column fragments for B: one shared load per operand element, 8 FMAs per lane per
// load pair), masked to the band, and subtracts them from the band in global memory.
template <int TU>
__global__ void __launch_bounds__(512) k_band_chol_panel(const SubDesc* __restrict__ sd, double* __restrict__ band,
                                                         int ld, int bw, int* __restrict__ fail) {
    extern __shared__ double P[];   // NBP * ld
    const SubDesc d = sd[blockIdx.x];
    const int n = d.nI;
    double* base = band + d.band_off;
    double* Mb = base + int64_t(n) * ld;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int j0 = 0; j0 < n; j0 += NBP) {
        const int nb = min(NBP, n - j0);
        for (int i = tid; i < nb * ld; i += nt) P[i] = base[int64_t(j0) * ld + i];
        __syncthreads();
        for (int jj = 0; jj < nb; ++jj) {
            double* cj = P + jj * ld;
            const double dj = cj[0];
            const bool bad = !(dj > 0.0);
            const double inv = bad ? 1.0 : 1.0 / sqrt(dj);
            if (bad && tid == 0) atomicCAS(fail, 0, d.gid + 1);
            __syncthreads();
            for (int k = tid + 1; k <= bw; k += nt) cj[k] *= inv;
            __syncthreads();
            if (tid == 0) cj[0] = inv;
            // update panel columns jj+mm (mm >= 1): rows offset r in [0, bw-mm]
            const int ncols = nb - 1 - jj;
            for (int t = tid; t < ncols * (bw + 1); t += nt) {
                const int mm = 1 + t / (bw + 1), r = t % (bw + 1);
                if (r <= bw - mm) P[(jj + mm) * ld + r] -= cj[mm + r] * cj[mm];
            }
            __syncthreads();
        }
        for (int i = tid; i < nb * ld; i += nt) base[int64_t(j0) * ld + i] = P[i];
        // M = P L^T P: row r of L is column n-1-r of M (entry L[r][j] at slot k = r - j). Written row-wise: the nb
        // entries of row r that lie in this panel are nb CONSECUTIVE slots of one M column (consecutive threads ->
        // consecutive addresses; the shared reads stride ld - 1, odd: no bank conflicts). The former per-entry write
        // (consecutive k -> stride ld - 1 in M) made the 3D factorisation move 34.7 GB of DRAM traffic for a 1.9 GB
        // factor (ncu, profiles/round2_c4_k_band_chol_panel.md).
        for (int idx = tid; idx < (bw + nb) * nb; idx += nt) {
            const int rr = idx / nb, jj = nb - 1 - (idx - rr * nb), r = j0 + rr, k = rr - jj;
            if (k >= 0 && k <= bw && r < n) Mb[int64_t(n - 1 - r) * ld + k] = P[jj * ld + k];
        }
        // trailing update of columns c in [j0+nb, j0+nb-1+bw], rows r = c + rr (rr in [0,bw])
        const int c_lo = j0 + nb, c_hi = min(j0 + nb - 1 + bw, n - 1);
        const int ncol = c_hi - c_lo + 1;
        if constexpr (TU == 1) {
            const int lane = tid & 31, wid = tid >> 5, nwarp = nt >> 5;
            const int ntc = (ncol + 7) / 8, ntr = (bw + 8 + 7) / 8 + 1;   // column tiles; row tiles per column tile
            const int ai = lane >> 2, ak = lane & 3;                      // A: row ai, k ak; B: k ak, column ai
            // TG tiles per warp in flight: the old band values are loaded first (the global read-modify-write latency
            // of one tile at a time was the whole cost of this loop: measured, the tensor-core update alone changed
            // nothing), accumulated into with the negated A fragments, and stored
            constexpr int TG = 4;
            for (int t0 = wid * TG; t0 < ntc * ntr; t0 += nwarp * TG) {
                int C0[TG], R0[TG];
                bool live[TG];
                double d0[TG], d1[TG];
#pragma unroll
                for (int g = 0; g < TG; ++g) {
                    const int t = t0 + g, tc = t / ntr, tr = t - tc * ntr;
                    C0[g] = c_lo + 8 * tc;
                    R0[g] = C0[g] + 8 * tr;               // tile rows start at the tile's first column
                    live[g] = t < ntc * ntr && R0[g] <= min(C0[g] + 7, c_hi) + bw && R0[g] < n;   // warp-uniform
                    const int r = R0[g] + ai, c = C0[g] + 2 * ak;
                    const bool w0 = live[g] && c <= c_hi && r >= c && r - c <= bw && r < n;
                    const bool w1 = live[g] && c + 1 <= c_hi && r >= c + 1 && r - c - 1 <= bw && r < n;
                    d0[g] = w0 ? base[int64_t(c) * ld + (r - c)] : 0.0;
                    d1[g] = w1 ? base[int64_t(c + 1) * ld + (r - c - 1)] : 0.0;
                }
#pragma unroll
                for (int g = 0; g < TG; ++g) {   // (k outer / g inner, interleaving the TG chains, measured slower: 67.3 vs 57.9 ms)
                    if (!live[g]) continue;      // warp-uniform
                    const int ra = R0[g] + ai, cb = C0[g] + ai;
#pragma unroll
                    for (int k0 = 0; k0 < NBP; k0 += 4) {
                        const int kk = k0 + ak, kcol = j0 + kk;
                        const int oa = ra - kcol, ob = cb - kcol;
                        const double av = (kk < nb && ra < n && oa <= bw) ? -P[kk * ld + oa] : 0.0;
                        const double bv = (kk < nb && cb <= c_hi && ob <= bw) ? P[kk * ld + ob] : 0.0;
                        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                                     : "+d"(d0[g]), "+d"(d1[g])
                                     : "d"(av), "d"(bv));
                    }
                }
#pragma unroll
                for (int g = 0; g < TG; ++g) {
                    const int r = R0[g] + ai, c = C0[g] + 2 * ak;
                    if (live[g] && c <= c_hi && r >= c && r - c <= bw && r < n) base[int64_t(c) * ld + (r - c)] = d0[g];
                    if (live[g] && c + 1 <= c_hi && r >= c + 1 && r - c - 1 <= bw && r < n) base[int64_t(c + 1) * ld + (r - c - 1)] = d1[g];
                }
            }
        } else
        for (int t = tid; t < ncol * (bw + 1); t += nt) {
            const int c = c_lo + t / (bw + 1), rr = t % (bw + 1);
            const int r = c + rr;
            if (r >= n) continue;
            double acc = 0.0;
            // panel columns k with c - k <= bw (then r - k <= bw requires k >= r - bw)
            const int kmin = max(j0, r - bw);
            for (int k = kmin; k < j0 + nb; ++k) {
                const double* pk = P + (k - j0) * ld;
                acc += pk[r - k] * pk[c - k];
            }
            if (kmin < j0 + nb) base[int64_t(c) * ld + rr] -= acc;
        }
        __syncthreads();
    }
}

int launch_band_cholesky(const SubDesc* sd, int nsl, double* band, int ld, int band_w, int* d_fail,
                         cudaStream_t st) {
    if (nsl == 0) return 0;
    const size_t smem = size_t(NBP) * ld * sizeof(double);
    // trailing update on the FP64 tensor cores (default; env DE_CHOL_SCALAR = the one-thread-per-entry update)
    // wide bands (3D) only: c4 77.7 -> 57.9 ms; on the 2D bands (b = 67: 99 tiles per panel, mostly masked) it measured
    // slower (c5 60.7 -> 70.3 ms); DE_CHOL_DMMA / DE_CHOL_SCALAR force either
    const bool dmma = getenv("DE_CHOL_SCALAR") ? false : (getenv("DE_CHOL_DMMA") ? true : band_w > 127);
    void (*fn)(const SubDesc*, double*, int, int, int*) = dmma ? k_band_chol_panel<1> : k_band_chol_panel<0>;
    raise_dyn_smem(reinterpret_cast<const void*>(fn), smem);
    fn<<<nsl, 512, smem, st>>>(sd, band, ld, band_w, d_fail);
    return 1;
}

// ---------------------------------------------------------------- true residual (matrix-free)

// Double-double helpers (error-free transformations) for an accurate residual f - K u: the
// computed residual is what iterative refinement (R11) and the reported final relres use.
struct dd_t {
    double hi, lo;
};
__device__ __forceinline__ dd_t two_sum(double a, double b) {
    const double s = a + b, bb = s - a;
    return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd_t dd_add(dd_t a, dd_t b) {
    dd_t s = two_sum(a.hi, b.hi);
    s.lo += a.lo + b.lo;
    return two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd_t dd_mul_d(dd_t a, double b) {
    const double p = a.hi * b;
    const double e = fma(a.hi, b, -p);
    return two_sum(p, e + a.lo * b);
}
__device__ __forceinline__ dd_t two_prod(double a, double b) {
    const double p = a * b;
    return {p, fma(a, b, -p)};
}

// res = f - K (u + ulo) on free dofs (0 on Dirichlet dofs): K u in double-double from the FP64 element data;
// ulo (optional, the low part of a double-double iterate, |ulo| ~ eps |u|) enters through an FP64 product
// whose rounding is ~eps^2 relative -- far below the result's own rounding
__global__ void k_apply_K(MeshDev m, const double* __restrict__ Ee, const double* __restrict__ u,
                          const double* __restrict__ ulo, const double* __restrict__ f,
                          const int8_t* __restrict__ cls, double* __restrict__ res, int64_t ndof) {
    const int dim = m.dim;
    for (int64_t d = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; d < ndof; d += int64_t(gridDim.x) * blockDim.x) {
        if (cls[d] == 2) {
            res[d] = 0.0;
            continue;
        }
        const int node = int(d / dim), c = int(d - int64_t(node) * dim);
        int co[3], r = node;
        for (int a = 0; a < 3; ++a) {
            co[a] = r % m.nn[a];
            r /= m.nn[a];
        }
        dd_t acc = {-f[d], 0.0};
        const int nz = dim == 3 ? 2 : 1;
        for (int oz = 0; oz < nz; ++oz)
            for (int oy = 0; oy < 2; ++oy)
                for (int ox = 0; ox < 2; ++ox) {
                    const int ex = co[0] - 1 + ox, ey = co[1] - 1 + oy, ez = dim == 3 ? co[2] - 1 + oz : 0;
                    if (ex < 0 || ey < 0 || ez < 0 || ex >= m.nel[0] || ey >= m.nel[1] || (dim == 3 && ez >= m.nel[2])) continue;
                    const int la = (co[0] - ex) + 2 * (co[1] - ey) + 4 * (co[2] - ez);
                    const int64_t e = ex + int64_t(m.nel[0]) * (ey + int64_t(m.nel[1]) * ez);
                    dd_t t = {0.0, 0.0};
                    double tl = 0.0;
                    for (int lb = 0; lb < (1 << dim); ++lb) {
                        const int64_t nbn = (ex + (lb & 1)) + int64_t(m.nn[0]) * ((ey + ((lb >> 1) & 1)) + int64_t(m.nn[1]) * (ez + ((lb >> 2) & 1)));
                        for (int cb = 0; cb < dim; ++cb) {
                            const double ke = c_KE[(dim * la + c) * m.nke + dim * lb + cb];
                            t = dd_add(t, two_prod(ke, u[dim * nbn + cb]));
                            if (ulo) tl = fma(ke, ulo[dim * nbn + cb], tl);
                        }
                    }
                    t.lo += tl;
                    acc = dd_add(acc, dd_mul_d(t, Ee[e]));
                }
        res[d] = -(acc.hi + acc.lo);   // f - K u, accurate to ~1 ulp of the result
    }
}

void launch_apply_K(const MeshDev& m, const double* Ee, const double* u, const double* f,
                    const int8_t* cls, double* res, int64_t ndof, cudaStream_t st, const double* ulo) {
    const int blocks = int(std::min<int64_t>((ndof + 255) / 256, 148 * 16));
    k_apply_K<<<blocks, 256, 0, st>>>(m, Ee, u, ulo, f, cls, res, ndof);
}

// (hi, lo) += d as a double-double sum (two_sum, then renormalised so hi = fl(hi + lo))
__global__ void k_dd_accum(double* __restrict__ hi, double* __restrict__ lo, const double* __restrict__ d,
                           int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const dd_t s = two_sum(hi[i], d[i]);
        const dd_t r = two_sum(s.hi, s.lo + lo[i]);
        hi[i] = r.hi;
        lo[i] = r.lo;
    }
}

void launch_dd_accum(double* hi, double* lo, const double* d, int64_t n, cudaStream_t st) {
    const int blocks = int(std::min<int64_t>((n + 255) / 256, 148 * 16));
    k_dd_accum<<<blocks, 256, 0, st>>>(hi, lo, d, n);
}

}  // namespace de
