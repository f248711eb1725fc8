// host_setup.cpp — density-independent setup of libde.
//
// A1: topology + canonical DOF map ("Gamma_i := dOmega_i \ dOmega, I := closure(Omega) \ Gamma";
//     PAPER.md:111-120 interior-first ordering with K_II block diagonal; R4/R5).
// A2: interface trace matrices M_c, L_c (component-wise per Eq. (9)) on element
//     facets separating subdomains (R6/R7), and the exact-elimination structure used by
//     the preconditioner's inner solves (faces with cross points removed; R10).
// Integer work here is bit-exact by construction; the floating-point matrices are tiny per face.
#include "de_internal.h"

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <map>
#include <numeric>

namespace de {

namespace {

// Unit-modulus Q1 element stiffness KE0 = int B^T D B over [0,h]^d with 2^d Gauss points
// (Hooke's law PAPER.md:48-55; plane stress in 2D, R2). Local node a has offsets
// (a&1, (a>>1)&1, (a>>2)&1); dofs are (node, component) component-fastest.
void compute_KE0(int dim, double nu, double h, double* KE, int& nke) {
    const double E = 1.0;
    const double mu = E / (2.0 * (1.0 + nu));
    double lam = nu * E / ((1.0 + nu) * (1.0 - 2.0 * nu));
    if (dim == 2) lam = 2.0 * mu * lam / (lam + 2.0 * mu);
    const int nv = dim == 2 ? 3 : 6;
    double D[6][6] = {{0}};
    for (int i = 0; i < dim; ++i)
        for (int j = 0; j < dim; ++j) D[i][j] = lam + (i == j ? 2.0 * mu : 0.0);
    for (int i = dim; i < nv; ++i) D[i][i] = mu;
    const int nnode = 1 << dim;
    nke = dim * nnode;
    std::fill(KE, KE + nke * nke, 0.0);
    const double g = 0.5 / std::sqrt(3.0);
    const double pts[2] = {0.5 - g, 0.5 + g};
    const double w = std::pow(h, dim) / double(nnode);
    const int shear[3][2] = {{0, 1}, {1, 2}, {0, 2}};
    const int nshear = dim == 2 ? 1 : 3;
    for (int q = 0; q < nnode; ++q) {
        double xi[3];
        for (int d = 0; d < dim; ++d) xi[d] = pts[(q >> d) & 1];
        double G[8][3];
        for (int a = 0; a < nnode; ++a)
            for (int d = 0; d < dim; ++d) {
                double v = 1.0;
                for (int e = 0; e < dim; ++e) {
                    const int o = (a >> e) & 1;
                    if (e == d) v *= o ? 1.0 : -1.0;
                    else v *= o ? xi[e] : 1.0 - xi[e];
                }
                G[a][d] = v / h;
            }
        double B[6][24] = {{0}};
        for (int a = 0; a < nnode; ++a) {
            for (int d = 0; d < dim; ++d) B[d][dim * a + d] = G[a][d];
            for (int s = 0; s < nshear; ++s) {
                const int i = shear[s][0], j = shear[s][1];
                B[dim + s][dim * a + i] = G[a][j];
                B[dim + s][dim * a + j] = G[a][i];
            }
        }
        for (int r = 0; r < nke; ++r)
            for (int c = 0; c < nke; ++c) {
                double acc = 0.0;
                for (int i = 0; i < nv; ++i) {
                    if (B[i][r] == 0.0) continue;
                    double t = 0.0;
                    for (int j = 0; j < nv; ++j) t += D[i][j] * B[j][c];
                    acc += B[i][r] * t;
                }
                KE[r * nke + c] += w * acc;
            }
    }
    for (int r = 0; r < nke; ++r)
        for (int c = r + 1; c < nke; ++c) {
            const double s = 0.5 * (KE[r * nke + c] + KE[c * nke + r]);
            KE[r * nke + c] = KE[c * nke + r] = s;
        }
}

struct Trip {
    int32_t r, c;
    double v;
};

HCsr csr_from_trips(int32_t n, std::vector<Trip>& t) {
    std::stable_sort(t.begin(), t.end(), [](const Trip& a, const Trip& b) {
        return a.r != b.r ? a.r < b.r : a.c < b.c;
    });
    HCsr A;
    A.n = A.m = n;
    A.ptr.assign(n + 1, 0);
    for (size_t i = 0; i < t.size();) {
        size_t j = i;
        double s = 0.0;
        while (j < t.size() && t[j].r == t[i].r && t[j].c == t[i].c) s += t[j++].v;
        A.col.push_back(t[i].c);
        A.val.push_back(s);
        A.ptr[t[i].r + 1]++;
        i = j;
    }
    for (int32_t i = 0; i < n; ++i) A.ptr[i + 1] += A.ptr[i];
    return A;
}

int32_t find_root(std::vector<int32_t>& p, int32_t x) {
    while (p[x] != x) {
        p[x] = p[p[x]];
        x = p[x];
    }
    return x;
}

// Band Cholesky of a small dense SPD matrix (row-major n x n) with half bandwidth b; stores the
// factor column-band (ld = b+1), slot 0 = 1/L_jj. Returns false on a non-positive pivot.
bool small_band_cholesky(int n, int b, std::vector<double> A, double* out) {
    const int ld = b + 1;
    for (int j = 0; j < n; ++j) {
        double d = A[j * n + j];
        if (!(d > 0.0)) return false;
        const double l = std::sqrt(d);
        out[j * ld] = 1.0 / l;
        for (int k = 1; k <= b; ++k) {
            const int r = j + k;
            const double v = r < n ? A[r * n + j] / l : 0.0;
            out[j * ld + k] = v;
            if (r < n) A[r * n + j] = v;
        }
        for (int k1 = 1; k1 <= b && j + k1 < n; ++k1)
            for (int k2 = 1; k2 <= k1; ++k2)
                A[(j + k1) * n + (j + k2)] -= A[(j + k1) * n + j] * A[(j + k2) * n + j];
    }
    return true;
}

// Solve (L L^T) x = rhs with the column-band factor above (host, tiny systems).
void small_band_solve(int n, int b, const double* fac, double* x) {
    const int ld = b + 1;
    for (int j = 0; j < n; ++j) {
        x[j] *= fac[j * ld];
        for (int k = 1; k <= b && j + k < n; ++k) x[j + k] -= fac[j * ld + k] * x[j];
    }
    for (int j = n - 1; j >= 0; --j) {
        double t = x[j];
        for (int k = 1; k <= b && j + k < n; ++k) t -= fac[j * ld + k] * x[j + k];
        x[j] = t * fac[j * ld];
    }
}

// Eigen-decomposition of a symmetric n x n matrix (row-major A, destroyed) by cyclic Jacobi: A = Q diag(lam) Q^T,
// Q row-major [i][a]. Setup only (n = cross points per skeleton line).
void sym_eig_jacobi(int n, std::vector<double>& A, std::vector<double>& Q, std::vector<double>& lam) {
    Q.assign(size_t(n) * n, 0.0);
    for (int i = 0; i < n; ++i) Q[size_t(i) * n + i] = 1.0;
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0, dia = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) (i == j ? dia : off) += A[size_t(i) * n + j] * A[size_t(i) * n + j];
        if (off <= 1e-32 * dia) break;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = A[size_t(p) * n + q];
                if (apq == 0.0) continue;
                const double d = A[size_t(q) * n + q] - A[size_t(p) * n + p];
                const double t = (d >= 0.0 ? 2.0 : -2.0) * apq / (std::fabs(d) + std::sqrt(d * d + 4.0 * apq * apq));
                const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = t * cs;
                for (int k = 0; k < n; ++k) {   // columns p, q of A and Q
                    const double x = A[size_t(k) * n + p], y = A[size_t(k) * n + q];
                    A[size_t(k) * n + p] = cs * x - sn * y;
                    A[size_t(k) * n + q] = sn * x + cs * y;
                    const double u = Q[size_t(k) * n + p], v = Q[size_t(k) * n + q];
                    Q[size_t(k) * n + p] = cs * u - sn * v;
                    Q[size_t(k) * n + q] = sn * u + cs * v;
                }
                for (int k = 0; k < n; ++k) {   // rows p, q of A
                    const double x = A[size_t(p) * n + k], y = A[size_t(q) * n + k];
                    A[size_t(p) * n + k] = cs * x - sn * y;
                    A[size_t(q) * n + k] = sn * x + cs * y;
                }
            }
    }
    lam.resize(n);
    for (int i = 0; i < n; ++i) lam[i] = A[size_t(i) * n + i];
}

// Fast-diagonalisation tables of a separable S_C (HElim::fd; R23). Leaves E.fd = 0 unless every
// component's cross points form a full tensor grid in index order and its dense S_C equals the Kronecker sum
// A_x (x) I + I (x) A_y entry by entry (relative 1e-13), with every lam_a + mu_b > 0.
void detect_fd(const HostSetup& hs, HElim& E) {
    E.fd = 0;
    // Opt-in (env DE_FD=1): measured on B200 (c5) the redundant per-block forward transforms cost 11.4 us per
    // elimination against 6.7 us for the dense S_C^-1 GEMV stream, although they save 0.3 GB of DRAM traffic per
    // application (R23)
    if (hs.dim != 2 || E.ncross == 0 || !getenv("DE_FD")) return;
    const int nstore = E.sc_shared ? 1 : hs.ncomp;
    int nx = 0, ny = 0;
    std::vector<double> qx, qy, il;
    for (int c = 0; c < hs.ncomp; ++c) {
        const int32_t base = E.cross_comp_off[c], nc = E.cross_comp_off[c + 1] - base;
        if (nc < 4) return;
        std::vector<int> xs, ys;
        for (int k = 0; k < nc; ++k) {
            const int64_t node = hs.cnode[E.cross_flat[base + k]];
            xs.push_back(int(node % hs.nn[0]));
            ys.push_back(int(node / hs.nn[0]));
        }
        std::vector<int> ux(xs), uy(ys);
        std::sort(ux.begin(), ux.end());
        ux.erase(std::unique(ux.begin(), ux.end()), ux.end());
        std::sort(uy.begin(), uy.end());
        uy.erase(std::unique(uy.begin(), uy.end()), uy.end());
        const int cnx = int(ux.size()), cny = int(uy.size());
        if (int64_t(cnx) * cny != nc || (c > 0 && (cnx != nx || cny != ny))) return;
        nx = cnx;
        ny = cny;
        for (int k = 0; k < nc; ++k)
            if (xs[k] != ux[k % nx] || ys[k] != uy[k / nx]) return;
        if (c >= nstore) continue;   // shared S_C: tables of component 0 only (grid layout checked for all)
        const double* S = &E.SC[E.sc_off[c]];
        auto at = [&](int ix, int iy, int jx, int jy) { return S[size_t(ix + nx * iy) * nc + (jx + nx * jy)]; };
        std::vector<double> Ax(size_t(nx) * nx, 0.0), Ay(size_t(ny) * ny, 0.0);
        const double d00 = at(0, 0, 0, 0);
        for (int ix = 0; ix < nx; ++ix) {
            Ax[size_t(ix) * nx + ix] = at(ix, 0, ix, 0) - 0.5 * d00;
            if (ix + 1 < nx) Ax[size_t(ix) * nx + ix + 1] = Ax[size_t(ix + 1) * nx + ix] = at(ix, 0, ix + 1, 0);
        }
        for (int iy = 0; iy < ny; ++iy) {
            Ay[size_t(iy) * ny + iy] = at(0, iy, 0, iy) - 0.5 * d00;
            if (iy + 1 < ny) Ay[size_t(iy) * ny + iy + 1] = Ay[size_t(iy + 1) * ny + iy] = at(0, iy, 0, iy + 1);
        }
        double smax = 0.0;
        for (size_t e = 0; e < size_t(nc) * nc; ++e) smax = std::max(smax, std::fabs(S[e]));
        for (int iy = 0; iy < ny; ++iy)
            for (int ix = 0; ix < nx; ++ix)
                for (int jy = 0; jy < ny; ++jy)
                    for (int jx = 0; jx < nx; ++jx) {
                        const double want = (iy == jy ? Ax[size_t(ix) * nx + jx] : 0.0) + (ix == jx ? Ay[size_t(iy) * ny + jy] : 0.0);
                        if (std::fabs(at(ix, iy, jx, jy) - want) > 1e-13 * smax) return;
                    }
        std::vector<double> Qx, Qy, lam, mu;
        sym_eig_jacobi(nx, Ax, Qx, lam);
        sym_eig_jacobi(ny, Ay, Qy, mu);
        for (int b = 0; b < ny; ++b)
            for (int a = 0; a < nx; ++a) {
                const double s = lam[a] + mu[b];
                if (!(s > 1e-12 * smax)) return;
                il.push_back(1.0 / s);
            }
        qx.insert(qx.end(), Qx.begin(), Qx.end());
        qy.insert(qy.end(), Qy.begin(), Qy.end());
    }
    E.fd = 1;
    E.fd_nx = nx;
    E.fd_ny = ny;
    E.fd_qx.swap(qx);
    E.fd_qy.swap(qy);
    E.fd_il.swap(il);
}

de_status_t build_elim(const HostSetup& hs, const HCsr& X, HElim& E) {
    // faces: grouped per component in (component, face id) order; nodes ascending
    const int64_t nflat = hs.comp_off[hs.ncomp];
    std::vector<int32_t> face_slot(nflat, -1);   // flat -> slot in face_nodes
    std::vector<int32_t> cross_idx(nflat, -1);
    E.face_off.assign(1, 0);
    E.face_nodes.clear();
    for (int c = 0; c < hs.ncomp; ++c) {
        const int nf = int(hs.n_faces_c[c]);
        std::vector<std::vector<int32_t>> faces(nf);
        for (int64_t f = hs.comp_off[c]; f < hs.comp_off[c + 1]; ++f)
            if (hs.face_of[f] >= 0) faces[hs.face_of[f]].push_back(int32_t(f));
        for (auto& fn : faces) {
            for (auto f : fn) {
                face_slot[f] = int32_t(E.face_nodes.size());
                E.face_nodes.push_back(f);
            }
            E.face_off.push_back(int32_t(E.face_nodes.size()));
        }
    }
    E.nfaces = int32_t(E.face_off.size()) - 1;
    E.cross_flat.clear();
    E.cross_comp_off[0] = 0;
    for (int c = 0; c < hs.ncomp; ++c) {
        for (int64_t f = hs.comp_off[c]; f < hs.comp_off[c + 1]; ++f)
            if (hs.face_of[f] < 0) {
                cross_idx[f] = int32_t(E.cross_flat.size());
                E.cross_flat.push_back(int32_t(f));
            }
        E.cross_comp_off[c + 1] = int32_t(E.cross_flat.size());
    }
    for (int c = hs.ncomp; c < MAXC; ++c) E.cross_comp_off[c + 1] = E.cross_comp_off[hs.ncomp];
    E.ncross = int32_t(E.cross_flat.size());
    // X_CF (rows cross points) and X_FC (rows face slots)
    std::vector<Trip> tcf, tfc;
    for (int32_t ci = 0; ci < E.ncross; ++ci) {
        const int32_t f = E.cross_flat[ci];
        for (int32_t k = X.ptr[f]; k < X.ptr[f + 1]; ++k)
            if (face_slot[X.col[k]] >= 0) tcf.push_back({ci, X.col[k], X.val[k]});
    }
    for (int32_t sl = 0; sl < int32_t(E.face_nodes.size()); ++sl) {
        const int32_t f = E.face_nodes[sl];
        for (int32_t k = X.ptr[f]; k < X.ptr[f + 1]; ++k)
            if (cross_idx[X.col[k]] >= 0) tfc.push_back({sl, cross_idx[X.col[k]], X.val[k]});
    }
    E.XCF = csr_from_trips(E.ncross, tcf);
    E.XCF.m = int32_t(nflat);
    E.XFC = csr_from_trips(int32_t(E.face_nodes.size()), tfc);
    E.XFC.m = E.ncross;
    // per-face band factors
    E.face_band.assign(E.nfaces, 0);
    E.face_fac_off.assign(E.nfaces + 1, 0);
    std::vector<std::vector<double>> dense(E.nfaces);
    for (int32_t F = 0; F < E.nfaces; ++F) {
        const int32_t o = E.face_off[F], n = E.face_off[F + 1] - o;
        std::vector<double> A(size_t(n) * n, 0.0);
        int b = 0;
        for (int32_t i = 0; i < n; ++i) {
            const int32_t f = E.face_nodes[o + i];
            for (int32_t k = X.ptr[f]; k < X.ptr[f + 1]; ++k) {
                const int32_t s = face_slot[X.col[k]];
                if (s >= o && s < o + n) {
                    A[size_t(i) * n + (s - o)] = X.val[k];
                    b = std::max(b, std::abs(s - o - i));
                }
            }
        }
        E.face_band[F] = b;
        E.face_fac_off[F + 1] = E.face_fac_off[F] + 2 * int64_t(n) * (b + 1);   // [L | M = P L^T P]
        dense[F].swap(A);
    }
    E.face_fac.assign(E.face_fac_off[E.nfaces], 0.0);
    for (int32_t F = 0; F < E.nfaces; ++F) {
        const int32_t n = E.face_off[F + 1] - E.face_off[F], b = E.face_band[F], ld = b + 1;
        double* Lf = &E.face_fac[E.face_fac_off[F]];
        if (!small_band_cholesky(n, b, dense[F], Lf)) {
            set_error("face block %d of the interface operator is not SPD", F);
            return DE_EINVAL;
        }
        double* Mf = Lf + size_t(n) * ld;   // column j' of M = row n-1-j' of L, reversed
        for (int32_t j = 0; j < n; ++j)
            for (int k = 0; k <= b && j + k < n; ++k) Mf[size_t(n - 1 - j - k) * ld + k] = Lf[size_t(j) * ld + k];
    }
    // block-bidiagonal form of the 3D face factors (HElim::fb)
    E.fb_off.clear();
    E.fb.clear();
    {
        int maxb = 0;
        for (int32_t F = 0; F < E.nfaces; ++F) maxb = std::max(maxb, E.face_band[F]);
        // opt-in (env DE_FB=1): measured on c4 the block form does not shorten the first face phase (25-27 us against
        // 27-28 us: 16 steps, each waiting for its 2 KB of block matrices from L2, cost what 2 x 121 shuffle rows cost)
        // and it takes 58 MB per operator
        if (hs.dim == 3 && maxb > 1 && maxb <= FB_BS && getenv("DE_FB")) {
            constexpr int BS = FB_BS;
            E.fb_off.assign(1, 0);
            std::vector<double> D(BS * BS), Ei(BS * BS), En(BS * BS), Fi(BS * BS);
            for (int32_t F = 0; F < E.nfaces; ++F) {
                const int32_t n = E.face_off[F + 1] - E.face_off[F], b = E.face_band[F], ld = b + 1;
                const double* Lf = &E.face_fac[E.face_fac_off[F]];
                auto Lent = [&](int r, int c) -> double {   // L[r][c], r >= c
                    if (r >= n || c >= n) return r == c ? 1.0 : 0.0;
                    if (r == c) return 1.0 / Lf[size_t(c) * ld];
                    return (r > c && r - c <= b) ? Lf[size_t(c) * ld + (r - c)] : 0.0;
                };
                const int nbk = (n + BS - 1) / BS;
                for (int i = 0; i < nbk; ++i) {
                    for (int r = 0; r < BS; ++r)
                        for (int c = 0; c < BS; ++c) {
                            D[r * BS + c] = r >= c ? Lent(BS * i + r, BS * i + c) : 0.0;
                            Ei[r * BS + c] = i > 0 ? Lent(BS * i + r, BS * (i - 1) + c) : 0.0;
                            En[r * BS + c] = i + 1 < nbk ? Lent(BS * (i + 1) + r, BS * i + c) : 0.0;   // E_{i+1}
                        }
                    for (int c = 0; c < BS; ++c)   // F = D^-1 column by column (forward substitution)
                        for (int r = 0; r < BS; ++r) {
                            double t = r == c ? 1.0 : 0.0;
                            for (int k = c; k < r; ++k) t -= D[r * BS + k] * Fi[k * BS + c];
                            Fi[r * BS + c] = r < c ? 0.0 : t / D[r * BS + r];
                        }
                    const size_t at = E.fb.size();
                    E.fb.resize(at + 4 * BS * BS, 0.0);
                    double* o = &E.fb[at];
                    for (int r = 0; r < BS; ++r)
                        for (int c = 0; c < BS; ++c) {
                            double g = 0.0, h = 0.0;
                            for (int k = 0; k < BS; ++k) {
                                g += Fi[r * BS + k] * Ei[k * BS + c];          // G = F E_i
                                h += Fi[k * BS + r] * En[c * BS + k];          // H = F^T E_{i+1}^T
                            }
                            o[0 * BS * BS + c * BS + r] = Fi[r * BS + c];
                            o[1 * BS * BS + c * BS + r] = g;
                            o[2 * BS * BS + c * BS + r] = Fi[c * BS + r];      // F^T
                            o[3 * BS * BS + c * BS + r] = h;
                        }
                }
                E.fb_off.push_back(E.fb_off.back() + nbk);
            }
        }
    }
    // dense cross-point Schur complements S_C = X_CC - X_CF X_FF^-1 X_FC per component
    E.sc_off.assign(hs.ncomp + 1, 0);
    for (int c = 0; c < hs.ncomp; ++c) {
        const int64_t nc = E.cross_comp_off[c + 1] - E.cross_comp_off[c];
        E.sc_off[c + 1] = E.sc_off[c] + nc * nc;
    }
    E.SC.assign(E.sc_off[hs.ncomp], 0.0);
    auto comp_of_cross = [&](int32_t ci) {
        int c = 0;
        while (ci >= E.cross_comp_off[c + 1]) ++c;
        return c;
    };
    for (int32_t ci = 0; ci < E.ncross; ++ci) {
        const int c = comp_of_cross(ci);
        const int32_t base = E.cross_comp_off[c];
        const int64_t nc = E.cross_comp_off[c + 1] - base;
        const int32_t f = E.cross_flat[ci];
        for (int32_t k = X.ptr[f]; k < X.ptr[f + 1]; ++k) {
            const int32_t cj = cross_idx[X.col[k]];
            if (cj >= 0) E.SC[E.sc_off[c] + int64_t(ci - base) * nc + (cj - base)] += X.val[k];
        }
    }
    std::vector<double> g;
    const bool keep_g = hs.dim == 3 && !getenv("DE_NO_G3");
    E.g3_off.assign(1, 0);
    E.g3.clear();
    E.g3_adj_ptr.assign(1, 0);
    E.g3_adj.clear();
    for (int32_t F = 0; F < E.nfaces; ++F) {
        const int32_t o = E.face_off[F], n = E.face_off[F + 1] - o;
        std::vector<int32_t> adj;
        for (int32_t i = 0; i < n; ++i)
            for (int32_t k = E.XFC.ptr[o + i]; k < E.XFC.ptr[o + i + 1]; ++k) adj.push_back(E.XFC.col[k]);
        std::sort(adj.begin(), adj.end());
        adj.erase(std::unique(adj.begin(), adj.end()), adj.end());
        if (keep_g) {
            E.g3_adj.insert(E.g3_adj.end(), adj.begin(), adj.end());
            E.g3_adj_ptr.push_back(int32_t(E.g3_adj.size()));
            E.g3_off.push_back(E.g3_off.back() + int64_t(n) * int64_t(adj.size()));
        }
        if (adj.empty()) continue;
        const int na = int(adj.size());
        std::vector<double> XF(size_t(n) * na, 0.0);   // X_F,adj (column-major: col e contiguous)
        for (int32_t i = 0; i < n; ++i)
            for (int32_t k = E.XFC.ptr[o + i]; k < E.XFC.ptr[o + i + 1]; ++k) {
                const int e = int(std::lower_bound(adj.begin(), adj.end(), E.XFC.col[k]) - adj.begin());
                XF[size_t(e) * n + i] = E.XFC.val[k];
            }
        const int c = comp_of_cross(adj[0]);
        const int32_t base = E.cross_comp_off[c];
        const int64_t nc = E.cross_comp_off[c + 1] - base;
        g.assign(n, 0.0);
        for (int e = 0; e < na; ++e) {
            for (int32_t i = 0; i < n; ++i) g[i] = XF[size_t(e) * n + i];
            small_band_solve(n, E.face_band[F], &E.face_fac[E.face_fac_off[F]], g.data());
            if (keep_g) E.g3.insert(E.g3.end(), g.begin(), g.end());   // column e of G_F
            for (int e2 = 0; e2 < na; ++e2) {
                double t = 0.0;
                for (int32_t i = 0; i < n; ++i) t += XF[size_t(e2) * n + i] * g[i];
                E.SC[E.sc_off[c] + int64_t(adj[e2] - base) * nc + (adj[e] - base)] -= t;
            }
        }
    }
    // identical components (e.g. every component clamped on the same Dirichlet face): keep one S_C
    E.sc_shared = hs.ncomp > 1 ? 1 : 0;
    for (int c = 1; c < hs.ncomp && E.sc_shared; ++c)
        if (E.sc_off[c + 1] - E.sc_off[c] != E.sc_off[1] - E.sc_off[0] ||
            !std::equal(E.SC.begin() + E.sc_off[c], E.SC.begin() + E.sc_off[c + 1], E.SC.begin()))
            E.sc_shared = 0;
    if (getenv("DE_NO_SC_SHARE")) E.sc_shared = 0;   // A/B switch
    detect_fd(hs, E);
    return DE_OK;
}

}  // namespace

de_status_t host_setup(const de_mesh_t* mesh, const de_partition_t* part, double nu,
                       HostSetup& hs) {
    hs.dim = mesh->dim;
    if (hs.dim != 2 && hs.dim != 3) {
        set_error("dim must be 2 or 3");
        return DE_EINVAL;
    }
    const int dim = hs.dim;
    hs.h = mesh->h;
    hs.nnodes = 1;
    hs.nelem = 1;
    hs.nsub = 1;
    for (int a = 0; a < 3; ++a) {
        hs.nel[a] = a < dim ? mesh->nel[a] : 1;
        hs.sub[a] = a < dim ? part->sub[a] : 1;
        if (a >= dim) {
            hs.nn[a] = 1;
            hs.ps[a] = 1;
            continue;
        }
        if (hs.nel[a] < 1 || hs.sub[a] < 1 || hs.nel[a] % hs.sub[a]) {
            set_error("partition does not divide the mesh along axis %d (nel=%d, sub=%d)", a,
                      hs.nel[a], hs.sub[a]);
            return DE_EINVAL;
        }
        hs.nn[a] = hs.nel[a] + 1;
        hs.ps[a] = hs.nel[a] / hs.sub[a];
        hs.nnodes *= hs.nn[a];
        hs.nelem *= hs.nel[a];
        hs.nsub *= hs.ps[a];
    }
    hs.ndof = dim * hs.nnodes;
    if (hs.ndof >= (int64_t(1) << 31)) {
        set_error("mesh too large for int32 dof indexing");
        return DE_EINVAL;
    }
    compute_KE0(dim, nu, hs.h, hs.KE0, hs.nke);

    // ---- A1: subdomains touching each node (per-axis slabs, product over axes)
    hs.node_nsub.assign(hs.nnodes, 0);
    hs.node_subs.assign(hs.nnodes * 8, -1);
    for (int64_t node = 0; node < hs.nnodes; ++node) {
        int64_t rem = node;
        int ids[3][2], cnt[3];
        for (int a = 0; a < 3; ++a) {
            const int i = int(rem % hs.nn[a]);
            rem /= hs.nn[a];
            cnt[a] = 0;
            if (a >= dim) {
                ids[a][cnt[a]++] = 0;
                continue;
            }
            const int lo = i > 0 ? (i - 1) / hs.sub[a] : -1;
            const int hi = i < hs.nel[a] ? i / hs.sub[a] : -1;
            if (lo >= 0) ids[a][cnt[a]++] = lo;
            if (hi >= 0 && hi != lo) ids[a][cnt[a]++] = hi;
        }
        int t = 0;
        for (int z = 0; z < cnt[2]; ++z)
            for (int y = 0; y < cnt[1]; ++y)
                for (int x = 0; x < cnt[0]; ++x)
                    hs.node_subs[node * 8 + t++] = ids[0][x] + hs.ps[0] * (ids[1][y] + hs.ps[1] * ids[2][z]);
        hs.node_nsub[node] = t;
    }
    // ---- per-dof classes (Dirichlet wins, then >= 2 subdomains -> Gamma)
    bool any_fixed = false;
    hs.cls.assign(hs.ndof, 0);
    hs.dof_sub.assign(hs.ndof, -1);
    for (int64_t d = 0; d < hs.ndof; ++d) {
        const int64_t node = d / dim;
        if (mesh->fixed[d]) {
            hs.cls[d] = 2;
            any_fixed = true;
        } else if (hs.node_nsub[node] >= 2) {
            hs.cls[d] = 1;
        } else {
            hs.cls[d] = 0;
            hs.dof_sub[d] = hs.node_subs[node * 8];
        }
    }
    if (!any_fixed) {
        set_error("no Dirichlet dof: the elasticity operator is singular");
        return DE_EINVAL;
    }
    // ---- canonical numbering: interior dofs by (s, dof), then Gamma dofs by dof
    hs.nI.assign(hs.nsub, 0);
    for (int64_t d = 0; d < hs.ndof; ++d)
        if (hs.cls[d] == 0) hs.nI[hs.dof_sub[d]]++;
    hs.ioff.assign(hs.nsub + 1, 0);
    for (int s = 0; s < hs.nsub; ++s) hs.ioff[s + 1] = hs.ioff[s] + hs.nI[s];
    hs.n_I = hs.ioff[hs.nsub];
    hs.idofs.assign(hs.n_I, -1);
    hs.lidx.assign(hs.ndof, -1);
    hs.reduced.assign(hs.ndof, -1);
    hs.gpos.assign(hs.ndof, -1);
    hs.gamma_dofs.clear();
    {
        std::vector<int64_t> fill(hs.ioff.begin(), hs.ioff.end() - 1);
        for (int64_t d = 0; d < hs.ndof; ++d) {
            if (hs.cls[d] == 0) {
                const int s = hs.dof_sub[d];
                hs.lidx[d] = int32_t(fill[s] - hs.ioff[s]);
                hs.reduced[d] = int32_t(fill[s]);
                hs.idofs[fill[s]++] = int32_t(d);
            } else if (hs.cls[d] == 1) {
                hs.gpos[d] = int32_t(hs.gamma_dofs.size());
                hs.gamma_dofs.push_back(int32_t(d));
            }
        }
    }
    hs.n_G = int64_t(hs.gamma_dofs.size());
    hs.n_free = hs.n_I + hs.n_G;
    for (int64_t g = 0; g < hs.n_G; ++g) hs.reduced[hs.gamma_dofs[g]] = int32_t(hs.n_I + g);
    // ---- Gamma dofs touched by each subdomain (ascending dof)
    hs.nGs.assign(hs.nsub, 0);
    for (int64_t g = 0; g < hs.n_G; ++g) {
        const int64_t node = hs.gamma_dofs[g] / dim;
        for (int t = 0; t < hs.node_nsub[node]; ++t) hs.nGs[hs.node_subs[node * 8 + t]]++;
    }
    hs.goff.assign(hs.nsub + 1, 0);
    for (int s = 0; s < hs.nsub; ++s) hs.goff[s + 1] = hs.goff[s] + hs.nGs[s];
    hs.gdofs.assign(hs.goff[hs.nsub], -1);
    {
        std::vector<int64_t> fill(hs.goff.begin(), hs.goff.end() - 1);
        for (int64_t g = 0; g < hs.n_G; ++g) {
            const int64_t node = hs.gamma_dofs[g] / dim;
            for (int t = 0; t < hs.node_nsub[node]; ++t) {
                const int s = hs.node_subs[node * 8 + t];
                hs.gdofs[fill[s]++] = hs.gamma_dofs[g];
            }
        }
    }
    // ---- half bandwidth of every A_II,s in local lexicographic order
    hs.band_s.assign(hs.nsub, 0);
    hs.band = 0;
    for (int64_t d = 0; d < hs.ndof; ++d) {
        if (hs.cls[d] != 0) continue;
        const int s = hs.dof_sub[d];
        const int64_t node = d / dim;
        int co[3];
        int64_t rem = node;
        for (int a = 0; a < 3; ++a) {
            co[a] = int(rem % hs.nn[a]);
            rem /= hs.nn[a];
        }
        const int a0 = hs.lidx[d];
        for (int dz = (dim == 3 ? -1 : 0); dz <= (dim == 3 ? 1 : 0); ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int x = co[0] + dx, y = co[1] + dy, z = co[2] + dz;
                    if (x < 0 || y < 0 || z < 0 || x >= hs.nn[0] || y >= hs.nn[1] || z >= hs.nn[2]) continue;
                    const int64_t nb = x + int64_t(hs.nn[0]) * (y + int64_t(hs.nn[1]) * z);
                    for (int c = 0; c < dim; ++c) {
                        const int64_t e = dim * nb + c;
                        if (hs.cls[e] == 0 && hs.dof_sub[e] == s && hs.lidx[e] < a0)
                            hs.band_s[s] = std::max(hs.band_s[s], a0 - hs.lidx[e]);
                    }
                }
    }
    for (int s = 0; s < hs.nsub; ++s) hs.band = std::max(hs.band, hs.band_s[s]);
    hs.ld = (hs.band + 1 + 1) & ~1;   // even => 16-byte aligned columns for bulk copies

    // ---- A2: component skeletons
    hs.ncomp = dim;
    hs.cmap.clear();
    hs.cnode.clear();
    hs.face_of.clear();
    hs.comp_off[0] = 0;
    hs.flat_of.assign(hs.ndof, -1);   // Gamma dof -> flat index
    std::vector<int32_t>& flat_of = hs.flat_of;
    for (int c = 0; c < dim; ++c) {
        std::map<std::pair<int32_t, int32_t>, int32_t> fid;
        // first pass: face keys in ascending key order
        for (int64_t node = 0; node < hs.nnodes; ++node) {
            const int64_t d = dim * node + c;
            if (hs.cls[d] == 1 && hs.node_nsub[node] == 2)
                fid[{hs.node_subs[node * 8], hs.node_subs[node * 8 + 1]}] = 0;
        }
        int32_t k = 0;
        for (auto& kv : fid) kv.second = k++;
        hs.n_faces_c[c] = k;
        hs.n_cross_c[c] = 0;
        for (int64_t node = 0; node < hs.nnodes; ++node) {
            const int64_t d = dim * node + c;
            if (hs.cls[d] != 1) continue;
            flat_of[d] = int32_t(hs.cmap.size());
            hs.cmap.push_back(hs.gpos[d]);
            hs.cnode.push_back(int32_t(node));
            if (hs.node_nsub[node] == 2) {
                hs.face_of.push_back(fid[{hs.node_subs[node * 8], hs.node_subs[node * 8 + 1]}]);
            } else {
                hs.face_of.push_back(-1);
                hs.n_cross_c[c]++;
            }
        }
        hs.comp_off[c + 1] = int64_t(hs.cmap.size());
        {   // face-major flattened order inside the component: faces by id (nodes ascending, i.e. along the
            // face), then the cross points; the nodes of a face are then contiguous (coalesced face-mapped work)
            const int64_t lo = hs.comp_off[c], n = hs.comp_off[c + 1] - lo;
            std::vector<int64_t> ord(n);
            std::iota(ord.begin(), ord.end(), 0);
            auto key = [&](int64_t q) { return hs.face_of[lo + q] < 0 ? INT32_MAX : hs.face_of[lo + q]; };
            std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return key(a) < key(b); });
            std::vector<int32_t> cm(n), cn(n), fo(n);
            for (int64_t q = 0; q < n; ++q) {
                cm[q] = hs.cmap[lo + ord[q]];
                cn[q] = hs.cnode[lo + ord[q]];
                fo[q] = hs.face_of[lo + ord[q]];
            }
            for (int64_t q = 0; q < n; ++q) {
                hs.cmap[lo + q] = cm[q];
                hs.cnode[lo + q] = cn[q];
                hs.face_of[lo + q] = fo[q];
                flat_of[int64_t(dim) * cn[q] + c] = int32_t(lo + q);
            }
        }
    }
    for (int c = dim; c < MAXC; ++c) hs.comp_off[c + 1] = hs.comp_off[dim];
    return build_trace(hs, hs.trace_E.empty() ? nullptr : hs.trace_E.data());
}

// Trace matrices M, L (and K), singular components, and the exact-elimination structures of K and M.
// Ee == nullptr: unweighted (R6); else every facet element is scaled by (E_a + E_b)/2 of its two adjacent
// elements (NEXT(3), R19). Re-run by de_factor when the weighted norm must follow new densities.
de_status_t build_trace(HostSetup& hs, const double* Ee) {
    const int dim = hs.dim;
    const std::vector<int32_t>& flat_of = hs.flat_of;
    const int32_t nflat = int32_t(hs.comp_off[dim]);

    // ---- trace facets (R6): element facets whose two elements lie in different subdomains
    double m1[2][2], k1[2][2];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) {
            m1[i][j] = hs.h / 6.0 * (i == j ? 2.0 : 1.0);
            k1[i][j] = (i == j ? 1.0 : -1.0) / hs.h;
        }
    const int nfn = 1 << (dim - 1);
    double Mf[4][4], Lf[4][4];
    for (int a = 0; a < nfn; ++a)
        for (int b = 0; b < nfn; ++b) {
            if (dim == 2) {
                Mf[a][b] = m1[a][b];
                Lf[a][b] = k1[a][b];
            } else {   // facet nodes (o_b, o_c) -> o_b + 2 o_c ; tensor product
                const int ab = a & 1, ac = a >> 1, bb = b & 1, bc = b >> 1;
                Mf[a][b] = m1[ac][bc] * m1[ab][bb];
                Lf[a][b] = k1[ac][bc] * m1[ab][bb] + m1[ac][bc] * k1[ab][bb];
            }
        }
    std::vector<Trip> tM, tL;
    std::vector<int32_t> uf(hs.nnodes);
    std::iota(uf.begin(), uf.end(), 0);
    std::vector<uint8_t> is_trace(hs.nnodes, 0);
    auto esub = [&](const int* e) {
        return (e[0] / hs.sub[0]) + hs.ps[0] * ((e[1] / hs.sub[1]) + hs.ps[1] * (e[2] / hs.sub[2]));
    };
    for (int a = 0; a < dim; ++a) {
        for (int64_t el = 0; el < hs.nelem; ++el) {
            int e[3];
            int64_t rem = el;
            for (int t = 0; t < 3; ++t) {
                e[t] = int(rem % hs.nel[t]);
                rem /= hs.nel[t];
            }
            if (e[a] >= hs.nel[a] - 1) continue;
            int e2[3] = {e[0], e[1], e[2]};
            e2[a]++;
            if (esub(e) == esub(e2)) continue;
            int64_t stride = 1;
            for (int t2 = 0; t2 < a; ++t2) stride *= hs.nel[t2];
            const double wgt = Ee ? 0.5 * (Ee[el] + Ee[el + stride]) : 1.0;
            // facet nodes: offsets with o_a = 1, lexicographic in remaining axes
            int64_t fn[4];
            int t = 0;
            for (int o = 0; o < (1 << dim); ++o) {
                if (((o >> a) & 1) == 0) continue;
                const int x = e[0] + (o & 1), y = e[1] + ((o >> 1) & 1), z = e[2] + ((o >> 2) & 1);
                fn[t++] = x + int64_t(hs.nn[0]) * (y + int64_t(hs.nn[1]) * z);
            }
            for (int i = 0; i < nfn; ++i) {
                is_trace[fn[i]] = 1;
                const int32_t ri = find_root(uf, int32_t(fn[i])), r0 = find_root(uf, int32_t(fn[0]));
                if (ri != r0) uf[ri] = r0;
            }
            for (int c = 0; c < dim; ++c)
                for (int i = 0; i < nfn; ++i) {
                    const int32_t fi = flat_of[dim * fn[i] + c];
                    if (fi < 0) continue;
                    for (int j = 0; j < nfn; ++j) {
                        const int32_t fj = flat_of[dim * fn[j] + c];
                        if (fj < 0) continue;
                        tM.push_back({fi, fj, wgt * Mf[i][j]});
                        tL.push_back({fi, fj, wgt * Lf[i][j]});
                    }
                }
        }
    }
    // every Gamma_c node must be a trace node (R6)
    for (int32_t f = 0; f < nflat; ++f)
        if (!is_trace[hs.cnode[f]]) {
            set_error("internal: Gamma node %d is on no trace facet", hs.cnode[f]);
            return DE_EINVAL;
        }
    // singular components (R7): a connected trace piece with no Dirichlet node of component c
    hs.singular_mask = 0;
    for (int c = 0; c < dim; ++c) {
        std::vector<uint8_t> root_has_d(hs.nnodes, 0);
        for (int64_t node = 0; node < hs.nnodes; ++node)
            if (is_trace[node] && hs.cls[dim * node + c] == 2) root_has_d[find_root(uf, int32_t(node))] = 1;
        for (int64_t node = 0; node < hs.nnodes; ++node)
            if (is_trace[node] && !root_has_d[find_root(uf, int32_t(node))]) {
                hs.singular_mask |= 1 << c;
                break;
            }
    }
    hs.M = csr_from_trips(nflat, tM);
    hs.L = csr_from_trips(nflat, tL);
    hs.elimK = HElim();
    hs.elimM = HElim();
    if (hs.M.ptr != hs.L.ptr || hs.M.col != hs.L.col) {   // the preconditioner fuses M and L SpMVs
        set_error("internal: trace M and L sparsity patterns differ");
        return DE_EINVAL;
    }
    {   // K_c = L_c, or L_c + M_c for singular components
        std::vector<Trip> tK;
        for (int32_t r = 0; r < nflat; ++r) {
            int c = 0;
            while (r >= hs.comp_off[c + 1]) ++c;
            for (int32_t k = hs.L.ptr[r]; k < hs.L.ptr[r + 1]; ++k) tK.push_back({r, hs.L.col[k], hs.L.val[k]});
            if (hs.singular_mask & (1 << c))
                for (int32_t k = hs.M.ptr[r]; k < hs.M.ptr[r + 1]; ++k) tK.push_back({r, hs.M.col[k], hs.M.val[k]});
        }
        hs.K = csr_from_trips(nflat, tK);
    }
    de_status_t st = build_elim(hs, hs.K, hs.elimK);
    if (st != DE_OK) return st;
    return build_elim(hs, hs.M, hs.elimM);
}

// Ring structures of the owned subdomains: A_IG (rows: interior, cols: local Gamma) and
// [A_GG | A_GI] (rows: local Gamma, cols: local Gamma or interior), from the elements of s.
void build_ring(const HostSetup& hs, const std::vector<int32_t>& owned, HRing& R) {
    const int dim = hs.dim;
    R.igp.clear();
    R.gxp.clear();
    R.ig_col.clear();
    R.ig_da.clear();
    R.ig_db.clear();
    R.gx_col.clear();
    R.gx_da.clear();
    R.gx_db.clear();
    R.igp_off.clear();
    R.gxp_off.clear();
    for (int32_t s : owned) {
        const int sx = s % hs.ps[0], sy = (s / hs.ps[0]) % hs.ps[1], sz = s / (hs.ps[0] * hs.ps[1]);
        const int32_t* gd = &hs.gdofs[hs.goff[s]];
        const int nG = hs.nGs[s], nI = hs.nI[s];
        auto gl = [&](int32_t dof) {
            return int32_t(std::lower_bound(gd, gd + nG, dof) - gd);
        };
        std::vector<std::pair<int32_t, int32_t>> ig, gx;   // (row, col-key) pairs
        std::vector<std::pair<int32_t, int32_t>> igd, gxd;
        std::map<std::pair<int32_t, int32_t>, std::pair<int32_t, int32_t>> igm, gxm;
        for (int ez = sz * hs.sub[2]; ez < (sz + 1) * hs.sub[2]; ++ez)
            for (int ey = sy * hs.sub[1]; ey < (sy + 1) * hs.sub[1]; ++ey)
                for (int ex = sx * hs.sub[0]; ex < (sx + 1) * hs.sub[0]; ++ex) {
                    int32_t dofs[24];
                    int nd = 0;
                    bool touches_gamma = false;
                    for (int o = 0; o < (1 << dim); ++o) {
                        const int64_t node = (ex + (o & 1)) +
                                             int64_t(hs.nn[0]) * ((ey + ((o >> 1) & 1)) + int64_t(hs.nn[1]) * (ez + ((o >> 2) & 1)));
                        for (int c = 0; c < dim; ++c) {
                            dofs[nd] = int32_t(dim * node + c);
                            if (hs.cls[dofs[nd]] == 1) touches_gamma = true;
                            ++nd;
                        }
                    }
                    if (!touches_gamma) continue;
                    for (int i = 0; i < nd; ++i) {
                        const int32_t da = dofs[i];
                        if (hs.cls[da] == 2) continue;
                        for (int j = 0; j < nd; ++j) {
                            const int32_t db = dofs[j];
                            if (hs.cls[db] == 2) continue;
                            if (hs.cls[da] == 0 && hs.cls[db] == 1)
                                igm[{hs.lidx[da], gl(db)}] = {da, db};
                            else if (hs.cls[da] == 1 && hs.cls[db] == 1)
                                gxm[{gl(da), gl(db)}] = {da, db};
                            else if (hs.cls[da] == 1 && hs.cls[db] == 0)
                                gxm[{gl(da), -hs.lidx[db] - 1}] = {da, db};
                        }
                    }
                }
        R.igp_off.push_back(int64_t(R.igp.size()));
        {
            std::vector<int32_t> cnt(nI + 1, 0);
            for (auto& kv : igm) cnt[kv.first.first + 1]++;
            const int32_t base = int32_t(R.ig_col.size());
            R.igp.push_back(base);
            int32_t acc = base;
            for (int i = 0; i < nI; ++i) {
                acc += cnt[i + 1];
                R.igp.push_back(acc);
            }
            for (auto& kv : igm) {   // map order = (row, col) ascending
                R.ig_col.push_back(kv.first.second);
                R.ig_da.push_back(kv.second.first);
                R.ig_db.push_back(kv.second.second);
            }
        }
        R.gxp_off.push_back(int64_t(R.gxp.size()));
        {
            std::vector<int32_t> cnt(nG + 1, 0);
            for (auto& kv : gxm) cnt[kv.first.first + 1]++;
            const int32_t base = int32_t(R.gx_col.size());
            R.gxp.push_back(base);
            int32_t acc = base;
            for (int i = 0; i < nG; ++i) {
                acc += cnt[i + 1];
                R.gxp.push_back(acc);
            }
            for (auto& kv : gxm) {
                R.gx_col.push_back(kv.first.second);
                R.gx_da.push_back(kv.second.first);
                R.gx_db.push_back(kv.second.second);
            }
        }
    }
}

}  // namespace de
