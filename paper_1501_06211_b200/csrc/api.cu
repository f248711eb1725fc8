// api.cu — the C ABI of include/de.h: context lifetime, device upload, de_factor, and the
// de_solve orchestration: condense -> interface PCG (CUDA-graph captured
// iterations with device-side scalars and early exit) -> back-substitution -> true residual.
// Multi-GPU: owned subdomain slabs, replicated interface vectors, one ncclAllReduce of the
// partial interface sums per iteration (NCCL resolved with dlopen; torch has it loaded).
#include "de_internal.h"

#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <map>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstring>

namespace de {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclId {
    char internal[128];
};
typedef int (*nccl_get_id_t)(NcclId*);
typedef int (*nccl_init_rank_t)(void**, int, NcclId, int);
typedef int (*nccl_allreduce_t)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_destroy_t)(void*);
typedef const char* (*nccl_errstr_t)(int);
struct NcclApi {
    bool ok = false;
    nccl_get_id_t get_id = nullptr;
    nccl_init_rank_t init_rank = nullptr;
    nccl_allreduce_t allreduce = nullptr;
    nccl_destroy_t destroy = nullptr;
    nccl_errstr_t errstr = nullptr;
};
static NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* p = getenv("DE_NCCL_LIB");
            if (p) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
        }
        if (h) {
            api.get_id = (nccl_get_id_t)dlsym(h, "ncclGetUniqueId");
            api.init_rank = (nccl_init_rank_t)dlsym(h, "ncclCommInitRank");
            api.allreduce = (nccl_allreduce_t)dlsym(h, "ncclAllReduce");
            api.destroy = (nccl_destroy_t)dlsym(h, "ncclCommDestroy");
            api.errstr = (nccl_errstr_t)dlsym(h, "ncclGetErrorString");
            api.ok = api.get_id && api.init_rank && api.allreduce && api.destroy;
        }
    }
    return api;
}

}  // namespace de

using namespace de;

// Loopback group (include/de.h de_loopback_create): host barrier + device slots [n][cap]
struct de_loopback {
    int n = 1;
    std::mutex coop_mu;   // one cooperative kernel of the group on the device at a time (see precond())
    std::mutex m;
    std::condition_variable cv;
    int count = 0;
    long gen = 0;
    double* slots = nullptr;
    size_t cap = 0;
    int device = 0;
    // false: the other ranks did not arrive within 60 s (one of them left the collective with an error): the caller
    // fails instead of blocking forever
    bool barrier() {
        std::unique_lock<std::mutex> lk(m);
        const long g = gen;
        if (++count == n) {
            count = 0;
            ++gen;
            cv.notify_all();
            return true;
        }
        if (cv.wait_for(lk, std::chrono::seconds(60), [&] { return gen != g; })) return true;
        --count;
        return false;
    }
};

struct de_ctx {
    HostSetup hs;
    de_options_t opt;
    double E0 = 1, Emin = 0, p = 3, nu = 0.3;
    cudaStream_t st = nullptr;
    bool own_stream = false;
    int rank = 0, nranks = 1;
    std::vector<int32_t> owned;
    std::vector<SubDesc> hsd;
    int nsl = 0, max_nI = 0, max_nG = 0;
    MeshDev md{};
    int64_t n_local_I = 0, n_local_G = 0;
    // device memory
    std::vector<void*> allocs;
    std::vector<void*> prec_allocs;   // preconditioner buffers (freed and rebuilt for the weighted norm)
    bool in_prec = false;             // dalloc records into prec_allocs
    bool dens_dirty = false;          // densities changed since the preconditioner was built
    SubDesc* d_sd = nullptr;
    double *d_rho = nullptr, *d_Ee = nullptr;
    int8_t* d_cls = nullptr;
    int32_t *d_idofs = nullptr, *d_Rg = nullptr, *d_igp = nullptr, *d_ig_col = nullptr, *d_ig_da = nullptr,
            *d_ig_db = nullptr, *d_ig_sub = nullptr, *d_gxp = nullptr, *d_gx_col = nullptr, *d_gx_da = nullptr,
            *d_gx_db = nullptr, *d_gx_sub = nullptr;
    double* d_dinv = nullptr;   // inverse diagonal blocks of the factors (wide bands, k_schur_blk)
    int dinv_np = 0, dinv_bs = 16;
    double *d_ig_val = nullptr, *d_gx_val = nullptr, *d_band = nullptr, *d_scratch = nullptr, *d_qloc = nullptr;
    int64_t n_ig = 0, n_gx = 0;
    int32_t *d_gptr = nullptr, *d_gsrc = nullptr, *d_gamma_dofs = nullptr;
    double *d_fG = nullptr, *d_res = nullptr, *d_ubuf = nullptr, *d_fbuf = nullptr;
    double *d_x = nullptr, *d_r = nullptr, *d_z = nullptr, *d_p = nullptr, *d_q = nullptr, *d_g = nullptr,
           *d_rold = nullptr, *d_xprev = nullptr;
    PcgState* d_state = nullptr;
    RedBuf rb{};
    double* d_scal = nullptr;
    int* d_fail = nullptr;
    PrecDev P{};
    bool have_prec = false;
    CoopBuffers coop{};
    bool use_coop = false;
    bool factored = false, have_prev = false;
    // graph
    cudaGraphExec_t gexec = nullptr;
    int graph_iters = 0;
    bool graph_prof = false;
    int launches_per_iter = 0;
    // profiling
    bool profiling = false;
    std::vector<cudaEvent_t> ev;
    double prof_ms = 0.0, prof_ms_prec = 0.0;
    int64_t prof_n = 0, prof_n_prec = 0;
    int64_t launches = 0;
    double* d_ubuf2 = nullptr;
    double* d_ulo = nullptr;          // low part of the double-double refinement iterate (R17)
    bool explicit_schur = false;
    double* d_sexp = nullptr;
    double* d_colscratch = nullptr;
    int col_batch = 0;
    int max_ig = 0;
    int64_t n_sexp = 0;
    // full-system FGMRES (outer = 1) work space, allocated on first use
    double *fg_V = nullptr, *fg_Z = nullptr, *fg_w = nullptr, *fg_r = nullptr, *fg_zero = nullptr, *fg_vG = nullptr,
           *fg_zG = nullptr, *fg_h = nullptr;
    RedBuf fg_rb{};
    // topology-optimisation design update (allocated on first use)
    double *oc_dc = nullptr, *oc_part = nullptr, *oc_rho = nullptr;
    OcState* oc_st = nullptr;
    bool oc_have_dc = false;
    int fg_m = 0;
    // nccl
    void* comm = nullptr;
    de_loopback* lb = nullptr;        // loopback group instead of NCCL (tests of the multi-rank path)
    de_stats_t stats{};
};

namespace {

template <class T>
de_status_t dalloc(de_ctx* c, T** p, size_t n) {
    *p = nullptr;
    if (n == 0) n = 1;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T));
    if (e != cudaSuccess) {
        set_error("cudaMalloc(%zu bytes) failed: %s", n * sizeof(T), cudaGetErrorString(e));
        return e == cudaErrorMemoryAllocation ? DE_ENOMEM : DE_ECUDA;
    }
    (c->in_prec ? c->prec_allocs : c->allocs).push_back(*p);
    return DE_OK;
}

template <class T>
de_status_t dupload(de_ctx* c, T** p, const std::vector<T>& h) {
    de_status_t s = dalloc(c, p, h.size());
    if (s != DE_OK) return s;
    if (!h.empty()) DE_CUDA(cudaMemcpyAsync(*p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, c->st));
    return DE_OK;
}

#define TRY(x)                          \
    do {                                \
        de_status_t s_ = (x);           \
        if (s_ != DE_OK) return s_;     \
    } while (0)

de_status_t check_launch() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("kernel launch failed: %s", cudaGetErrorString(e));
        return DE_ECUDA;
    }
    return DE_OK;
}

de_status_t allreduce(de_ctx* c, double* buf, size_t n) {
    if (c->nranks <= 1) return DE_OK;
    if (c->lb) {   // loopback: host-synchronised, fixed-order sum of the ranks' slots (bitwise equal on every rank)
        de_loopback* g = c->lb;
        if (n > g->cap) {
            set_error("loopback all-reduce of %zu doubles exceeds the group's capacity %zu", n, g->cap);
            return DE_EINVAL;
        }
        DE_CUDA(cudaMemcpyAsync(g->slots + size_t(c->rank) * g->cap, buf, n * sizeof(double),
                                cudaMemcpyDeviceToDevice, c->st));
        DE_CUDA(cudaStreamSynchronize(c->st));
        if (!g->barrier()) {
            set_error("loopback exchange timed out: another rank left the collective");
            return DE_ENCCL;
        }
        launch_sum_slots(buf, g->slots, g->n, g->cap, int64_t(n), c->st);
        DE_CUDA(cudaStreamSynchronize(c->st));
        if (!g->barrier()) {
            set_error("loopback exchange timed out: another rank left the collective");
            return DE_ENCCL;
        }
        return check_launch();
    }
    int r = nccl().allreduce(buf, buf, n, 8 /*ncclFloat64*/, 0 /*ncclSum*/, c->comm, c->st);
    if (r != 0) {
        set_error("ncclAllReduce failed: %s", nccl().errstr ? nccl().errstr(r) : "?");
        return DE_ENCCL;
    }
    return DE_OK;
}

SchurArgs schur_args(de_ctx* c, int mode, const double* xin, const double* f, double* u, const PcgState* s) {
    SchurArgs a{};
    a.sd = c->d_sd;
    a.nsl = c->nsl;
    a.band = c->d_band;
    a.dinv = c->d_dinv;
    a.dinv_np = c->dinv_np;
    a.dinv_bs = c->dinv_bs;
    a.ld = c->hs.ld;
    a.band_w = c->hs.band;
    a.idofs = c->d_idofs;
    a.Rg = c->d_Rg;
    a.igp = c->d_igp;
    a.ig_col = c->d_ig_col;
    a.ig_val = c->d_ig_val;
    a.gxp = c->d_gxp;
    a.gx_col = c->d_gx_col;
    a.gx_val = c->d_gx_val;
    a.scratch = c->d_scratch;
    a.xin = xin;
    a.f = f;
    a.qloc = c->d_qloc;
    a.u = u;
    a.state = s;
    a.mode = mode;
    a.maxG = c->max_nG;
    a.max_nI = c->max_nI;
    return a;
}

// q = S x (assembled over ranks). Used outside the captured loop.
void launch_apply(de_ctx* c, const double* x, const PcgState* s) {
    if (c->explicit_schur)
        launch_schur_explicit(c->d_sd, c->nsl, c->d_sexp, c->d_Rg, x, c->d_qloc, c->max_nG, s, c->st);
    else
        launch_schur_local(schur_args(c, SCHUR_APPLY, x, nullptr, nullptr, s), c->st);
}

de_status_t schur_apply(de_ctx* c, const double* x, double* q) {
    launch_apply(c, x, nullptr);
    launch_gather(c->d_gptr, c->d_gsrc, c->d_qloc, nullptr, q, c->hs.n_G, nullptr, c->st);
    TRY(check_launch());
    return allreduce(c, q, size_t(c->hs.n_G));
}

de_status_t precond(de_ctx* c, const double* r, double* z, const PcgState* s, int* nl, bool literal = false) {
    if (c->have_prec && c->use_coop) {
        // Loopback group: the ranks' host threads would launch whole-device cooperative kernels concurrently on their
        // own streams; two such grids can each become partially resident and wait in their grid barriers for blocks
        // the other one keeps off the SMs (observed: an intermittent hang of the 8-rank loopback test). One rank's
        // application at a time, held until it has finished (test path only; real ranks own their device).
        std::unique_lock<std::mutex> lk;
        if (c->lb) lk = std::unique_lock<std::mutex>(c->lb->coop_mu);
        if (prec_apply_coop(c->P, c->coop, r, z, s, c->st, literal) < 0) {
            set_error("cooperative preconditioner launch failed: %s", cudaGetErrorString(cudaGetLastError()));
            return DE_ECUDA;
        }
        if (c->lb) DE_CUDA(cudaStreamSynchronize(c->st));
        if (nl) *nl = 3;   // k_prec_coop, k_prec_ritz, k_prec_combine
    } else if (c->have_prec) {
        prec_apply(c->P, r, z, s, c->st, nl);
    } else {
        launch_copy(z, r, c->hs.n_G, s, c->st);
        if (nl) *nl = 1;
    }
    return check_launch();
}

// one PCG iteration (all on c->st; capturable)
de_status_t pcg_iteration(de_ctx* c, int* nl, cudaEvent_t e0, cudaEvent_t e1, cudaEvent_t e2 = nullptr,
                          cudaEvent_t e3 = nullptr) {
    const int64_t nG = c->hs.n_G;
    int n = 0;
    if (e0) cudaEventRecordWithFlags(e0, c->st, cudaEventRecordExternal);   // a real node when captured
    launch_apply(c, c->d_p, c->d_state);
    if (e1) cudaEventRecordWithFlags(e1, c->st, cudaEventRecordExternal);
    const bool pr = c->opt.beta_variant == 1;
    if (c->nranks == 1) {   // assembly and p.q in one pass
        launch_gather_pq(c->d_gptr, c->d_gsrc, c->d_qloc, c->d_p, c->d_q, nG, c->rb, c->d_state, c->st);
        n += 2;
    } else {
        launch_gather(c->d_gptr, c->d_gsrc, c->d_qloc, nullptr, c->d_q, nG, c->d_state, c->st);
        TRY(allreduce(c, c->d_q, size_t(nG)));
        launch_pcg_pq(c->d_p, c->d_q, nG, c->rb, c->d_state, c->st);
        n += 3;
    }
    launch_pcg_update_xr(c->d_x, c->d_r, pr ? c->d_rold : nullptr, c->d_p, c->d_q, nG, c->rb, c->d_state, c->st);
    n += 1;
    int np = 0;
    if (e2) cudaEventRecordWithFlags(e2, c->st, cudaEventRecordExternal);
    TRY(precond(c, c->d_r, c->d_z, c->d_state, &np));
    if (e3) cudaEventRecordWithFlags(e3, c->st, cudaEventRecordExternal);
    n += np;
    launch_pcg_rz(c->d_r, c->d_z, c->d_rold, nG, pr ? 1 : 0, c->rb, c->d_state, c->st);
    launch_pcg_update_p(c->d_p, c->d_z, nG, c->d_state, c->st);
    n += 2;
    if (nl) *nl = n;
    return check_launch();
}

de_status_t build_graph(de_ctx* c) {
    if (c->gexec) {
        cudaGraphExecDestroy(c->gexec);
        c->gexec = nullptr;
    }
    const int ni = std::max(1, c->opt.check_every);
    const bool prof = c->profiling;
    if (prof && int(c->ev.size()) < 4 * ni) {
        for (auto e : c->ev) cudaEventDestroy(e);
        c->ev.assign(4 * ni, nullptr);
        for (auto& e : c->ev) DE_CUDA(cudaEventCreate(&e));
    }
    cudaGraph_t g;
    DE_CUDA(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
    de_status_t s = DE_OK;
    for (int i = 0; i < ni && s == DE_OK; ++i)
        s = pcg_iteration(c, &c->launches_per_iter, prof ? c->ev[4 * i] : nullptr, prof ? c->ev[4 * i + 1] : nullptr,
                          prof ? c->ev[4 * i + 2] : nullptr, prof ? c->ev[4 * i + 3] : nullptr);
    cudaError_t e = cudaStreamEndCapture(c->st, &g);
    if (s != DE_OK) return s;
    DE_CUDA(e);
    e = cudaGraphInstantiate(&c->gexec, g, 0);
    cudaGraphDestroy(g);
    DE_CUDA(e);
    c->graph_iters = ni;
    c->graph_prof = prof;
    return DE_OK;
}

de_status_t read_state(de_ctx* c, PcgState* h) {
    DE_CUDA(cudaMemcpyAsync(h, c->d_state, sizeof(PcgState), cudaMemcpyDeviceToHost, c->st));
    DE_CUDA(cudaStreamSynchronize(c->st));
    return DE_OK;
}

de_status_t run_loop(de_ctx* c, PcgState& hsv) {
    const bool use_graph = c->opt.use_graph != 0 && !c->lb;   // loopback exchanges are host-synchronised
    if (use_graph && (!c->gexec || c->graph_prof != c->profiling)) TRY(build_graph(c));
    while (true) {
        const int it_before = hsv.it;
        if (use_graph) {
            DE_CUDA(cudaGraphLaunch(c->gexec, c->st));
            c->launches += int64_t(c->launches_per_iter) * c->graph_iters;
        } else {
            const int ni = std::max(1, c->opt.check_every);
            for (int i = 0; i < ni; ++i) TRY(pcg_iteration(c, &c->launches_per_iter, nullptr, nullptr));
            c->launches += int64_t(c->launches_per_iter) * ni;
        }
        TRY(read_state(c, &hsv));
        if (use_graph && c->graph_prof) {
            const int ran = std::min(hsv.it - it_before, c->graph_iters);
            for (int i = 0; i < ran; ++i) {
                float ms = 0.f;
                if (cudaEventElapsedTime(&ms, c->ev[4 * i], c->ev[4 * i + 1]) == cudaSuccess) {
                    c->prof_ms += ms;
                    c->prof_n += 1;
                }
                if (cudaEventElapsedTime(&ms, c->ev[4 * i + 2], c->ev[4 * i + 3]) == cudaSuccess) {
                    c->prof_ms_prec += ms;
                    c->prof_n_prec += 1;
                }
            }
        }
        if (hsv.done) break;
    }
    return DE_OK;
}

de_status_t masked_norm2(de_ctx* c, const double* f, double* out_host) {
    launch_copy(c->d_res, f, c->hs.ndof, nullptr, c->st);
    launch_zero_dirichlet(c->d_cls, c->d_res, c->hs.ndof, c->st);
    launch_norm2(c->d_res, c->hs.ndof, c->rb, c->d_scal, c->st);
    TRY(check_launch());
    DE_CUDA(cudaMemcpyAsync(out_host, c->d_scal, sizeof(double), cudaMemcpyDeviceToHost, c->st));
    DE_CUDA(cudaStreamSynchronize(c->st));
    return DE_OK;
}

de_status_t upload_prec_impl(de_ctx* c);

// Every preconditioner buffer is recorded in c->prec_allocs, so the weighted norm (R19) can rebuild it.
de_status_t upload_prec(de_ctx* c) {
    c->in_prec = true;
    const de_status_t s = upload_prec_impl(c);
    c->in_prec = false;
    return s;
}

// Weighted trace norm after a density update (R19): host rebuild of M, L, K and the eliminations from the new
// element moduli, then a fresh device upload (the PCG graph holds the old pointers: rebuilt on next use).
de_status_t rebuild_weighted_prec(de_ctx* c) {
    HostSetup& hs = c->hs;
    std::vector<double> rho(hs.nelem);
    DE_CUDA(cudaMemcpyAsync(rho.data(), c->d_rho, sizeof(double) * hs.nelem, cudaMemcpyDeviceToHost, c->st));
    DE_CUDA(cudaStreamSynchronize(c->st));
    hs.trace_E.resize(hs.nelem);
    for (int64_t e = 0; e < hs.nelem; ++e) hs.trace_E[e] = c->Emin + std::pow(rho[e], c->p) * (c->E0 - c->Emin);
    TRY(build_trace(hs, hs.trace_E.data()));
    c->stats.cross_fd = (hs.elimK.fd ? 1 : 0) | (hs.elimM.fd ? 2 : 0);
    if (c->gexec) {
        cudaGraphExecDestroy(c->gexec);
        c->gexec = nullptr;
    }
    for (void* p : c->prec_allocs) cudaFree(p);
    c->prec_allocs.clear();
    c->P = PrecDev{};
    c->coop = CoopBuffers{};
    c->have_prec = c->use_coop = false;
    TRY(upload_prec(c));
    c->dens_dirty = false;
    return DE_OK;
}

de_status_t upload_prec_impl(de_ctx* c) {
    HostSetup& hs = c->hs;
    PrecDev& P = c->P;
    P.ncomp = hs.ncomp;
    P.nflat = int32_t(hs.comp_off[hs.ncomp]);
    P.kmax = std::min(std::max(1, c->opt.lanczos_k), KMAX);
    P.jacobi_reg = getenv("DE_JACOBI_REG") ? 1 : (getenv("DE_JACOBI_WARP") ? 2 : 0);   // A/B: one-warp Jacobi variants
    for (int i = 0; i <= MAXC; ++i) P.comp_off[i] = hs.comp_off[std::min(i, hs.ncomp)];
    for (int i = 0; i < MAXC; ++i) P.singular[i] = (hs.singular_mask >> i) & 1;
    P.theta = c->opt.theta;
    P.max_face_band = 0;
    for (const HElim* E : {&hs.elimK, &hs.elimM})
        for (int F = 0; F < E->nfaces; ++F) P.max_face_band = std::max(P.max_face_band, E->face_band[F]);
    TRY(dupload(c, &P.cmap, hs.cmap));
    auto up_csr = [&](const HCsr& A, CsrDev& D) -> de_status_t {
        D.n = A.n;
        TRY(dupload(c, &D.ptr, A.ptr));
        TRY(dupload(c, &D.col, A.col));
        TRY(dupload(c, &D.val, A.val));
        return DE_OK;
    };
    TRY(up_csr(hs.M, P.M));
    TRY(up_csr(hs.L, P.L));
    TRY(up_csr(hs.K, P.K));
    double* gjbuf = nullptr;
    int64_t maxsc = 0;
    for (const HElim* E : {&hs.elimK, &hs.elimM})
        for (int cc = 0; cc < hs.ncomp; ++cc) maxsc = std::max(maxsc, E->sc_off[cc + 1] - E->sc_off[cc]);
    TRY(dalloc(c, &gjbuf, size_t(std::max<int64_t>(maxsc, 1))));
    auto up_elim = [&](const HElim& E, const HCsr& X, ElimDev& D) -> de_status_t {
        D.nfaces = E.nfaces;
        D.ncross = E.ncross;
        D.ncomp = hs.ncomp;
        int mf = 1, mfac = 1;
        for (int F = 0; F < E.nfaces; ++F) {
            const int n = E.face_off[F + 1] - E.face_off[F];
            mf = std::max(mf, n);
            mfac = std::max(mfac, int(E.face_fac_off[F + 1] - E.face_fac_off[F]));
        }
        int maxb = 0;
        for (int F = 0; F < E.nfaces; ++F) maxb = std::max(maxb, E.face_band[F]);
        if (mf > 256 || maxb > 31) {
            set_error("interface face too large for the face-solve kernel (nodes %d > 256 or band %d > 31)", mf, maxb);
            return DE_EINVAL;
        }
        mfac = std::min(mfac, 0x7fff);
        D.maxface = (mfac << 16) | mf;
        D.maxld = maxb + 1;
        D.face_comp_off[0] = 0;
        for (int cc = 0; cc < MAXC; ++cc)
            D.face_comp_off[cc + 1] = D.face_comp_off[cc] + (cc < hs.ncomp ? int32_t(hs.n_faces_c[cc]) : 0);
        if (D.face_comp_off[hs.ncomp] != E.nfaces) {
            set_error("internal: faces are not grouped by component");
            return DE_EINVAL;
        }
        TRY(dupload(c, &D.face_off, E.face_off));
        TRY(dupload(c, &D.face_nodes, E.face_nodes));
        TRY(dupload(c, &D.face_band, E.face_band));
        TRY(dupload(c, &D.face_fac_off, E.face_fac_off));
        TRY(dupload(c, &D.face_fac, E.face_fac));
        TRY(dupload(c, &D.cross_flat, E.cross_flat));
        for (int i = 0; i <= MAXC; ++i) D.cross_comp_off[i] = E.cross_comp_off[i];
        TRY(dupload(c, &D.xcf_ptr, E.XCF.ptr));
        TRY(dupload(c, &D.xcf_col, E.XCF.col));
        TRY(dupload(c, &D.xcf_val, E.XCF.val));
        TRY(dupload(c, &D.xfc_ptr, E.XFC.ptr));
        TRY(dupload(c, &D.xfc_col, E.XFC.col));
        TRY(dupload(c, &D.xfc_val, E.XFC.val));
        // one S_C^-1 for all components when they are identical (HElim::sc_shared): every component points at it
        D.sc_shared = E.sc_shared;
        for (int i = 0; i <= MAXC; ++i) D.sc_off[i] = E.sc_shared ? 0 : E.sc_off[std::min(i, hs.ncomp)];
        if (E.sc_shared) {
            TRY(dupload(c, &D.Sinv, std::vector<double>(E.SC.begin(), E.SC.begin() + E.sc_off[1])));
        } else {
            TRY(dupload(c, &D.Sinv, E.SC));
        }
        for (int cc = 0; cc < (E.sc_shared ? 1 : hs.ncomp); ++cc) {   // S_C^-1 by Gauss-Jordan (setup only)
            const int nc = E.cross_comp_off[cc + 1] - E.cross_comp_off[cc];
            if (nc > 0) launch_gauss_jordan(D.Sinv + E.sc_off[cc], gjbuf, nc, c->st);
        }
        D.fb_off = nullptr;   // 3D: block-bidiagonal face factors (HElim::fb)
        D.fb = nullptr;
        if (!E.fb.empty() && int(E.fb_off.size()) == E.nfaces + 1) {
            TRY(dupload(c, &D.fb_off, E.fb_off));
            TRY(dupload(c, &D.fb, E.fb));
        }
        D.g3_items = 0;   // 3D: dense G_F = X_FF^-1 X_F,adj per face for the second face phase (HElim::g3)
        D.g3_item_face = D.g3_item_i0 = D.g3_adj_ptr = D.g3_adj = nullptr;
        D.g3_off = nullptr;
        D.g3 = nullptr;
        if (!E.g3.empty() && int(E.g3_off.size()) == E.nfaces + 1) {
            std::vector<int32_t> itf, iti;
            for (int F = 0; F < E.nfaces; ++F)
                for (int i0 = 0; i0 < E.face_off[F + 1] - E.face_off[F]; i0 += 32) {
                    itf.push_back(F);
                    iti.push_back(i0);
                }
            TRY(dupload(c, &D.g3_item_face, itf));
            TRY(dupload(c, &D.g3_item_i0, iti));
            TRY(dupload(c, &D.g3_off, E.g3_off));
            TRY(dupload(c, &D.g3, E.g3));
            TRY(dupload(c, &D.g3_adj_ptr, E.g3_adj_ptr));
            TRY(dupload(c, &D.g3_adj, E.g3_adj));
            D.g3_items = int32_t(itf.size());
        }
        D.fd = E.fd;   // fast diagonalisation of a separable S_C (HElim::fd): the cooperative kernel's cross-point solve
        D.fd_nx = E.fd_nx;
        D.fd_ny = E.fd_ny;
        D.fd_qx = D.fd_qy = D.fd_il = nullptr;
        if (E.fd) {
            TRY(dupload(c, &D.fd_qx, E.fd_qx));
            TRY(dupload(c, &D.fd_qy, E.fd_qy));
            TRY(dupload(c, &D.fd_il, E.fd_il));
        }
        {   // padded X_CF for the general (non-tridiagonal) path
            int w = 0;
            for (int ci = 0; ci < E.ncross; ++ci) w = std::max(w, E.XCF.ptr[ci + 1] - E.XCF.ptr[ci]);
            w = (w + 7) / 8 * 8;
            D.xcf_w = 0;
            D.xcfw_col = nullptr;
            D.xcfw_val = nullptr;
            if (w > 0 && w <= 64 && E.ncross > 0) {
                std::vector<int32_t> wc(size_t(w) * E.ncross, 0);
                std::vector<double> wv(size_t(w) * E.ncross, 0.0);
                for (int ci = 0; ci < E.ncross; ++ci)
                    for (int e = E.XCF.ptr[ci], k = 0; e < E.XCF.ptr[ci + 1]; ++e, ++k) {
                        wc[size_t(k) * E.ncross + ci] = E.XCF.col[e];
                        wv[size_t(k) * E.ncross + ci] = E.XCF.val[e];
                    }
                TRY(dupload(c, &D.xcfw_col, wc));
                TRY(dupload(c, &D.xcfw_val, wv));
                D.xcf_w = w;
            }
        }
        // face-interleaved tridiagonal copy (2D faces are paths): coalesced thread-per-face solves
        D.pat_id = nullptr;
        D.td_start = D.td_len = nullptr;
        D.tri = 1;
        for (int F = 0; F < E.nfaces && D.tri; ++F) {
            const int o = E.face_off[F], n = E.face_off[F + 1] - o;
            int nx = 0;
            for (int i = 0; i < n; ++i) nx += E.XFC.ptr[o + i + 1] - E.XFC.ptr[o + i];
            if (E.face_band[F] > 1 || n > TRI_N || nx > 2) D.tri = 0;
        }
        for (int ci = 0; ci < E.ncross && D.tri; ++ci)
            if (E.XCF.ptr[ci + 1] - E.XCF.ptr[ci] > XCF_W) D.tri = 0;
        if (D.tri && E.nfaces > 0) {
            const int ng = (E.nfaces + 31) / 32;
            std::vector<int32_t> tn(E.nfaces), tnode(size_t(ng) * TRI_N * 32, 0), txj(2 * E.nfaces, -1),
                txc(2 * E.nfaces, 0);
            std::vector<double> tinv(size_t(ng) * TRI_N * 32, 0.0), tsub(size_t(ng) * TRI_N * 32, 0.0),
                txv(2 * E.nfaces, 0.0);
            for (int F = 0; F < E.nfaces; ++F) {
                const int o = E.face_off[F], n = E.face_off[F + 1] - o, ld = E.face_band[F] + 1;
                const double* fac = &E.face_fac[E.face_fac_off[F]];
                tn[F] = n;
                const size_t g = F / 32, lane = F % 32;
                for (int j = 0; j < n; ++j) {
                    const size_t at = (g * TRI_N + j) * 32 + lane;
                    tnode[at] = E.face_nodes[o + j];
                    tinv[at] = fac[size_t(j) * ld];
                    tsub[at] = ld > 1 ? fac[size_t(j) * ld + 1] : 0.0;
                }
                int k = 0;
                for (int j = 0; j < n; ++j)
                    for (int e = E.XFC.ptr[o + j]; e < E.XFC.ptr[o + j + 1]; ++e, ++k) {
                        txj[2 * F + k] = j;
                        txc[2 * F + k] = E.XFC.col[e];
                        txv[2 * F + k] = E.XFC.val[e];
                    }
            }
            TRY(dupload(c, &D.tri_n, tn));
            TRY(dupload(c, &D.tri_node, tnode));
            TRY(dupload(c, &D.tri_inv, tinv));
            TRY(dupload(c, &D.tri_sub, tsub));
            TRY(dupload(c, &D.tri_xj, txj));
            TRY(dupload(c, &D.tri_xc, txc));
            TRY(dupload(c, &D.tri_xv, txv));
            // G_F = X_FF^-1 X_FC column by column (the same tridiagonal factor), per flat skeleton index
            const size_t nfl = size_t(hs.comp_off[hs.ncomp]);
            std::vector<int32_t> gc0(nfl, 0), gc1(nfl, 0);
            std::vector<double> gv0(nfl, 0.0), gv1(nfl, 0.0);
            std::vector<double> g;
            for (int F = 0; F < E.nfaces; ++F) {
                const int o = E.face_off[F], n = E.face_off[F + 1] - o;
                const size_t grp = F / 32, lane = F % 32;
                for (int k = 0; k < 2; ++k) {
                    const int jx = txj[2 * F + k];
                    if (jx < 0) continue;
                    g.assign(n, 0.0);
                    double prev = 0.0, lprev = 0.0;
                    for (int j = 0; j < n; ++j) {
                        const size_t at = (grp * TRI_N + j) * 32 + lane;
                        prev = ((j == jx ? txv[2 * F + k] : 0.0) - lprev * prev) * tinv[at];
                        g[j] = prev;
                        lprev = tsub[at];
                    }
                    double nxt = 0.0;
                    for (int j = n - 1; j >= 0; --j) {
                        const size_t at = (grp * TRI_N + j) * 32 + lane;
                        nxt = (g[j] - tsub[at] * nxt) * tinv[at];
                        g[j] = nxt;
                    }
                    for (int j = 0; j < n; ++j) {
                        const int fl = E.face_nodes[o + j];
                        (k == 0 ? gc0 : gc1)[fl] = txc[2 * F + k];
                        (k == 0 ? gv0 : gv1)[fl] = g[j];
                    }
                }
            }
            for (int ci = 0; ci < E.ncross; ++ci) {
                gc0[E.cross_flat[ci]] = ci;
                gv0[E.cross_flat[ci]] = -1.0;
            }
            TRY(dupload(c, &D.g_c0, gc0));
            TRY(dupload(c, &D.g_c1, gc1));
            TRY(dupload(c, &D.g_v0, gv0));
            TRY(dupload(c, &D.g_v1, gv1));
            // Row patterns of the fused consumer (x = y - G x_C of a row's neighbours, then (M x)_i, (L x)_i): a face
            // node's neighbours are its flat neighbours i-1, i+1 in the same face and the face's own end cross points, so
            // its x values need only row i's couplings; the (source codes, M values, L values) triples of a uniform
            // skeleton take a handful of distinct values, kept in a small table that stays in L1. pat_id[i] = -1
            // (cross points, irregular rows) -> the general path. Source codes: 0 / 1 / 2 = flat i-1 / i / i+1,
            // 3 / 4 = x_C of the face's first / second coupling, 7 = unused entry; 3 bits per entry.
            D.pat_id = nullptr;
            D.pat_code = nullptr;
            D.pat_m = D.pat_l = nullptr;
            if (!getenv("DE_NO_PAT")) {
                const HCsr& Mh = hs.M;
                const HCsr& Lh = hs.L;
                std::vector<int32_t> faceid(nfl, -1), pid(nfl, -1), codes;
                std::vector<double> pm, pl;
                for (int F = 0; F < E.nfaces; ++F)
                    for (int sl = E.face_off[F]; sl < E.face_off[F + 1]; ++sl) faceid[E.face_nodes[sl]] = F;
                std::vector<int32_t> cross_of(nfl, -1);
                for (int ci = 0; ci < E.ncross; ++ci) cross_of[E.cross_flat[ci]] = ci;
                std::map<std::vector<double>, int32_t> pats;
                bool ok = true;
                for (size_t i = 0; i < nfl && ok; ++i) {
                    const int F = faceid[i];
                    if (F < 0) continue;
                    const int e0 = Mh.ptr[i], e1 = Mh.ptr[i + 1];
                    if (e1 - e0 > 3) continue;
                    int code = 0;
                    std::vector<double> key;
                    bool fast = true;
                    for (int k = 0; k < 3 && fast; ++k) {
                        const int e = e0 + k;
                        int src = 7;
                        double mv = 0.0, lv = 0.0;
                        if (e < e1) {
                            const int col = Mh.col[e];
                            if (Lh.col[e] != col) fast = false;
                            mv = Mh.val[e];
                            lv = Lh.val[e];
                            if (faceid[col] == F && std::abs(col - int(i)) <= 1) src = col - int(i) + 1;
                            else if (cross_of[col] >= 0 && txj[2 * F] >= 0 && txc[2 * F] == cross_of[col]) src = 3;
                            else if (cross_of[col] >= 0 && txj[2 * F + 1] >= 0 && txc[2 * F + 1] == cross_of[col]) src = 4;
                            else fast = false;
                        }
                        code |= src << (3 * k);
                        key.push_back(double(src));
                        key.push_back(mv);
                        key.push_back(lv);
                    }
                    if (!fast) continue;
                    auto it = pats.find(key);
                    if (it == pats.end()) {
                        if (pats.size() >= 4096) {   // no small table (e.g. the weighted trace norm): general path
                            ok = false;
                            break;
                        }
                        it = pats.emplace(key, int32_t(pats.size())).first;
                        codes.push_back(code);
                        for (int k = 0; k < 3; ++k) {
                            pm.push_back(key[3 * k + 1]);
                            pl.push_back(key[3 * k + 2]);
                        }
                    }
                    pid[i] = it->second;
                }
                // cross-point rows: own value x_C[k] plus up to XELL_W - 1 face-end neighbours, each with its own
                // couplings, in one ELL (two load levels instead of the CSR walk's four); pat_id = -2 - cross index
                D.xell_col = nullptr;
                if (ok && !pats.empty() && E.ncross > 0 && !getenv("DE_NO_XELL")) {
                    const size_t nx = size_t(E.ncross);
                    std::vector<int32_t> xc(XELL_W * nx, 0), x0(XELL_W * nx, 0), x1(XELL_W * nx, 0);
                    std::vector<double> xv0(XELL_W * nx, 0.0), xv1(XELL_W * nx, 0.0), xm(XELL_W * nx, 0.0), xl(XELL_W * nx, 0.0);
                    bool xok = true;
                    for (int ci = 0; ci < E.ncross && xok; ++ci) {
                        const int i = E.cross_flat[ci];
                        const int e0 = Mh.ptr[i], e1 = Mh.ptr[i + 1];
                        if (e1 - e0 > XELL_W) {
                            xok = false;
                            break;
                        }
                        for (int k = 0; k < XELL_W; ++k) {
                            const size_t at = size_t(k) * nx + ci;
                            const int e = e0 + k;
                            const int col = e < e1 ? Mh.col[e] : i;
                            if (e < e1 && Lh.col[e] != col) xok = false;
                            xc[at] = col;
                            x0[at] = gc0[col];
                            x1[at] = gc1[col];
                            xv0[at] = gv0[col];
                            xv1[at] = gv1[col];
                            xm[at] = e < e1 ? Mh.val[e] : 0.0;
                            xl[at] = e < e1 ? Lh.val[e] : 0.0;
                        }
                    }
                    if (xok) {
                        for (int ci = 0; ci < E.ncross; ++ci) pid[E.cross_flat[ci]] = -2 - ci;
                        TRY(dupload(c, &D.xell_col, xc));
                        TRY(dupload(c, &D.xell_c0, x0));
                        TRY(dupload(c, &D.xell_c1, x1));
                        TRY(dupload(c, &D.xell_v0, xv0));
                        TRY(dupload(c, &D.xell_v1, xv1));
                        TRY(dupload(c, &D.xell_m, xm));
                        TRY(dupload(c, &D.xell_l, xl));
                    }
                }
                if (ok && !pats.empty()) {
                    TRY(dupload(c, &D.pat_id, pid));
                    TRY(dupload(c, &D.pat_code, codes));
                    TRY(dupload(c, &D.pat_m, pm));
                    TRY(dupload(c, &D.pat_l, pl));
                    if (getenv("DE_VERBOSE")) fprintf(stderr, "[de] consumer row patterns: %zu\n", pats.size());
                }
            }
            D.fell_col = nullptr;
            if (&D == &P.eK && !getenv("DE_NO_FELL")) {   // fold ELL of the M/L rows with eK's couplings
                const HCsr& Mh = hs.M;
                const HCsr& Lh = hs.L;
                std::vector<int32_t> fc(FELL_W * nfl, 0), f0(FELL_W * nfl, 0), f1(FELL_W * nfl, 0);
                std::vector<double> v0(FELL_W * nfl, 0.0), v1(FELL_W * nfl, 0.0), fm(FELL_W * nfl, 0.0),
                    fl(FELL_W * nfl, 0.0);
                for (size_t i = 0; i < nfl; ++i) {
                    const int e0 = Mh.ptr[i], e1 = Mh.ptr[i + 1];
                    if (e1 - e0 > FELL_W) {
                        fc[i] = -1;   // CSR fallback (cross points with > FELL_W neighbours)
                        continue;
                    }
                    for (int k = 0; k < FELL_W; ++k) {
                        const size_t at = size_t(k) * nfl + i;
                        const int e = e0 + k;
                        const int col = e < e1 ? Mh.col[e] : int(i);
                        fc[at] = col;
                        f0[at] = gc0[col];
                        f1[at] = gc1[col];
                        v0[at] = gv0[col];
                        v1[at] = gv1[col];
                        fm[at] = e < e1 ? Mh.val[e] : 0.0;
                        fl[at] = e < e1 ? Lh.val[e] : 0.0;
                    }
                }
                TRY(dupload(c, &D.fell_col, fc));
                TRY(dupload(c, &D.fell_c0, f0));
                TRY(dupload(c, &D.fell_c1, f1));
                TRY(dupload(c, &D.fell_v0, v0));
                TRY(dupload(c, &D.fell_v1, v1));
                TRY(dupload(c, &D.fell_m, fm));
                TRY(dupload(c, &D.fell_l, fl));
            }
            D.fuse = getenv("DE_NO_E3_FUSE") ? 0 : 1;
            std::vector<int32_t> x4c(size_t(XCF_W) * E.ncross, 0);
            std::vector<double> x4v(size_t(XCF_W) * E.ncross, 0.0);
            for (int ci = 0; ci < E.ncross; ++ci)
                for (int e = E.XCF.ptr[ci], k = 0; e < E.XCF.ptr[ci + 1]; ++e, ++k) {
                    x4c[size_t(k) * E.ncross + ci] = E.XCF.col[e];
                    x4v[size_t(k) * E.ncross + ci] = E.XCF.val[e];
                }
            TRY(dupload(c, &D.xcf4_col, x4c));
            TRY(dupload(c, &D.xcf4_val, x4v));
            {   // PCR coefficients of every face block X_FF (tridiagonal along face_nodes)
                std::vector<double> pq(size_t(E.nfaces) * PCR_Q * 32, 0.0);
                std::vector<int32_t> pn(size_t(E.nfaces) * 32, 0);
                auto entry = [&](int r, int col) {
                    for (int e = X.ptr[r]; e < X.ptr[r + 1]; ++e)
                        if (X.col[e] == col) return X.val[e];
                    return 0.0;
                };
                for (int F = 0; F < E.nfaces; ++F) {
                    const int o = E.face_off[F], n = E.face_off[F + 1] - o;
                    double av[32], dv[32], cv[32];
                    for (int j = 0; j < 32; ++j) {
                        av[j] = cv[j] = 0.0;
                        dv[j] = 1.0;
                        if (j < n) {
                            const int fj = E.face_nodes[o + j];
                            pn[size_t(F) * 32 + j] = fj;
                            dv[j] = entry(fj, fj);
                            if (j > 0) av[j] = entry(fj, E.face_nodes[o + j - 1]);
                            if (j + 1 < n) cv[j] = entry(fj, E.face_nodes[o + j + 1]);
                        }
                    }
                    double* q = &pq[size_t(F) * PCR_Q * 32];
                    for (int l = 0; l < PCR_L; ++l) {
                        const int sg = 1 << l;
                        double na[32], nd[32], nc[32];
                        for (int j = 0; j < 32; ++j) {
                            const double al = j - sg >= 0 ? -av[j] / dv[j - sg] : 0.0;
                            const double ga = j + sg < 32 ? -cv[j] / dv[j + sg] : 0.0;
                            q[(2 * l) * 32 + j] = al;
                            q[(2 * l + 1) * 32 + j] = ga;
                            na[j] = j - sg >= 0 ? al * av[j - sg] : 0.0;
                            nc[j] = j + sg < 32 ? ga * cv[j + sg] : 0.0;
                            nd[j] = dv[j] + (j - sg >= 0 ? al * cv[j - sg] : 0.0) + (j + sg < 32 ? ga * av[j + sg] : 0.0);
                        }
                        for (int j = 0; j < 32; ++j) {
                            av[j] = na[j];
                            cv[j] = nc[j];
                            dv[j] = nd[j];
                        }
                    }
                    for (int j = 0; j < 32; ++j) q[(2 * PCR_L) * 32 + j] = 1.0 / dv[j];
                }
                // Faces with bitwise-identical coefficient blocks (uniform skeleton: a handful of face types) share one
                // block, so the per-face coefficient loads hit L1 instead of streaming 11 doubles per node from L2
                std::vector<double> uq;
                std::vector<int32_t> nt(E.nfaces, 0);
                {
                    std::map<std::vector<double>, int32_t> types;
                    for (int F = 0; F < E.nfaces; ++F) {
                        std::vector<double> blk(pq.begin() + size_t(F) * PCR_Q * 32, pq.begin() + size_t(F + 1) * PCR_Q * 32);
                        auto it = types.find(blk);
                        int32_t ty;
                        if (it == types.end()) {
                            ty = int32_t(types.size());
                            types.emplace(blk, ty);
                            uq.insert(uq.end(), blk.begin(), blk.end());
                        } else {
                            ty = it->second;
                        }
                        nt[F] = (E.face_off[F + 1] - E.face_off[F]) | (ty << 8);
                    }
                }
                TRY(dupload(c, &D.pcr, uq));
                TRY(dupload(c, &D.pcr_nt, nt));
                TRY(dupload(c, &D.pcr_node, pn));
            }
            {   // G^T rows per cross point from the per-node couplings (face nodes only; ascending column)
                std::vector<int32_t> gp(E.ncross + 1, 0), gcol;
                std::vector<double> gval;
                std::vector<std::vector<std::pair<int32_t, double>>> rows(E.ncross);
                std::vector<char> isc(nfl, 0);
                for (int ci = 0; ci < E.ncross; ++ci) isc[E.cross_flat[ci]] = 1;
                for (size_t fl = 0; fl < nfl; ++fl) {
                    if (isc[fl]) continue;   // cross points carry (-1, own index): not part of G^T
                    if (gv0[fl] != 0.0) rows[gc0[fl]].push_back({int32_t(fl), gv0[fl]});
                    if (gv1[fl] != 0.0) rows[gc1[fl]].push_back({int32_t(fl), gv1[fl]});
                }
                for (int ci = 0; ci < E.ncross; ++ci) {
                    gp[ci + 1] = gp[ci] + int32_t(rows[ci].size());
                    for (auto& q : rows[ci]) {
                        gcol.push_back(q.first);
                        gval.push_back(q.second);
                    }
                }
                D.td_start = D.td_len = nullptr;
                if (!getenv("DE_NO_TD")) {   // face descriptors of the same rows
                    std::vector<int32_t> ts(size_t(XCF_W) * E.ncross, 0), tl(size_t(XCF_W) * E.ncross, 0), cnt(E.ncross, 0);
                    bool ok = true;
                    for (int F = 0; F < E.nfaces && ok; ++F) {
                        const int o = E.face_off[F], n = E.face_off[F + 1] - o;
                        for (int j = 0; j < n; ++j)
                            if (E.face_nodes[o + j] != E.face_nodes[o] + j) ok = false;   // contiguous flat indices
                        for (int k = 0; k < 2 && ok; ++k) {
                            if (txj[2 * F + k] < 0) continue;
                            const int ci = txc[2 * F + k];
                            if (cnt[ci] >= XCF_W || n > 32) {
                                ok = false;
                                break;
                            }
                            ts[size_t(cnt[ci]) * E.ncross + ci] = E.face_nodes[o];
                            tl[size_t(cnt[ci]) * E.ncross + ci] = n | (k << 8);
                            ++cnt[ci];
                        }
                    }
                    if (ok) {
                        TRY(dupload(c, &D.td_start, ts));
                        TRY(dupload(c, &D.td_len, tl));
                    }
                }
                TRY(dupload(c, &D.gt_ptr, gp));
                TRY(dupload(c, &D.gt_col, gcol));
                TRY(dupload(c, &D.gt_val, gval));
            }
        }
        return check_launch();
    };
    TRY(up_elim(hs.elimK, hs.K, P.eK));
    TRY(up_elim(hs.elimM, hs.M, P.eM));
    const size_t nf = size_t(P.nflat);
    TRY(dalloc(c, &P.rf, nf));
    TRY(dalloc(c, &P.s, nf));
    TRY(dalloc(c, &P.v, nf));
    TRY(dalloc(c, &P.w, nf));
    TRY(dalloc(c, &P.Mw, nf));
    TRY(dalloc(c, &P.y, 2 * nf + 16));
    DE_CUDA(cudaMemsetAsync(P.y, 0, (2 * nf + 16) * sizeof(double), c->st));   // y stays 0 on cross points
    TRY(dalloc(c, &P.zf, nf));
    TRY(dalloc(c, &P.W, nf * KMAX));
    TRY(dalloc(c, &P.LW, nf * KMAX));
    TRY(dalloc(c, &P.MW, nf * KMAX));
    DE_CUDA(cudaMemsetAsync(P.W, 0, nf * KMAX * sizeof(double), c->st));
    TRY(dalloc(c, &P.lz, MAXC));
    DE_CUDA(cudaMemsetAsync(P.lz, 0, MAXC * sizeof(LzState), c->st));
    int64_t maxc = 1;
    for (int cc = 0; cc < hs.ncomp; ++cc) maxc = std::max(maxc, hs.comp_off[cc + 1] - hs.comp_off[cc]);
    P.nblk = int(std::max<int64_t>(1, std::min<int64_t>(256, (maxc + 1023) / 1024)));
    const int nslots = 8 + MAXC * KMAX + MAXC * KMAX * (2 * KMAX + 1);
    TRY(dalloc(c, &P.part, size_t(nslots) * P.nblk));
    TRY(dalloc(c, &P.counter, size_t(nslots)));
    DE_CUDA(cudaMemsetAsync(P.counter, 0, size_t(nslots) * sizeof(unsigned int), c->st));
    prec_prepare(P);
    c->have_prec = true;
    if (c->opt.inner_mode == 0) {   // SPEC face-PCG inner solves (multi-kernel path + k_face_pcg)
        if (fpcg_prepare(P, c->opt.device) <= 0) {
            set_error("inner_mode 0 needs a cooperative launch of k_face_pcg (device or shared memory limit)");
            return DE_ECUDA;
        }
        P.inner_f = 1;
        P.fp_tol = c->opt.inner_tol;
        P.fp_maxit = c->opt.inner_max_iter;
        TRY(dalloc(c, &P.fr, nf));
        TRY(dalloc(c, &P.fz, nf));
        TRY(dalloc(c, &P.fp, nf));
        TRY(dalloc(c, &P.fq, nf));
        TRY(dalloc(c, &P.fpart, size_t(2) * MAXC * P.fp_nb));
        TRY(dalloc(c, &P.fits, 1));
        DE_CUDA(cudaMemsetAsync(P.fits, 0, sizeof(unsigned long long), c->st));
        return DE_OK;
    }
    if (c->opt.prec_kernels == 0 && prec_coop_prepare(P, c->opt.device, c->coop)) {
        TRY(dalloc(c, &c->coop.red, prec_coop_red_doubles(c->coop)));
        TRY(dalloc(c, &c->coop.gram, prec_coop_gram_doubles(c->coop)));
        TRY(dalloc(c, &c->coop.gram_tot, size_t(MAXC) * KMAX * (2 * KMAX + 1)));
        TRY(dalloc(c, &c->coop.w1, nf));
        TRY(dalloc(c, &c->coop.mw1, nf));
        TRY(dalloc(c, &c->coop.lw1, nf));
        if (c->coop.fold) TRY(dalloc(c, &c->coop.ucross, size_t(KMAX) * std::max(1, P.eK.ncross)));
        TRY(dalloc(c, &c->coop.arrive, 4));
        TRY(dalloc(c, &c->coop.redf, size_t(2) * MAXC * (KMAX + 2) * c->coop.nb));
        DE_CUDA(cudaMemsetAsync(c->coop.arrive, 0, 4 * sizeof(unsigned int), c->st));
        if (getenv("DE_PREC_TIMERS")) {
            TRY(dalloc(c, &c->coop.timers, 200 + 8192));
            DE_CUDA(cudaMemsetAsync(c->coop.timers, 0, (200 + 8192) * sizeof(unsigned long long), c->st));
        }
        c->use_coop = true;
    }
    return DE_OK;
}

// Algorithmic bytes of one preconditioner application: every
// phase reads its operands and writes its results once, neighbour values of an SpMV come from cache
// (counted once as the vector), k = lanczos_k basis vectors, no breakdown.
double elim_bytes_model(const HElim& E, bool tri) {
    const double nfn = double(E.face_nodes.size());
    double b = 0.0;
    if (tri)   // per face solve: forward + backward read (node, 1/L_jj, L_j+1,j); rhs read; result write
        b += 2.0 * nfn * (2.0 * (4 + 8 + 8) + 8 + 8);
    else       // per face solve: the [L | M] band copies, node ids, rhs read, result write
        b += 2.0 * (double(E.face_fac.size()) * 8.0 + nfn * (4 + 8 + 8));
    b += double(E.XFC.val.size()) * 12.0;                                   // X_FC x_C in the second face solve
    b += double(E.XCF.val.size()) * (12.0 + 8.0) + double(E.ncross) * (4 + 4 + 8 + 8 + 8);   // t_C
    for (size_t cc = 0; cc + 1 < E.sc_off.size(); ++cc) {
        const double nc = double(E.cross_comp_off[cc + 1] - E.cross_comp_off[cc]);
        if (cc == 0 || !E.sc_shared) b += nc * nc * 8.0;                    // dense S_C^-1 rows (once if shared)
    }
    return b;
}

double prec_bytes_model(const HostSetup& hs, int k, bool gram_cgs2, bool fold) {
    const double n = double(hs.comp_off[hs.ncomp]), nnz = double(hs.M.val.size()), d = 8.0;
    bool tri = true;
    for (const HElim* E : {&hs.elimK, &hs.elimM})
        for (int F = 0; F < E->nfaces && tri; ++F) {
            const int o = E->face_off[F], nf = E->face_off[F + 1] - o;
            if (E->face_band[F] > 1 || nf > TRI_N) tri = false;
        }
    const double spmv = nnz * (4 + 8 + 8) + (n + 1) * 4 + n * d;            // M and L values, shared cols, x
    double b = n * (4 + d + d);                                             // gather r_c
    b += elim_bytes_model(hs.elimM, tri) + double(k - 1) * elim_bytes_model(hs.elimK, tri);
    b += spmv + n * d * 3;                                                  // seed: Ms, Ls, s.r
    for (int j = 1; j < k; ++j) {
        b += spmv + n * d * (fold ? j + 1 : j + 2);   // A: M w, L w, h (fold: (M W)^T y in the elimination, R22)
        if (!gram_cgs2) b += n * d * (3.0 * j + 3 + 3);                     // B: w1, M w1, L w1 (two-pass)
        b += n * d * (3.0 * j + 4 + 3);                                     // C: w2, M w2, L w2, Gram row j
    }
    b += n * d * k + n * (4 + d);                                           // z = W coef, scatter
    return b;
}

// Distinct bytes one preconditioner application touches, each counted once: a lower bound on its HBM traffic
// (perfect on-chip reuse inside the application; DESIGN.md §6 "minimum bytes"). r in, z out, the skeleton
// operators M and L (shared CSR pattern), per elimination operator (K and M) the face data, the face/cross
// couplings and S_C^-1 (once when the components share it), and the k basis vectors W, M W, L W written once.
double prec_min_bytes(const HostSetup& hs, int k) {
    const double n = double(hs.comp_off[hs.ncomp]), nnz = double(hs.M.val.size());
    bool tri = true;
    for (const HElim* E : {&hs.elimK, &hs.elimM})
        for (int F = 0; F < E->nfaces && tri; ++F)
            if (E->face_band[F] > 1 || E->face_off[F + 1] - E->face_off[F] > TRI_N) tri = false;
    double b = n * (4 + 8 + 8) + (n + 1) * 4 + nnz * (4 + 8 + 8);
    for (const HElim* E : {&hs.elimK, &hs.elimM}) {
        const double nfn = double(E->face_nodes.size()), ncr = double(E->ncross);
        if (tri)   // PCR coefficients + node ids per face, per-node couplings g (2 per node), G^T rows, cross ids
            b += double(E->nfaces) * (PCR_Q * 32 * 8 + 32 * 4) + n * 2 * (4 + 8) + 2 * nfn * 12 + ncr * 12;
        else       // band factors [L | M], node ids, X_FC and X_CF
            b += double(E->face_fac.size()) * 8 + nfn * 4 + double(E->XFC.val.size() + E->XCF.val.size()) * 12 + ncr * 4;
        for (int cc = 0; cc < hs.ncomp; ++cc)
            if (cc == 0 || !E->sc_shared) b += double(E->sc_off[cc + 1] - E->sc_off[cc]) * 8;
    }
    return b + 3.0 * k * n * 8;
}

de_status_t setup_impl(const de_mesh_t* mesh, const double* density, double E0, double Emin, double p,
                       double nu, const de_partition_t* part, const de_options_t* opt_in, de_ctx* c) {
    de_options_t opt;
    if (opt_in) opt = *opt_in;
    else de_default_options(&opt);
    if (!mesh || !part || !density || !mesh->fixed) {
        set_error("null argument");
        return DE_EINVAL;
    }
    if (!(E0 > 0) || !(Emin >= 0) || !(p > 0) || !(nu > -1.0 && nu < 0.5) || !(mesh->h > 0)) {
        set_error("invalid material parameters (E0 > 0, Emin >= 0, p > 0, -1 < nu < 1/2, h > 0)");
        return DE_EINVAL;
    }
    if (opt.inner_mode != 0 && opt.inner_mode != 1 && opt.inner_mode != 3) {
        set_error("inner_mode %d not supported on the GPU path (0 = face-PCG inner solves, 1 = exact-inner "
                  "inverse Lanczos, 3 = identity)", opt.inner_mode);
        return DE_EINVAL;
    }
    if (opt.inner_mode == 0 && (!(opt.inner_tol > 0.0) || opt.inner_max_iter < 1)) {
        set_error("inner_mode 0 needs inner_tol > 0 and inner_max_iter >= 1");
        return DE_EINVAL;
    }
    if ((opt.inner_mode == 0 || opt.inner_mode == 1) && (opt.lanczos_k < 1 || opt.lanczos_k > KMAX)) {
        set_error("lanczos_k must be in [1, %d]", KMAX);
        return DE_EINVAL;
    }
    if (opt.nranks < 1 || opt.rank < 0 || opt.rank >= opt.nranks) {
        set_error("bad rank/nranks");
        return DE_EINVAL;
    }
    c->opt = opt;
    c->E0 = E0;
    c->Emin = Emin;
    c->p = p;
    c->nu = nu;
    c->rank = opt.rank;
    c->nranks = opt.nranks;
    if (opt.weighted_trace) {   // R19: element moduli of the setup densities
        int64_t ne = 1;
        for (int a = 0; a < mesh->dim; ++a) ne *= mesh->nel[a];
        c->hs.trace_E.resize(ne);
        for (int64_t e = 0; e < ne; ++e) c->hs.trace_E[e] = Emin + std::pow(density[e], p) * (E0 - Emin);
    }
    TRY(host_setup(mesh, part, nu, c->hs));
    HostSetup& hs = c->hs;
    for (int64_t e = 0; e < hs.nelem; ++e)
        if (!(density[e] > 0.0) || !std::isfinite(density[e])) {
            set_error("density[%lld] = %g must be positive and finite", (long long)e, density[e]);
            return DE_EINVAL;
        }
    c->stats.ndof = hs.ndof;
    c->stats.n_free = hs.n_free;
    c->stats.n_I = hs.n_I;
    c->stats.n_Gamma = hs.n_G;
    c->stats.n_sub = hs.nsub;
    for (int cc = 0; cc < hs.ncomp; ++cc) c->stats.n_gamma_c[cc] = hs.comp_off[cc + 1] - hs.comp_off[cc];
    c->stats.cross_fd = (hs.elimK.fd ? 1 : 0) | (hs.elimM.fd ? 2 : 0);
    // ---- ownership: slabs of subdomain columns along x
    const int px = hs.ps[0];
    const int lo = int((int64_t(c->rank) * px) / c->nranks), hi = int((int64_t(c->rank + 1) * px) / c->nranks);
    for (int s = 0; s < hs.nsub; ++s) {
        const int sx = s % px;
        if (sx >= lo && sx < hi) c->owned.push_back(s);
    }
    c->nsl = int(c->owned.size());
    c->stats.n_sub_local = c->nsl;
    if (opt.host_only) return DE_OK;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        set_error("no CUDA device available (libde has no CPU path)");
        return DE_ECUDA;
    }
    DE_CUDA(cudaSetDevice(opt.device));
    if (opt.stream) {
        c->st = static_cast<cudaStream_t>(opt.stream);
    } else {
        DE_CUDA(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    HRing ring;
    build_ring(hs, c->owned, ring);
    std::vector<int32_t> idofs, Rg, ig_sub, gx_sub;
    int64_t ioff = 0, goff = 0;
    for (int k = 0; k < c->nsl; ++k) {
        const int s = c->owned[k];
        SubDesc d{};
        d.gid = s;
        d.nI = hs.nI[s];
        d.nG = hs.nGs[s];
        d.ioff = ioff;
        d.band_off = 2 * ioff * hs.ld;   // [L | M] per subdomain
        d.goff = goff;
        d.igp_off = ring.igp_off[k];
        d.gxp_off = ring.gxp_off[k];
        d.sexp_off = c->n_sexp;
        c->n_sexp += sexp_packed_doubles(hs.nGs[s]);
        c->hsd.push_back(d);
        idofs.insert(idofs.end(), hs.idofs.begin() + hs.ioff[s], hs.idofs.begin() + hs.ioff[s + 1]);
        for (int l = 0; l < d.nG; ++l) Rg.push_back(hs.gpos[hs.gdofs[hs.goff[s] + l]]);
        c->max_nI = std::max(c->max_nI, d.nI);
        c->max_nG = std::max(c->max_nG, d.nG);
        ioff += d.nI;
        goff += d.nG;
        const int32_t ig0 = ring.igp[ring.igp_off[k]], ig1 = ring.igp[ring.igp_off[k] + d.nI];
        ig_sub.insert(ig_sub.end(), size_t(ig1 - ig0), s);
        c->max_ig = std::max(c->max_ig, int(ig1 - ig0));
        const int32_t gx0 = ring.gxp[ring.gxp_off[k]], gx1 = ring.gxp[ring.gxp_off[k] + d.nG];
        gx_sub.insert(gx_sub.end(), size_t(gx1 - gx0), s);
    }
    c->n_local_I = ioff;
    c->n_local_G = goff;
    // ---- interface gather table (owned contributions, ascending subdomain)
    std::vector<int32_t> gcnt(hs.n_G + 1, 0);
    for (int32_t g : Rg) gcnt[g + 1]++;
    for (int64_t g = 0; g < hs.n_G; ++g) gcnt[g + 1] += gcnt[g];
    std::vector<int32_t> gsrc(Rg.size());
    {
        std::vector<int32_t> fill(gcnt.begin(), gcnt.end() - 1);
        for (size_t i = 0; i < Rg.size(); ++i) gsrc[fill[Rg[i]]++] = int32_t(i);
    }
    // ---- device upload
    c->md.dim = hs.dim;
    for (int a = 0; a < 3; ++a) {
        c->md.nel[a] = hs.nel[a];
        c->md.nn[a] = hs.nn[a];
        c->md.sub[a] = hs.sub[a];
        c->md.ps[a] = hs.ps[a];
    }
    c->md.nke = hs.nke;
    upload_KE0(hs.KE0, hs.nke, c->st);
    upload_KE0_oc(hs.KE0, hs.nke, c->st);
    TRY(dupload(c, &c->d_sd, c->hsd));
    TRY(dalloc(c, &c->d_rho, hs.nelem));
    DE_CUDA(cudaMemcpyAsync(c->d_rho, density, sizeof(double) * hs.nelem, cudaMemcpyHostToDevice, c->st));
    TRY(dalloc(c, &c->d_Ee, hs.nelem));
    TRY(dupload(c, &c->d_cls, hs.cls));
    TRY(dupload(c, &c->d_idofs, idofs));
    TRY(dupload(c, &c->d_Rg, Rg));
    TRY(dupload(c, &c->d_igp, ring.igp));
    TRY(dupload(c, &c->d_ig_col, ring.ig_col));
    TRY(dupload(c, &c->d_ig_da, ring.ig_da));
    TRY(dupload(c, &c->d_ig_db, ring.ig_db));
    TRY(dupload(c, &c->d_ig_sub, ig_sub));
    TRY(dupload(c, &c->d_gxp, ring.gxp));
    TRY(dupload(c, &c->d_gx_col, ring.gx_col));
    TRY(dupload(c, &c->d_gx_da, ring.gx_da));
    TRY(dupload(c, &c->d_gx_db, ring.gx_db));
    TRY(dupload(c, &c->d_gx_sub, gx_sub));
    c->n_ig = int64_t(ring.ig_col.size());
    c->n_gx = int64_t(ring.gx_col.size());
    TRY(dalloc(c, &c->d_ig_val, size_t(c->n_ig)));
    TRY(dalloc(c, &c->d_gx_val, size_t(c->n_gx)));
    TRY(dalloc(c, &c->d_band, 2 * size_t(c->n_local_I) * hs.ld));
    if ((hs.band + 1 + 31) / 32 > 4 && !getenv("DE_NO_DINV")) {   // wide bands (3D): k_schur_blk applies inverse diagonal blocks
        c->dinv_bs = schur_blk_panel_width(hs.ld, c->max_nI, c->max_nG);
        c->dinv_np = (c->max_nI + c->dinv_bs - 1) / c->dinv_bs;
        TRY(dalloc(c, &c->d_dinv, size_t(c->nsl) * c->dinv_np * c->dinv_bs * c->dinv_bs));
    }
    {   // explicit local Schur complements: decide, then allocate S_s and a column batch
        const double fac_one_pass = double(c->n_local_I) * (hs.band + 1);
        const bool fits = c->max_nG <= 1024;
        if (opt.schur_mode == 2 && !fits) {
            set_error("schur_mode = 2 needs n_Gamma,s <= 1024 per subdomain");
            return DE_EINVAL;
        }
        c->explicit_schur = fits && (opt.schur_mode == 2 || (opt.schur_mode == 0 && double(c->n_sexp) < fac_one_pass));
        if (c->explicit_schur) {
            TRY(dalloc(c, &c->d_sexp, size_t(c->n_sexp)));
            DE_CUDA(cudaMemsetAsync(c->d_sexp, 0, size_t(c->n_sexp) * sizeof(double), c->st));   // tile padding
            prepare_schur_explicit(c->max_nG);
            // scratch per subdomain: the thread-per-column formation keeps n_I x FORM_THREADS solutions, the
            // warp-per-8-columns one (n_Gamma,s + 8) x n_I; one launch per batch, a multiple of the SM count
            const size_t per = size_t(std::max(std::max(1, c->max_nG) + 8, FORM_THREADS)) * size_t(std::max(1, c->max_nI));
            int nsm = 148;
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->opt.device);
            size_t cap = (size_t(1) << 30) / (per * 8);
            if (cap >= size_t(nsm)) cap = cap / size_t(nsm) * size_t(nsm);
            c->col_batch = int(std::max<size_t>(1, std::min<size_t>(c->nsl, cap)));
            TRY(dalloc(c, &c->d_colscratch, size_t(c->col_batch) * per));
        }
    }
    TRY(dalloc(c, &c->d_scratch, size_t(c->n_local_I) + 32));
    prepare_schur_blk(hs.ld, hs.band, c->max_nI, c->max_nG);
    TRY(dalloc(c, &c->d_qloc, size_t(c->n_local_G) + 32));
    TRY(dupload(c, &c->d_gptr, gcnt));
    TRY(dupload(c, &c->d_gsrc, gsrc));
    TRY(dupload(c, &c->d_gamma_dofs, hs.gamma_dofs));
    const size_t nG = size_t(hs.n_G) + 32, nd = size_t(hs.ndof);
    for (double** v : {&c->d_x, &c->d_r, &c->d_z, &c->d_p, &c->d_q, &c->d_g, &c->d_rold, &c->d_xprev, &c->d_fG})
        TRY(dalloc(c, v, nG));
    DE_CUDA(cudaMemsetAsync(c->d_x, 0, nG * sizeof(double), c->st));
    DE_CUDA(cudaMemsetAsync(c->d_rold, 0, nG * sizeof(double), c->st));
    TRY(dalloc(c, &c->d_res, nd));
    TRY(dalloc(c, &c->d_ubuf, nd));
    TRY(dalloc(c, &c->d_fbuf, nd));
    TRY(dalloc(c, &c->d_ubuf2, nd));
    TRY(dalloc(c, &c->d_ulo, nd));
    TRY(dalloc(c, &c->d_state, 1));
    TRY(dalloc(c, &c->d_scal, 8));
    TRY(dalloc(c, &c->d_fail, 1));
    c->rb.nblk = 148 * 8;   // enough blocks for one interface dof per thread in k_gather_pq
    TRY(dalloc(c, &c->rb.part, size_t(c->rb.nblk) * 4));
    TRY(dalloc(c, &c->rb.counter, 1));
    DE_CUDA(cudaMemsetAsync(c->rb.counter, 0, sizeof(unsigned int), c->st));
    if (opt.inner_mode == 0 || opt.inner_mode == 1) TRY(upload_prec(c));
    DE_CUDA(cudaStreamSynchronize(c->st));
    TRY(check_launch());
    // ---- NCCL (or the loopback group)
    if (c->nranks > 1 && opt.loopback) {
        de_loopback* g = static_cast<de_loopback*>(opt.loopback);
        if (g->n != c->nranks) {
            set_error("loopback group has %d ranks, options.nranks = %d", g->n, c->nranks);
            return DE_EINVAL;
        }
        {   // capacity: the largest all-reduce is the full displacement vector (dd_pass)
            std::lock_guard<std::mutex> lk(g->m);
            if (g->cap < size_t(hs.ndof)) {
                if (g->slots) cudaFree(g->slots);
                g->slots = nullptr;
                g->cap = 0;
                DE_CUDA(cudaMalloc(&g->slots, size_t(g->n) * hs.ndof * sizeof(double)));
                g->cap = size_t(hs.ndof);
            }
        }
        c->lb = g;
        g->barrier();   // every rank's setup (and the slot allocation) is done before any exchange
    } else if (c->nranks > 1) {
        if (!nccl().ok) {
            set_error("nranks > 1 but libnccl.so.2 could not be loaded");
            return DE_ENCCL;
        }
        if (!opt.nccl_id) {
            set_error("nranks > 1 requires options.nccl_id");
            return DE_EINVAL;
        }
        NcclId id;
        memcpy(id.internal, opt.nccl_id, 128);
        int r = nccl().init_rank(&c->comm, c->nranks, id, c->rank);
        if (r != 0) {
            set_error("ncclCommInitRank failed: %s", nccl().errstr ? nccl().errstr(r) : "?");
            return DE_ENCCL;
        }
    }
    // ---- stats
    de_stats_t& S = c->stats;
    S.ndof = hs.ndof;
    S.n_free = hs.n_free;
    S.n_I = hs.n_I;
    S.n_Gamma = hs.n_G;
    S.n_sub = hs.nsub;
    S.n_sub_local = c->nsl;
    S.band = hs.band;
    S.singular_components = hs.singular_mask;
    for (int cc = 0; cc < hs.ncomp; ++cc) {
        S.n_cross[cc] = hs.n_cross_c[cc];
        S.n_faces[cc] = hs.n_faces_c[cc];
        S.n_gamma_c[cc] = hs.comp_off[cc + 1] - hs.comp_off[cc];
    }
    // algorithmic bytes of one Schur apply on this rank: one pass over the factor band entries
    // (b+1 per row) + the ring matrices + the local interface vectors
    double fb = 0.0;
    for (const auto& d : c->hsd) fb += double(d.nI) * (hs.band + 1) * 8.0;
    S.bytes_factor = fb;
    S.schur_explicit = c->explicit_schur ? 1 : 0;
    S.bytes_schur_explicit = double(c->n_sexp) * 8.0 + double(c->n_local_G) * (8.0 * 3 + 4.0);
    S.bytes_schur = fb + double(c->n_ig + c->n_gx) * 12.0 + double(c->n_local_G) * (8.0 * 3 + 4.0) +
                    double(c->n_local_I + c->nsl) * 4.0;
    S.bytes_iter = fb + double(c->n_ig + c->n_gx) * 12.0 + double(c->n_local_G) * 8.0 * 3.0 +
                   double(hs.n_G) * 8.0 * 11.0;
    S.bytes_prec = c->have_prec ? prec_bytes_model(hs, c->P.kmax, c->use_coop && c->coop.gram_cgs2,
                                                   c->use_coop && c->coop.fold) : 0.0;
    S.bytes_prec_min = c->have_prec ? prec_min_bytes(hs, c->P.kmax) : 0.0;
    return DE_OK;
}

de_status_t factor_impl(de_ctx* c) {
    HostSetup& hs = c->hs;
    if (c->opt.host_only) {
        set_error("context was created with host_only = 1");
        return DE_ESTATE;
    }
    if (c->opt.weighted_trace && c->dens_dirty && c->have_prec) TRY(rebuild_weighted_prec(c));
    cudaEvent_t e0, e1;
    DE_CUDA(cudaEventCreate(&e0));
    DE_CUDA(cudaEventCreate(&e1));
    DE_CUDA(cudaEventRecord(e0, c->st));
    launch_simp(c->d_rho, c->d_Ee, hs.nelem, c->E0, c->Emin, c->p, c->st);
    launch_assemble_band(c->md, c->d_sd, c->nsl, c->d_idofs, c->d_Ee, c->d_band, hs.ld, hs.band, c->max_nI, c->st);
    launch_assemble_pairs(c->md, c->d_ig_da, c->d_ig_db, c->d_ig_sub, c->d_Ee, c->d_ig_val, c->n_ig, c->st);
    launch_assemble_pairs(c->md, c->d_gx_da, c->d_gx_db, c->d_gx_sub, c->d_Ee, c->d_gx_val, c->n_gx, c->st);
    DE_CUDA(cudaMemsetAsync(c->d_fail, 0, sizeof(int), c->st));
    launch_band_cholesky(c->d_sd, c->nsl, c->d_band, hs.ld, hs.band, c->d_fail, c->st);
    if (c->d_dinv) launch_blk_diag_inv(c->d_sd, c->nsl, c->d_band, hs.ld, c->d_dinv, c->dinv_np, c->dinv_bs, c->st);
    if (c->explicit_schur)   // S_s e_t for every local Gamma dof t, through the same interior solves
        for (int s0 = 0; s0 < c->nsl; s0 += c->col_batch) {
            SchurArgs a = schur_args(c, SCHUR_COLUMNS, nullptr, nullptr, nullptr, nullptr);
            a.col_s0 = s0;
            a.nsl = std::min(c->col_batch, c->nsl - s0);
            a.sexp = c->d_sexp;
            a.colscratch = c->d_colscratch;
            a.max_nI = c->max_nI;
            a.max_ig = c->max_ig;
            launch_schur_local(a, c->st);
        }
    TRY(check_launch());
    DE_CUDA(cudaEventRecord(e1, c->st));
    int fail = 0;
    DE_CUDA(cudaMemcpyAsync(&fail, c->d_fail, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    DE_CUDA(cudaStreamSynchronize(c->st));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    c->stats.ms_factor = ms;
    double any_fail = fail ? 1.0 : 0.0;
    if (c->nranks > 1) {   // every rank must agree, or the healthy ranks would block in the next exchange
        DE_CUDA(cudaMemcpyAsync(c->d_scal, &any_fail, sizeof(double), cudaMemcpyHostToDevice, c->st));
        TRY(allreduce(c, c->d_scal, 1));
        DE_CUDA(cudaMemcpyAsync(&any_fail, c->d_scal, sizeof(double), cudaMemcpyDeviceToHost, c->st));
        DE_CUDA(cudaStreamSynchronize(c->st));
    }
    if (fail || any_fail > 0.0) {
        c->factored = false;
        if (fail)
            set_error("non-positive pivot in the interior factorisation of subdomain %d", fail - 1);
        else
            set_error("non-positive pivot in the interior factorisation on another rank");
        return DE_ENOTSPD;
    }
    c->factored = true;
    return DE_OK;
}

// One pass of Eq. (7) for load vector d_rhs: condense, interface PCG to the
// absolute recursive tolerance tol_abs (x0 = previous u_Gamma when warm), back-substitute into d_out.
de_status_t dd_pass(de_ctx* c, const double* d_rhs, double tol_abs, bool warm, int maxit, double* d_out,
                    PcgState& hsv) {
    const int64_t nG = c->hs.n_G;
    launch_gather_gamma(c->d_gamma_dofs, d_rhs, c->d_fG, nG, c->st);
    launch_schur_local(schur_args(c, SCHUR_CONDENSE, nullptr, d_rhs, nullptr, nullptr), c->st);
    launch_gather(c->d_gptr, c->d_gsrc, c->d_qloc, c->rank == 0 ? c->d_fG : nullptr, c->d_g, nG, nullptr, c->st);
    c->launches += 3;
    TRY(check_launch());
    TRY(allreduce(c, c->d_g, size_t(nG)));
    hsv = PcgState{};
    hsv.tol2 = tol_abs * tol_abs;
    hsv.maxit = maxit;
    DE_CUDA(cudaMemcpyAsync(c->d_state, &hsv, sizeof(PcgState), cudaMemcpyHostToDevice, c->st));
    if (warm) {
        launch_copy(c->d_x, c->d_xprev, nG, nullptr, c->st);
        TRY(schur_apply(c, c->d_x, c->d_q));
        launch_pcg_init(c->d_r, c->d_p, c->d_z, c->d_g, c->d_q, nG, 1, c->rb, c->d_state, c->st);
        c->launches += 4;
    } else {
        DE_CUDA(cudaMemsetAsync(c->d_x, 0, sizeof(double) * nG, c->st));
        launch_pcg_init(c->d_r, c->d_p, c->d_z, c->d_g, nullptr, nG, 0, c->rb, c->d_state, c->st);
        c->launches += 1;
    }
    int np = 0;
    TRY(precond(c, c->d_r, c->d_z, c->d_state, &np));
    launch_pcg_init(c->d_r, c->d_p, c->d_z, c->d_g, nullptr, nG, 2, c->rb, c->d_state, c->st);
    c->launches += np + 1;
    TRY(check_launch());
    TRY(read_state(c, &hsv));
    if (!hsv.done && maxit > 0) TRY(run_loop(c, hsv));
    // back-substitution u_I = A_II^-1 (rhs_I - A_IG u_G); u_G = x; u_D = 0
    DE_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double) * c->hs.ndof, c->st));
    if (c->rank == 0) launch_scatter_gamma(c->d_gamma_dofs, c->d_x, d_out, nG, c->st);
    launch_schur_local(schur_args(c, SCHUR_BACKSUB, c->d_x, d_rhs, d_out, nullptr), c->st);
    c->launches += 2;
    TRY(check_launch());
    return allreduce(c, d_out, size_t(c->hs.ndof));
}

// res = f - K (u + ulo) (free dofs; ulo may be null), returns ||res||^2 on the host
de_status_t true_residual(de_ctx* c, const double* d_f, const double* d_u, double* r2, const double* d_ulo = nullptr) {
    launch_apply_K(c->md, c->d_Ee, d_u, d_f, c->d_cls, c->d_res, c->hs.ndof, c->st, d_ulo);
    launch_norm2(c->d_res, c->hs.ndof, c->rb, c->d_scal, c->st);
    c->launches += 2;
    TRY(check_launch());
    DE_CUDA(cudaMemcpyAsync(r2, c->d_scal, sizeof(double), cudaMemcpyDeviceToHost, c->st));
    DE_CUDA(cudaStreamSynchronize(c->st));
    return DE_OK;
}

// DE_EBREAKDOWN when the last preconditioner application met a non-positive Ritz value or a non-SPD Gram matrix in
// some component (reading R9); the caller has synchronised the stream
de_status_t prec_breakdown_status(de_ctx* c) {
    if (!c->have_prec) return DE_OK;
    LzState lz[MAXC];
    DE_CUDA(cudaMemcpy(lz, c->P.lz, sizeof(lz), cudaMemcpyDeviceToHost));
    for (int cc = 0; cc < c->hs.ncomp; ++cc)
        if (lz[cc].status == DE_EBREAKDOWN) {
            set_error("non-positive Ritz value in component %d", cc);
            return DE_EBREAKDOWN;
        }
    return DE_OK;
}

// z = P~^-1 v on full dof vectors: z_Gamma = S~^-1 v_Gamma (the interface preconditioner),
// z_I = K_II^-1 (v_I - K_IGamma z_Gamma) (the back-substitution of the Schur kernels), Dirichlet entries 0
de_status_t prec_full(de_ctx* c, const double* v, double* z) {
    HostSetup& hs = c->hs;
    launch_gather_gamma(c->d_gamma_dofs, v, c->fg_vG, hs.n_G, c->st);
    // the literal two-pass CGS2 inside the preconditioner under FGMRES: measured, the one-pass form (R21) lets
    // FGMRES on the paper problem (h = 1/32, N = 16) stall at 1.06e-8 (tests/test_fgmres_gpu.py)
    TRY(precond(c, c->fg_vG, c->fg_zG, nullptr, nullptr, true));
    DE_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * hs.ndof, c->st));
    launch_scatter_gamma(c->d_gamma_dofs, c->fg_zG, z, hs.n_G, c->st);
    launch_schur_local(schur_args(c, SCHUR_BACKSUB, c->fg_zG, v, z, nullptr), c->st);
    c->launches += 3;
    return check_launch();
}

// Right-preconditioned flexible GMRES(m) on K u = f over the free dofs (NEXT(4)); Arnoldi by
// classical Gram-Schmidt applied twice (two batched fixed-order dot products per step), Givens rotations on the
// host; stop when the estimate reaches rtol ||f|| (the true residual is recomputed at every restart).
de_status_t fgmres_impl(de_ctx* c, const double* d_f, double rtol, double fnorm, double* d_u, int32_t* iters,
                        double* relres) {
    HostSetup& hs = c->hs;
    if (c->nranks > 1) {
        set_error("outer = 1 (full-system FGMRES) is single-rank in this version");
        return DE_EINVAL;
    }
    const int m = std::min(std::max(1, c->opt.restart), FG_ND - 1);
    const size_t nd = size_t(hs.ndof);
    if (c->fg_m != m) {
        TRY(dalloc(c, &c->fg_V, (m + 1) * nd));
        TRY(dalloc(c, &c->fg_Z, m * nd));
        TRY(dalloc(c, &c->fg_w, nd));
        TRY(dalloc(c, &c->fg_r, nd));
        TRY(dalloc(c, &c->fg_zero, nd));
        TRY(dalloc(c, &c->fg_vG, size_t(hs.n_G)));
        TRY(dalloc(c, &c->fg_zG, size_t(hs.n_G)));
        TRY(dalloc(c, &c->fg_h, size_t(2 * FG_ND + 8)));
        c->fg_rb.nblk = c->rb.nblk;
        TRY(dalloc(c, &c->fg_rb.part, size_t(c->fg_rb.nblk) * FG_ND));
        TRY(dalloc(c, &c->fg_rb.counter, 1));
        DE_CUDA(cudaMemsetAsync(c->fg_rb.counter, 0, sizeof(unsigned int), c->st));
        DE_CUDA(cudaMemsetAsync(c->fg_zero, 0, sizeof(double) * nd, c->st));
        c->fg_m = m;
    }
    const int maxit = c->opt.max_iter > 0 ? c->opt.max_iter : 20000;
    const double tol = rtol * fnorm;
    DE_CUDA(cudaMemsetAsync(d_u, 0, sizeof(double) * nd, c->st));
    std::vector<double> H(size_t(m + 1) * m), cs(m), sn(m), g(m + 1), hb(2 * FG_ND + 2);
    int its = 0, cycles = 0;
    double r2 = 0.0;
    double* hd = c->fg_h;   // [0, FG_ND): first pass, [FG_ND, 2 FG_ND): second pass, [2 FG_ND]: ||w||^2
    while (true) {
        TRY(true_residual(c, d_f, d_u, &r2));   // d_res = K u - f (Dirichlet 0)
        if (std::sqrt(r2) <= tol || its >= maxit) break;
        DE_CUDA(cudaMemsetAsync(c->fg_r, 0, sizeof(double) * nd, c->st));
        launch_axpy(c->fg_r, c->d_res, -1.0, hs.ndof, c->st);
        DE_CUDA(cudaMemcpyAsync(c->d_scal, &r2, sizeof(double), cudaMemcpyHostToDevice, c->st));
        launch_scale_invnorm(c->fg_V, c->fg_r, c->d_scal, hs.ndof, c->st);
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = std::sqrt(r2);
        int k = 0;
        for (int j = 0; j < m; ++j) {
            double* Vj = c->fg_V + j * nd;
            double* Zj = c->fg_Z + j * nd;
            TRY(prec_full(c, Vj, Zj));
            launch_apply_K(c->md, c->d_Ee, Zj, c->fg_zero, c->d_cls, c->fg_w, hs.ndof, c->st);
            launch_multidot(c->fg_V, nd, j + 1, c->fg_w, hs.ndof, c->fg_rb, hd, c->st);
            launch_multi_axpy(c->fg_w, c->fg_V, nd, j + 1, hd, -1.0, hs.ndof, c->st);
            launch_multidot(c->fg_V, nd, j + 1, c->fg_w, hs.ndof, c->fg_rb, hd + FG_ND, c->st);
            launch_multi_axpy(c->fg_w, c->fg_V, nd, j + 1, hd + FG_ND, -1.0, hs.ndof, c->st);
            launch_norm2(c->fg_w, hs.ndof, c->rb, hd + 2 * FG_ND, c->st);
            launch_scale_invnorm(c->fg_V + (j + 1) * nd, c->fg_w, hd + 2 * FG_ND, hs.ndof, c->st);
            c->launches += 8;
            TRY(check_launch());
            DE_CUDA(cudaMemcpyAsync(hb.data(), hd, sizeof(double) * (2 * FG_ND + 1), cudaMemcpyDeviceToHost, c->st));
            DE_CUDA(cudaStreamSynchronize(c->st));
            TRY(prec_breakdown_status(c));   // z_Gamma = 0 from a broken-down application is not a direction
            for (int i = 0; i <= j; ++i) H[size_t(i) * m + j] = hb[i] + hb[FG_ND + i];
            H[size_t(j + 1) * m + j] = std::sqrt(std::max(hb[2 * FG_ND], 0.0));
            for (int i = 0; i < j; ++i) {   // previous rotations
                const double a = H[size_t(i) * m + j], b = H[size_t(i + 1) * m + j];
                H[size_t(i) * m + j] = cs[i] * a + sn[i] * b;
                H[size_t(i + 1) * m + j] = -sn[i] * a + cs[i] * b;
            }
            const double a = H[size_t(j) * m + j], b = H[size_t(j + 1) * m + j], rho = std::hypot(a, b);
            cs[j] = rho > 0.0 ? a / rho : 1.0;
            sn[j] = rho > 0.0 ? b / rho : 0.0;
            H[size_t(j) * m + j] = rho;
            H[size_t(j + 1) * m + j] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            ++its;
            k = j + 1;
            if (std::fabs(g[j + 1]) <= tol || its >= maxit) break;
        }
        std::vector<double> y(k);
        for (int i = k - 1; i >= 0; --i) {   // H y = g (upper triangular)
            double t = g[i];
            for (int jj = i + 1; jj < k; ++jj) t -= H[size_t(i) * m + jj] * y[jj];
            y[i] = t / H[size_t(i) * m + i];
        }
        DE_CUDA(cudaMemcpyAsync(hd, y.data(), sizeof(double) * k, cudaMemcpyHostToDevice, c->st));
        launch_multi_axpy(d_u, c->fg_Z, nd, k, hd, 1.0, hs.ndof, c->st);
        c->launches += 1;
        ++cycles;
    }
    c->stats.iterations = c->stats.iterations_pass1 = its;
    c->stats.restarts = cycles;
    c->stats.relres_true = c->stats.relres_recursive = c->stats.relres_dd = std::sqrt(r2) / fnorm;
    c->stats.kernels_launched = c->launches;
    if (iters) *iters = its;
    if (relres) *relres = c->stats.relres_true;
    if (std::sqrt(r2) > tol) {
        set_error("FGMRES did not reach rtol in %d iterations (true relres %.3e)", its, c->stats.relres_true);
        return DE_ENOCONV;
    }
    return DE_OK;
}

de_status_t solve_impl(de_ctx* c, const double* d_f, double rtol, double* d_u, int32_t* iters, double* relres) {
    if (!c->factored) {
        set_error("de_solve called before a successful de_factor");
        return DE_ESTATE;
    }
    if (!(rtol > 0)) {
        set_error("rtol must be positive");
        return DE_EINVAL;
    }
    HostSetup& hs = c->hs;
    auto t0 = std::chrono::steady_clock::now();
    c->launches = 0;
    double f2 = 0.0;
    TRY(masked_norm2(c, d_f, &f2));
    c->launches += 3;
    const double fnorm = std::sqrt(f2);
    if (!std::isfinite(fnorm)) {
        set_error("rhs has non-finite entries on free dofs");
        return DE_EINVAL;
    }
    c->stats.iterations = 0;
    c->stats.restarts = 0;
    if (fnorm == 0.0) {
        DE_CUDA(cudaMemsetAsync(d_u, 0, sizeof(double) * hs.ndof, c->st));
        DE_CUDA(cudaStreamSynchronize(c->st));
        if (iters) *iters = 0;
        if (relres) *relres = 0.0;
        c->stats.relres_true = c->stats.relres_recursive = c->stats.relres_dd = 0.0;
        return DE_OK;
    }
    if (c->opt.outer == 1) {
        auto ta = std::chrono::steady_clock::now();
        const de_status_t st = fgmres_impl(c, d_f, rtol, fnorm, d_u, iters, relres);
        c->stats.ms_solve = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ta).count();
        return st;
    }
    const int maxit = c->opt.max_iter > 0 ? c->opt.max_iter : 20000;
    cudaEvent_t l0, l1;
    DE_CUDA(cudaEventCreate(&l0));
    DE_CUDA(cudaEventCreate(&l1));
    DE_CUDA(cudaEventRecord(l0, c->st));
    PcgState hsv{};
    TRY(dd_pass(c, d_f, rtol * fnorm, c->opt.warm_start && c->have_prev, maxit, d_u, hsv));
    int its = hsv.it, status = hsv.status, refines = 0;
    c->stats.iterations_pass1 = hsv.it;
    bool conv = hsv.rr <= hsv.tol2;
    double rec = std::sqrt(std::max(hsv.rr, 0.0)) / fnorm;
    double r2 = 0.0;
    TRY(true_residual(c, d_f, d_u, &r2));
    // iterative refinement on the full system (R11/R17): (u_hi, u_lo) += DD(f - K (u_hi + u_lo)) with
    // the iterate carried as a double-double sum, so the FP64 rounding of u does not stop the refinement; stop
    // when the double-double iterate meets rtol or a round no longer halves its residual
    DE_CUDA(cudaMemsetAsync(c->d_ulo, 0, sizeof(double) * hs.ndof, c->st));
    double r2_prev = HUGE_VAL;
    bool have_lo = false;
    while (std::sqrt(r2) > rtol * fnorm && conv && status != DE_EBREAKDOWN && its < maxit && refines < 3 &&
           r2 < 0.25 * r2_prev) {
        r2_prev = r2;
        TRY(dd_pass(c, c->d_res, 0.5 * rtol * fnorm, false, maxit - its, c->d_ubuf2, hsv));
        launch_dd_accum(d_u, c->d_ulo, c->d_ubuf2, hs.ndof, c->st);
        c->launches += 1;
        have_lo = true;
        its += hsv.it;
        status = hsv.status;
        conv = hsv.rr <= hsv.tol2;
        ++refines;
        TRY(true_residual(c, d_f, d_u, &r2, c->d_ulo));
    }
    const double r2_dd = r2;   // residual of the double-double iterate u_hi + u_lo
    if (have_lo) TRY(true_residual(c, d_f, d_u, &r2));   // of the returned u = u_hi = fl(u_hi + u_lo)
    DE_CUDA(cudaEventRecord(l1, c->st));
    launch_gather_gamma(c->d_gamma_dofs, d_u, c->d_xprev, hs.n_G, c->st);   // warm start for the next solve
    c->launches += 1;
    c->have_prev = true;
    DE_CUDA(cudaStreamSynchronize(c->st));
    float lms = 0.f;
    cudaEventElapsedTime(&lms, l0, l1);
    cudaEventDestroy(l0);
    cudaEventDestroy(l1);
    auto t1 = std::chrono::steady_clock::now();
    c->stats.iterations = its;
    c->stats.restarts = refines;
    c->stats.relres_recursive = rec;
    c->stats.relres_true = std::sqrt(r2) / fnorm;
    c->stats.relres_dd = std::sqrt(r2_dd) / fnorm;
    c->stats.ms_pcg = lms;
    c->stats.ms_solve = std::chrono::duration<double, std::milli>(t1 - t0).count();
    c->stats.launches_per_iter = c->launches_per_iter;
    c->stats.kernels_launched = c->launches;
    if (iters) *iters = its;
    if (relres) *relres = c->stats.relres_true;
    if (status == DE_EBREAKDOWN) {
        set_error("PCG breakdown (p^T S p <= 0 or a non-positive Ritz value) at iteration %d", its);
        return DE_EBREAKDOWN;
    }
    // R17: the computed (double-double) solution must meet rtol; the returned FP64 u = fl(u_hi + u_lo) may sit
    // above rtol only by its own rounding (relres_true, >= the FP64 floor of the problem)
    if (!conv || c->stats.relres_dd > rtol) {
        set_error("did not reach rtol in %d iterations (true relres %.3e, double-double iterate %.3e, "
                  "recursive %.3e)", its, c->stats.relres_true, c->stats.relres_dd, rec);
        return DE_ENOCONV;
    }
    return DE_OK;
}

}  // namespace

// ====================================================================== C ABI

static de_status_t need_device(const de_ctx_t* c) {
    if (c->opt.host_only) {
        set_error("context was created with host_only = 1");
        return DE_ESTATE;
    }
    return DE_OK;
}


extern "C" {

void de_default_options(de_options_t* o) {
    if (!o) return;
    memset(o, 0, sizeof(*o));
    o->theta = 0.5;
    o->lanczos_k = 10;
    o->inner_mode = 1;
    o->inner_tol = 1e-3;
    o->inner_max_iter = 1000;
    o->max_iter = 20000;
    o->beta_variant = 0;
    o->warm_start = 0;
    o->rank = 0;
    o->nranks = 1;
    o->device = 0;
    o->nccl_id = nullptr;
    o->stream = nullptr;
    o->check_every = 8;
    o->use_graph = 1;
    o->outer = 0;
    o->restart = 30;
}

const char* de_last_error(void) { return g_err; }

de_status_t de_setup(const de_mesh_t* mesh, const double* density, double E0, double Emin, double p, double nu,
                     const de_partition_t* part, const de_options_t* opt, de_ctx_t** out) {
    if (!out) {
        set_error("null out pointer");
        return DE_EINVAL;
    }
    *out = nullptr;
    de_ctx* c = new (std::nothrow) de_ctx();
    if (!c) return DE_ENOMEM;
    de_status_t s;
    try {
        s = setup_impl(mesh, density, E0, Emin, p, nu, part, opt, c);
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed");
        s = DE_ENOMEM;
    }
    if (s != DE_OK) {
        std::string keep = g_err;
        de_destroy(c);
        snprintf(g_err, sizeof(g_err), "%s", keep.c_str());
        return s;
    }
    *out = c;
    return DE_OK;
}

de_status_t de_update_densities(de_ctx_t* c, const double* density) {
    if (!c || !density) {
        set_error("null argument");
        return DE_EINVAL;
    }
    for (int64_t e = 0; e < c->hs.nelem; ++e)
        if (!(density[e] > 0.0) || !std::isfinite(density[e])) {
            set_error("density[%lld] must be positive and finite", (long long)e);
            return DE_EINVAL;
        }
    TRY(need_device(c));
    DE_CUDA(cudaSetDevice(c->opt.device));
    DE_CUDA(cudaMemcpyAsync(c->d_rho, density, sizeof(double) * c->hs.nelem, cudaMemcpyHostToDevice, c->st));
    c->factored = false;
    c->dens_dirty = true;
    return DE_OK;
}

de_status_t de_update_densities_device(de_ctx_t* c, const double* d_density) {
    if (!c || !d_density) {
        set_error("null argument");
        return DE_EINVAL;
    }
    TRY(need_device(c));
    DE_CUDA(cudaSetDevice(c->opt.device));
    DE_CUDA(cudaMemcpyAsync(c->d_rho, d_density, sizeof(double) * c->hs.nelem, cudaMemcpyDeviceToDevice, c->st));
    c->factored = false;
    c->dens_dirty = true;
    return DE_OK;
}

de_status_t de_factor(de_ctx_t* c) {
    if (!c) {
        set_error("null context");
        return DE_EINVAL;
    }
    TRY(need_device(c));
    DE_CUDA(cudaSetDevice(c->opt.device));
    return factor_impl(c);
}

de_status_t de_solve_device(de_ctx_t* c, const double* d_rhs, double rtol, double* d_u, int32_t* iterations,
                            double* final_relres) {
    if (!c || !d_rhs || !d_u) {
        set_error("null argument");
        return DE_EINVAL;
    }
    TRY(need_device(c));
    DE_CUDA(cudaSetDevice(c->opt.device));
    return solve_impl(c, d_rhs, rtol, d_u, iterations, final_relres);
}

de_status_t de_solve(de_ctx_t* c, const double* rhs, double rtol, double* u, int32_t* iterations,
                     double* final_relres) {
    if (!c || !rhs || !u) {
        set_error("null argument");
        return DE_EINVAL;
    }
    TRY(need_device(c));
    DE_CUDA(cudaSetDevice(c->opt.device));
    const size_t nb = sizeof(double) * size_t(c->hs.ndof);
    DE_CUDA(cudaMemcpyAsync(c->d_fbuf, rhs, nb, cudaMemcpyHostToDevice, c->st));
    de_status_t s = solve_impl(c, c->d_fbuf, rtol, c->d_ubuf, iterations, final_relres);
    if (s != DE_OK && s != DE_ENOCONV) return s;
    DE_CUDA(cudaMemcpyAsync(u, c->d_ubuf, nb, cudaMemcpyDeviceToHost, c->st));
    DE_CUDA(cudaStreamSynchronize(c->st));
    return s;
}

de_status_t de_get_dofmap(const de_ctx_t* c, int8_t* cls, int32_t* sub, int32_t* reduced, int64_t* n_I,
                          int64_t* n_Gamma) {
    if (!c) {
        set_error("null context");
        return DE_EINVAL;
    }
    const HostSetup& hs = c->hs;
    if (cls) memcpy(cls, hs.cls.data(), hs.ndof);
    if (sub) memcpy(sub, hs.dof_sub.data(), hs.ndof * sizeof(int32_t));
    if (reduced) memcpy(reduced, hs.reduced.data(), hs.ndof * sizeof(int32_t));
    if (n_I) *n_I = hs.n_I;
    if (n_Gamma) *n_Gamma = hs.n_G;
    return DE_OK;
}

de_status_t de_get_skeleton(const de_ctx_t* c, int32_t comp, int32_t* nodes, int32_t* face_of_node) {
    if (!c || comp < 0 || comp >= c->hs.ncomp) {
        set_error("bad component");
        return DE_EINVAL;
    }
    const HostSetup& hs = c->hs;
    // ascending node order (the internal flattened order is face-major)
    std::vector<std::pair<int32_t, int32_t>> nf;
    for (int64_t f = hs.comp_off[comp]; f < hs.comp_off[comp + 1]; ++f) nf.push_back({hs.cnode[f], hs.face_of[f]});
    std::sort(nf.begin(), nf.end());
    for (size_t q = 0; q < nf.size(); ++q) {
        if (nodes) nodes[q] = nf[q].first;
        if (face_of_node) face_of_node[q] = nf[q].second;
    }
    return DE_OK;
}

de_status_t de_get_owned(const de_ctx_t* c, int32_t* ids, int32_t* n) {
    if (!c || !n) {
        set_error("null argument");
        return DE_EINVAL;
    }
    *n = c->nsl;
    if (ids)
        for (int k = 0; k < c->nsl; ++k) ids[k] = c->owned[k];
    return DE_OK;
}

de_status_t de_get_stats(const de_ctx_t* c, de_stats_t* s) {
    if (!c || !s) {
        set_error("null argument");
        return DE_EINVAL;
    }
    *s = c->stats;
    s->inner_iterations = 0;
    if (c->have_prec && c->P.inner_f && c->P.fits) {
        unsigned long long n = 0;
        DE_CUDA(cudaMemcpyAsync(&n, c->P.fits, sizeof(n), cudaMemcpyDeviceToHost, c->st));
        DE_CUDA(cudaStreamSynchronize(c->st));
        s->inner_iterations = int64_t(n);
    }
    return DE_OK;
}

de_status_t de_schur_apply_device(de_ctx_t* c, const double* d_p, double* d_q) {
    if (!c || !d_p || !d_q) {
        set_error("null argument");
        return DE_EINVAL;
    }
    if (!c->factored) {
        set_error("de_schur_apply_device before de_factor");
        return DE_ESTATE;
    }
    TRY(need_device(c));
    DE_CUDA(cudaSetDevice(c->opt.device));
    TRY(schur_apply(c, d_p, d_q));
    DE_CUDA(cudaStreamSynchronize(c->st));
    return DE_OK;
}

de_status_t de_precond_apply_device(de_ctx_t* c, const double* d_r, double* d_z) {
    if (!c || !d_r || !d_z) {
        set_error("null argument");
        return DE_EINVAL;
    }
    TRY(need_device(c));
    DE_CUDA(cudaSetDevice(c->opt.device));
    TRY(precond(c, d_r, d_z, nullptr, nullptr));
    DE_CUDA(cudaStreamSynchronize(c->st));
    return prec_breakdown_status(c);
}

de_status_t de_get_factor_band(const de_ctx_t* c, int32_t sl, double* out, int32_t* n_I_s) {
    if (!c || sl < 0 || sl >= c->nsl) {
        set_error("bad local subdomain index");
        return DE_EINVAL;
    }
    const SubDesc& d = c->hsd[sl];
    if (n_I_s) *n_I_s = d.nI;
    if (out) {
        const int ld = c->hs.ld, w = c->hs.band + 1;
        std::vector<double> tmp(size_t(d.nI) * ld);
        DE_CUDA(cudaMemcpy(tmp.data(), c->d_band + d.band_off, tmp.size() * sizeof(double), cudaMemcpyDeviceToHost));
        for (int j = 0; j < d.nI; ++j)
            for (int k = 0; k < w; ++k) out[size_t(j) * w + k] = tmp[size_t(j) * ld + k];
        if (c->factored)   // slot 0 holds 1/L_jj internally
            for (int j = 0; j < d.nI; ++j) out[size_t(j) * w] = 1.0 / out[size_t(j) * w];
    }
    return DE_OK;
}

de_status_t de_get_assembled_band(de_ctx_t* c, int32_t sl, double* out, int32_t* n_I_s) {
    if (!c || sl < 0 || sl >= c->nsl) {
        set_error("bad local subdomain index");
        return DE_EINVAL;
    }
    TRY(need_device(c));
    DE_CUDA(cudaSetDevice(c->opt.device));
    const HostSetup& hs = c->hs;
    launch_simp(c->d_rho, c->d_Ee, hs.nelem, c->E0, c->Emin, c->p, c->st);
    launch_assemble_band(c->md, c->d_sd, c->nsl, c->d_idofs, c->d_Ee, c->d_band, hs.ld, hs.band, c->max_nI, c->st);
    TRY(check_launch());
    DE_CUDA(cudaStreamSynchronize(c->st));
    c->factored = false;   // the band now holds A_II, not its factor
    return de_get_factor_band(c, sl, out, n_I_s);
}

de_status_t de_nccl_unique_id(void* out128) {
    if (!out128) {
        set_error("null argument");
        return DE_EINVAL;
    }
    if (!nccl().ok) {
        set_error("libnccl.so.2 could not be loaded");
        return DE_ENCCL;
    }
    NcclId id;
    int r = nccl().get_id(&id);
    if (r != 0) {
        set_error("ncclGetUniqueId failed");
        return DE_ENCCL;
    }
    memcpy(out128, id.internal, 128);
    return DE_OK;
}

de_status_t de_set_profiling(de_ctx_t* c, int32_t on) {
    if (!c) {
        set_error("null context");
        return DE_EINVAL;
    }
    c->profiling = on != 0;
    c->prof_ms = 0.0;
    c->prof_n = 0;
    c->prof_ms_prec = 0.0;
    c->prof_n_prec = 0;
    return DE_OK;
}

// diagnostics: copy the cooperative preconditioner's phase stamps (ns) of the last application
extern "C" int de_debug_prec_timers(const de_ctx_t* c, unsigned long long* out, int n) {
    if (!c || !c->coop.timers || n > 200 + 8192) return -1;
    cudaMemcpy(out, c->coop.timers, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost);
    return 0;
}

de_status_t de_get_kernel_time(const de_ctx_t* c, double* ms, int64_t* launches) {
    if (!c) {
        set_error("null context");
        return DE_EINVAL;
    }
    if (ms) *ms = c->prof_n ? c->prof_ms / double(c->prof_n) : 0.0;
    if (launches) *launches = c->prof_n;
    return DE_OK;
}

de_status_t de_get_prec_time(const de_ctx_t* c, double* ms, int64_t* launches) {
    if (!c) {
        set_error("null context");
        return DE_EINVAL;
    }
    if (ms) *ms = c->prof_n_prec ? c->prof_ms_prec / double(c->prof_n_prec) : 0.0;
    if (launches) *launches = c->prof_n_prec;
    return DE_OK;
}

void de_default_oc_params(de_oc_params_t* p) {
    if (!p) return;
    p->volfrac = 0.5;
    p->move = 0.2;
    p->rho_min = 1e-3;
    p->eta = 0.5;
    p->tol = 1e-12;
    p->maxit = 200;
}

namespace {
de_status_t oc_alloc(de_ctx* c) {
    if (c->oc_dc) return DE_OK;
    const int64_t n = c->hs.nelem;
    TRY(dalloc(c, &c->oc_dc, size_t(n)));
    TRY(dalloc(c, &c->oc_rho, size_t(n)));
    TRY(dalloc(c, &c->oc_part, size_t(2 * oc_blocks(n))));
    TRY(dalloc(c, &c->oc_st, 1));
    return DE_OK;
}

de_status_t oc_check(const de_oc_params_t* p) {
    if (!p) {
        set_error("null OC parameters");
        return DE_EINVAL;
    }
    if (!(p->volfrac > 0.0 && p->volfrac <= 1.0) || !(p->move > 0.0) || !(p->rho_min > 0.0 && p->rho_min < 1.0) ||
        !(p->eta > 0.0) || !(p->tol > 0.0) || p->maxit < 1 || p->maxit > 10000) {
        set_error("OC parameters out of range (volfrac in (0,1], move > 0, rho_min in (0,1), eta > 0, tol > 0, "
                  "maxit in [1, 10000])");
        return DE_EINVAL;
    }
    return DE_OK;
}

OcParams oc_params(const de_oc_params_t* p) {
    return OcParams{p->volfrac, p->move, p->rho_min, p->eta, p->tol, p->maxit};
}
}  // namespace

de_status_t de_sensitivities_device(de_ctx_t* c, const double* d_u, double* d_dc, double* compliance) {
    if (!c || !d_u) {
        set_error("null argument");
        return DE_EINVAL;
    }
    TRY(need_device(c));
    DE_CUDA(cudaSetDevice(c->opt.device));
    TRY(oc_alloc(c));
    const int64_t n = c->hs.nelem;
    launch_simp(c->d_rho, c->d_Ee, n, c->E0, c->Emin, c->p, c->st);
    c->launches += 1 + launch_sensitivities(c->md, d_u, c->d_rho, c->d_Ee, c->E0, c->Emin, c->p, n, c->oc_dc,
                                            c->oc_part, c->oc_st, c->st);
    c->oc_have_dc = true;
    if (d_dc && d_dc != c->oc_dc)
        DE_CUDA(cudaMemcpyAsync(d_dc, c->oc_dc, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->st));
    if (compliance) {
        OcState h{};
        DE_CUDA(cudaMemcpyAsync(&h, c->oc_st, sizeof(OcState), cudaMemcpyDeviceToHost, c->st));
        DE_CUDA(cudaStreamSynchronize(c->st));
        *compliance = h.compliance;
    }
    return DE_OK;
}

de_status_t de_oc_update_device(de_ctx_t* c, const double* d_dc, const de_oc_params_t* prm, double* d_rho_new,
                                double* lambda) {
    if (!c) {
        set_error("null context");
        return DE_EINVAL;
    }
    TRY(oc_check(prm));
    TRY(need_device(c));
    DE_CUDA(cudaSetDevice(c->opt.device));
    TRY(oc_alloc(c));
    const int64_t n = c->hs.nelem;
    if (!d_dc && !c->oc_have_dc) {
        set_error("de_oc_update_device: d_dc is NULL and no de_sensitivities_device call preceded it");
        return DE_EINVAL;
    }
    if (d_dc && d_dc != c->oc_dc)
        DE_CUDA(cudaMemcpyAsync(c->oc_dc, d_dc, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->st));
    c->launches += launch_oc_update(c->d_rho, c->oc_dc, n, oc_params(prm), c->oc_part, c->oc_st, c->oc_rho, c->st);
    DE_CUDA(cudaMemcpyAsync(c->d_rho, c->oc_rho, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->st));
    if (d_rho_new)
        DE_CUDA(cudaMemcpyAsync(d_rho_new, c->oc_rho, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->st));
    c->factored = false;
    c->dens_dirty = true;
    if (lambda) {
        OcState h{};
        DE_CUDA(cudaMemcpyAsync(&h, c->oc_st, sizeof(OcState), cudaMemcpyDeviceToHost, c->st));
        DE_CUDA(cudaStreamSynchronize(c->st));
        *lambda = h.lambda;
    }
    return DE_OK;
}

de_status_t de_oc_step(de_ctx_t* c, const double* u, const de_oc_params_t* prm, double* rho_new,
                       double* compliance, double* lambda) {
    if (!c || !u) {
        set_error("null argument");
        return DE_EINVAL;
    }
    TRY(oc_check(prm));
    TRY(need_device(c));
    DE_CUDA(cudaSetDevice(c->opt.device));
    const int64_t nd = c->hs.ndof, n = c->hs.nelem;
    DE_CUDA(cudaMemcpyAsync(c->d_ubuf, u, sizeof(double) * nd, cudaMemcpyHostToDevice, c->st));
    TRY(de_sensitivities_device(c, c->d_ubuf, nullptr, compliance));
    TRY(de_oc_update_device(c, nullptr, prm, nullptr, lambda));
    if (rho_new) {
        DE_CUDA(cudaMemcpyAsync(rho_new, c->oc_rho, sizeof(double) * n, cudaMemcpyDeviceToHost, c->st));
        DE_CUDA(cudaStreamSynchronize(c->st));
    }
    return DE_OK;
}

de_status_t de_loopback_create(int32_t nranks, de_loopback_t** out) {
    if (!out || nranks < 1) {
        set_error("de_loopback_create: nranks >= 1 and a non-null out pointer required");
        return DE_EINVAL;
    }
    de_loopback_t* g = new de_loopback_t();
    g->n = nranks;
    *out = g;
    return DE_OK;
}

void de_loopback_destroy(de_loopback_t* g) {
    if (!g) return;
    if (g->slots) cudaFree(g->slots);
    delete g;
}

void de_destroy(de_ctx_t* c) {
    if (!c) return;
    if (c->opt.host_only && c->allocs.empty()) {
        delete c;
        return;
    }
    cudaSetDevice(c->opt.device);
    if (c->st) cudaStreamSynchronize(c->st);
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    for (auto e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->comm && nccl().destroy) nccl().destroy(c->comm);
    for (void* p : c->allocs) cudaFree(p);
    for (void* p : c->prec_allocs) cudaFree(p);
    if (c->own_stream && c->st) cudaStreamDestroy(c->st);
    delete c;
}

}  // extern "C"
