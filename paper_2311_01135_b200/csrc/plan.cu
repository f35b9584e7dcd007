// C ABI (include/qm1b_b200.h): batch planning, device memory, stage launches.
//
// Host-side planning is native C++ (it sits on the e2e critical path): shell-pair
// lists per molecule grouped by class, quartet-count prefixes, CTA tables for the
// J/K and XC kernels and every buffer offset are computed here, packed into one
// host blob and uploaded with a single cudaMemcpyAsync.  One stream-ordered device
// allocation holds every buffer of the batch.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "md.cuh"

namespace dftb {
void launch_pairs(const DevBatch &b, cudaStream_t s);
void launch_schwarz(const DevBatch &b, const int64_t *host_totals, cudaStream_t s);
void launch_eri(const DevBatch &b, const int64_t *tot, double eps, double prim_cut, cudaStream_t s, int *nlaunch);
void launch_enn(const DevBatch &b, cudaStream_t s);
void launch_onee(const DevBatch &b, cudaStream_t s);
void launch_grid(const DevBatch &b, int max_atoms, cudaStream_t s);
int launch_jk(const DevBatch &b, const int *bucket_ctas, const int *bucket_n, cudaStream_t s);
int launch_xc(const DevBatch &b, const int *bucket_ctas, const int *bucket_n, int nsh_max, cudaStream_t s);
void launch_orth(const DevBatch &b, int nmax, cudaStream_t s);
void launch_post(const DevBatch &b, int nmax, int it, int diis_start, int diis_hist, double damping,
                 double conv_std, cudaStream_t s);
void launch_reduce(const DevBatch &b, int which, cudaStream_t s);
void launch_fetch_dev(const DevBatch &b, double *E, double *hist, cudaStream_t s);
void launch_roothaan(const DevBatch &b, int nmax, cudaStream_t s);
void launch_diis_single(const double *F, const double *E, int mh, int n, double *out, cudaStream_t s);
void launch_eval_ao(const DevBatch &b, int mol, double *out, cudaStream_t s);
void launch_b3lyp(const double *n, const double *s, int64_t np, double *e, double *vr, double *vs, cudaStream_t st);
void launch_compact_count(const DevBatch &b, int mol, double eps, const double *qsp, int64_t *rowcnt, cudaStream_t s);
void launch_compact_write(const DevBatch &b, int mol, double eps, const double *qsp, const int64_t *rowoff,
                          uint16_t *oi, uint16_t *oj, uint16_t *ok, uint16_t *ol, double *ov, cudaStream_t s);
double fma_peak(int fp64, cudaStream_t s);
}  // namespace dftb

using namespace dftb;

static thread_local std::string g_err;
static int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}
#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) return fail(DFTB_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

static constexpr int XC_CHUNK = 2048;
// Target J/K CTAs per molecule (largest slab permitting).  A CTA's fixed costs (density load,
// zeroing and later summing its N x N exchange partial, J_Q flush, pipeline fill) favour few,
// long CTAs once the batch alone fills the GPU: measured on B200 with 256 molecules x 9 heavy
// atoms, J/K per iteration 1.05 ms at 12, 0.97 at 8, 0.95 at 4, 0.94 at 3 (296 resident CTAs).
// Small batches keep more CTAs per molecule so a single molecule still spreads over the SMs.
// QM1B_JK_SPLIT overrides (tuning runs).
static int jk_split(int n_mol, int f32_store) {
    static const int env = [] { const char *e = getenv("QM1B_JK_SPLIT"); return e ? atoi(e) : 0; }();
    if (env > 0) return env;
    if (!f32_store) return 12;                 // f64 store: k_jk (one warp per row, 4-8 warps per CTA) as tuned in round 1
    const int per = (600 + n_mol - 1) / std::max(1, n_mol);
    return std::max(4, std::min(16, per));
}
#ifndef ERI64_F32
#define ERI64_F32 0     // f32 build: keep the (f32-rounded) ERI store in f64 (no f32->f64 in J/K)
#endif     // target J/K CTAs per molecule (largest slab permitting)

struct dftb_plan {
    DevBatch d{};
    dftb_opts opts{};
    unsigned char *mem = nullptr;
    size_t mem_bytes = 0, in_bytes = 0, work_off = 0, eri_off = 0, eri_bytes = 0;
    int nmax = 0, nsh_max = 0, natom_max = 0;
    int64_t cls_tot[NCLS] = {0}, pair_tot[3] = {0};
    std::vector<int> nao, nocc, jkc0, xcc0;
    std::vector<int64_t> mat0, npp0, grid0, eri0;
    int64_t launches = 0;
    int *xc_bucket_ctas = nullptr;  // device
    int xc_bucket_n[6] = {0};
    int *jk_bucket_ctas = nullptr;  // device
    int jk_bucket_n[6] = {0};
    bool timing = false;
    cudaEvent_t ev[8] = {nullptr};
    double stage_ms[8] = {0};
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t aux = nullptr;     // J/K runs here, concurrently with XC on the caller's stream
    cudaEvent_t fork = nullptr, join = nullptr;
    cudaEvent_t fin = nullptr;      // this plan's last work on the caller's stream (fetch / free wait on it)
    bool fin_rec = false;           // fin holds the end of the last completed enqueueing call
    bool dirty = false;             // an enqueueing call started after fin was last recorded
    cudaStream_t last = nullptr;    // stream of the last enqueueing call
};

// Every entry point that enqueues device work brackets it with enq_begin / enq_end: fin then
// marks the end of this plan's submitted work on the stream the caller used, so fetch and
// the stream-ordered free wait for exactly this plan's work (not later batches the caller has
// queued on the same stream), and a call that failed partway is still covered (dirty).
static void enq_begin(dftb_plan *p, cudaStream_t st) {
    p->dirty = true;
    p->last = st;
}
static void enq_end(dftb_plan *p, cudaStream_t st) {
    if (p->fin && cudaEventRecord(p->fin, st) == cudaSuccess) {
        p->fin_rec = true;
        p->dirty = false;
    }
}

// ------------------------------------------------------------------ Boys table (per device)
static double *g_boys[64] = {nullptr};
static std::mutex g_boys_mu;   // plans are created from several host threads (pipeline workers)
static int ensure_boys(int dev, const double **out) {
    if (dev < 0 || dev >= 64) return fail(DFTB_EINVAL, "device index out of range");
    std::lock_guard<std::mutex> lock(g_boys_mu);
    if (!g_boys[dev]) {
        std::vector<double> full(BOYS_NT * BOYS_NCOL), tab((size_t)(kBoysLMax + 1) * kBoysNT * 8);
        boys_table_host(full.data());
        boys_slices_host(full.data(), tab.data());
        double *p = nullptr;
        CK(cudaMalloc(&p, tab.size() * sizeof(double)));
        CK(cudaMemcpy(p, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice));
        g_boys[dev] = p;
    }
    *out = g_boys[dev];
    return 0;
}

// ------------------------------------------------------------------ layout helper
struct Lay {
    size_t off = 0;
    template <class T>
    size_t add(size_t n) {
        size_t o = (off + 255) & ~(size_t)255;
        off = o + n * sizeof(T);
        return o;
    }
};

extern "C" {
#pragma GCC visibility push(default)

const char *dftb_last_error(void) { return g_err.c_str(); }
const char *dftb_version(void) { return "qm1b_b200 0.1.0 (sm_100a)"; }

int dftb_device_count(int *count) {
    CK(cudaGetDeviceCount(count));
    return 0;
}

// Per-device pool of {aux stream, fork event, join event}: plans take one at creation and
// return it at destruction, never destroying it.  Creating and destroying streams / events per
// plan blocked the pipeline's host threads for the duration of other batches' device work
// (measured: plan creation stalled 152 ms in cudaStreamCreateWithFlags while another batch ran),
// which cut the batches in flight of the public labeling path from 3 to ~1.
struct AuxSet { cudaStream_t s; cudaEvent_t fork, join, fin; };
static std::mutex g_aux_mu;
static std::vector<AuxSet> g_aux_free[64];

static bool aux_take(int dev, AuxSet &a) {
    {
        std::lock_guard<std::mutex> lock(g_aux_mu);
        auto &v = g_aux_free[dev & 63];
        if (!v.empty()) {
            a = v.back();
            v.pop_back();
            return true;
        }
    }
    a = AuxSet{nullptr, nullptr, nullptr, nullptr};
    if (cudaStreamCreateWithFlags(&a.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&a.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&a.join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&a.fin, cudaEventDisableTiming) != cudaSuccess)
        return false;
    return true;
}
static void aux_give(int dev, const AuxSet &a) {
    std::lock_guard<std::mutex> lock(g_aux_mu);
    g_aux_free[dev & 63].push_back(a);
}

int dftb_plan_destroy(dftb_plan *p) {
    if (!p) return 0;
    // the free is ordered after this plan's last submitted work (fin) on the aux stream, not
    // after whatever the caller's stream holds by now (the pipeline queues the next batch there)
    if (p->aux && p->fin) {
        // nothing recorded yet, or a call that failed partway: everything on its stream so far
        // (NULL = the legacy stream is a valid record target)
        if (!p->fin_rec || p->dirty) cudaEventRecord(p->fin, p->dirty ? p->last : p->stream);
        cudaStreamWaitEvent(p->aux, p->fin, 0);
    }
    if (p->mem) cudaFreeAsync(p->mem, p->aux ? p->aux : p->stream);   // back to the retained pool
    if (p->aux) cudaStreamSynchronize(p->aux);
    for (auto &e : p->ev)
        if (e) cudaEventDestroy(e);
    if (p->aux && p->fork && p->join && p->fin) aux_give(p->device, AuxSet{p->aux, p->fork, p->join, p->fin});
    delete p;
    return 0;
}

#ifndef PLAN_THREADS
#define PLAN_THREADS 4   // host threads for the per-molecule pair planning
#endif

// QM1B_TRACE=1: host-time trace of plan creation phases (stderr)
static double trace_ms() {
    static const bool on = std::getenv("QM1B_TRACE") != nullptr;
    if (!on) return -1.0;
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
#define TRACE(label, t0) do { const double t_ = trace_ms(); if (t_ >= 0) { std::fprintf(stderr, "[qm1b] %s %.2f ms\n", label, t_ - (t0)); (t0) = t_; } } while (0)

int dftb_plan_create(const dftb_batch_in *in, const dftb_opts *opts, void *stream, dftb_plan **out) {
    double tr = trace_ms();
    if (!in || !opts || !out) return fail(DFTB_EINVAL, "null argument");
    if (opts->max_iterations < 1) return fail(DFTB_EINVAL, "max_iterations must be >= 1");
    if (opts->diis_history < 1 || opts->diis_history > DIIS_MAX) return fail(DFTB_EINVAL, "diis_history must be in 1..64");
    cudaStream_t st = (cudaStream_t)stream;
    const int nm = in->n_mol;
    if (nm <= 0) return fail(DFTB_EINVAL, "empty batch");
    dftb_plan *p = new dftb_plan();
    p->opts = *opts;
    cudaGetDevice(&p->device);
    // ---------------- host-side planning
    std::vector<int> atom0(nm + 1, 0), shell0(nm + 1, 0), pair0(nm + 1, 0), npl(3 * nm, 0);
    std::vector<int> s_ao(in->n_shell), s_atom_g(in->n_shell), p_sa, p_sb;
    p->nao.resize(nm);
    p->nocc.assign(in->mol_nocc, in->mol_nocc + nm);
    for (int m = 0; m < nm; ++m) {
        atom0[m + 1] = atom0[m] + in->mol_natom[m];
        shell0[m + 1] = shell0[m] + in->mol_nshell[m];
        p->natom_max = std::max(p->natom_max, in->mol_natom[m]);
        p->nsh_max = std::max(p->nsh_max, in->mol_nshell[m]);
    }
    if (atom0[nm] != in->n_atom || shell0[nm] != in->n_shell) {
        delete p;
        return fail(DFTB_EINVAL, "atom/shell counts do not add up");
    }
    if (p->natom_max > 96) { delete p; return fail(DFTB_ERESOURCE, "more than 96 atoms in a molecule"); }
    if (in->n_tmpl < 0 || (in->n_tmpl > 0 && (!in->tmpl_xyzw || !in->atom_tmpl0 || !in->atom_tmpln))) {
        delete p;
        return fail(DFTB_EINVAL, "grid templates: bad count or null arrays");
    }
    if (in->n_tmpl > 0)
        for (int a = 0; a < in->n_atom; ++a) {
            const int64_t t0 = in->atom_tmpl0[a], tn = in->atom_tmpln[a];
            if (t0 < 0 || tn < 0 || t0 + tn > in->n_tmpl) {   // k_grid reads tmpl[t0 .. t0 + tn)
                delete p;
                return fail(DFTB_EINVAL, "atom grid template range outside [0, n_tmpl)");
            }
        }
    std::vector<double> emin(in->n_shell);
    for (int s = 0; s < in->n_shell; ++s)
        emin[s] = std::min(in->shell_exp[3 * s], std::min(in->shell_exp[3 * s + 1], in->shell_exp[3 * s + 2]));
    for (int m = 0; m < nm; ++m) {
        int n = 0, nl = 0;
        const int s0 = shell0[m], ns = in->mol_nshell[m];
        for (int s = s0; s < s0 + ns; ++s) {
            s_ao[s] = n;
            n += in->shell_kind[s] ? 4 : 1;
            nl += in->shell_kind[s] ? 1 : 0;
            const int la = in->shell_atom[s];
            if (la < 0 || la >= in->mol_natom[m]) { delete p; return fail(DFTB_EINVAL, "shell_atom out of range"); }
            s_atom_g[s] = atom0[m] + la;
        }
        if (n > NMAX) { delete p; return fail(DFTB_ERESOURCE, "N_ao exceeds the device maximum (96)"); }
        if (in->mol_nocc[m] > n) { delete p; return fail(DFTB_EINVAL, "more occupied orbitals than basis functions"); }
        p->nao[m] = n;
        p->nmax = std::max(p->nmax, n);
        const int nsg = ns - nl;   // class sizes: 0 LL, 1 LS (L first), 2 SS
        npl[3 * m] = nl * (nl + 1) / 2;
        npl[3 * m + 1] = nl * nsg;
        npl[3 * m + 2] = nsg * (nsg + 1) / 2;
        pair0[m + 1] = pair0[m] + npl[3 * m] + npl[3 * m + 1] + npl[3 * m + 2];
    }
    p_sa.resize((size_t)pair0[nm]);
    p_sb.resize((size_t)pair0[nm]);
    // class lists of every molecule, each ordered by how slowly the pair's overlap decays:
    // key mu_min R^2 with mu_min the smallest alpha beta / (alpha + beta) of its primitive
    // pairs (= that of the two smallest exponents: the expression increases in both), a
    // geometric stand-in for the Schwarz bound.  The ERI kernels run 32 consecutive kets per
    // warp; kets of similar extent share their primitive screens and Schwarz outcome.  Ties
    // by list position, so the order is deterministic.  Molecules are independent: a few
    // host threads share them (the sorts took 7 ms per 256-molecule batch on one core).
    auto fill = [&](int m_begin, int m_end) {
        struct PairKey { double key; int x, y, pos; };
        std::vector<PairKey> cls_pairs[3];
        for (int m = m_begin; m < m_end; ++m) {
            const int s0 = shell0[m], ns = in->mol_nshell[m];
            for (int c = 0; c < 3; ++c) cls_pairs[c].clear();
            for (int a = s0; a < s0 + ns; ++a)
                for (int b2 = s0; b2 <= a; ++b2) {
                    const int ka = in->shell_kind[a], kb = in->shell_kind[b2];
                    const int c = (ka && kb) ? 0 : (ka || kb) ? 1 : 2;
                    int x = a, y = b2;
                    if (ka < kb) std::swap(x, y);
                    const double *A = in->atom_xyz + 3 * (size_t)(atom0[m] + in->shell_atom[x]);
                    const double *B = in->atom_xyz + 3 * (size_t)(atom0[m] + in->shell_atom[y]);
                    const double r2 = (A[0] - B[0]) * (A[0] - B[0]) + (A[1] - B[1]) * (A[1] - B[1]) +
                                      (A[2] - B[2]) * (A[2] - B[2]);
                    const double al = emin[x], be = emin[y];
                    cls_pairs[c].push_back({al * be / (al + be) * r2, x, y, (int)cls_pairs[c].size()});
                }
            int o = pair0[m];
            for (int cls = 0; cls < 3; ++cls) {
                auto &v = cls_pairs[cls];
#ifndef PAIR_SORT
#define PAIR_SORT 1
#endif
                if (PAIR_SORT && v.size() > 1)
                    std::sort(v.begin(), v.end(), [](const PairKey &u, const PairKey &w) {
                        return u.key < w.key || (u.key == w.key && u.pos < w.pos);
                    });
                for (const PairKey &k : v) { p_sa[o] = k.x; p_sb[o] = k.y; ++o; }
            }
        }
    };
    {
        const int nth = std::max(1, std::min(PLAN_THREADS, nm / 16));
        std::vector<std::thread> th;
        for (int t = 1; t < nth; ++t) th.emplace_back(fill, (int)((int64_t)nm * t / nth), (int)((int64_t)nm * (t + 1) / nth));
        fill(0, nm / nth);
        for (auto &x : th) x.join();
    }
    const int npair = pair0[nm];
    TRACE("plan:pairs", tr);
    // quartet-class prefixes (6 classes) + Schwarz pair-class prefixes (3)
    std::vector<int64_t> cls0((NCLS + 3) * (size_t)(nm + 1), 0);
    for (int m = 0; m < nm; ++m) {
        const int64_t L = npl[3 * m], X = npl[3 * m + 1], S = npl[3 * m + 2];
        const int64_t q[NCLS + 3] = {L * (L + 1) / 2, L * X, L * S, X * (X + 1) / 2, X * S, S * (S + 1) / 2, L, X, S};
        for (int c = 0; c < NCLS + 3; ++c) cls0[c * (nm + 1) + m + 1] = cls0[c * (nm + 1) + m] + q[c];
    }
    for (int c = 0; c < NCLS; ++c) p->cls_tot[c] = cls0[c * (nm + 1) + nm];
    for (int c = 0; c < 3; ++c) p->pair_tot[c] = cls0[(NCLS + c) * (nm + 1) + nm];
    // matrices, ERI store, partials, grid
    p->mat0.assign(nm + 1, 0);
    p->npp0.assign(nm + 1, 0);
    p->grid0.assign(nm + 1, 0);
    std::vector<int64_t> eri0(nm + 1, 0), G0(nm + 1, 0), Jp0(nm + 1, 0), V0(nm + 1, 0);
    std::vector<int64_t> a_grid0(in->n_atom + 1, 0);
    for (int a = 0; a < in->n_atom; ++a) a_grid0[a + 1] = a_grid0[a] + (in->n_tmpl ? in->atom_tmpln[a] : 0);
    p->jkc0.assign(nm + 1, 0);
    p->xcc0.assign(nm + 1, 0);
    std::vector<int> jk_mol, jk_i0, jk_i1, xc_mol;
    std::vector<int64_t> xc_p0, xc_p1;
    int xc_main_bucket = 0;
    {
        int cnt[6] = {0};
        for (int m = 0; m < nm; ++m) ++cnt[std::min(5, std::max(0, (p->nao[m] + 15) / 16 - 1))];
        for (int k = 1; k < 6; ++k)
            if (cnt[k] > cnt[xc_main_bucket]) xc_main_bucket = k;
    }
    for (int m = 0; m < nm; ++m) {
        const int64_t N = p->nao[m], npp = N * (N + 1) / 2;
        p->mat0[m + 1] = p->mat0[m] + N * N;
        p->npp0[m + 1] = p->npp0[m] + npp;
        eri0[m + 1] = eri0[m] + eri_size((int)N);
        // J/K CTAs: contiguous whole-slab ranges [i0, i1) of about equal tile-row work
        // (slab i = the i + 1 store rows (i, j); its work is (i + 1) * tri(i/4 + 1) tiles)
        int ncj = 0;
        {
            std::vector<int64_t> wk((size_t)N);
            int64_t tot = 0, wmax = 0;
            for (int i = 0; i < N; ++i) {
                const int64_t A = i / 4 + 1;
                wk[i] = (int64_t)(i + 1) * (A * (A + 1) / 2);
                tot += wk[i];
                wmax = std::max(wmax, wk[i]);
            }
            int js = jk_split(nm, opts->precision && !ERI64_F32);
            // f32 store: J_Q is summed in f32 over a CTA's rows - keep that to ~600 rows per CTA on
            // average for the larger molecules as well (N = 92: 8 CTAs)
            if (opts->precision && !ERI64_F32) js = std::max(js, (int)((npp + 599) / 600));
            const int64_t target = std::max(wmax, (tot + js - 1) / js);
            int hi = (int)N;
            int64_t acc = 0;
            for (int i = (int)N - 1; i >= 0; --i) {
                if (acc > 0 && acc + wk[i] > target) {
                    jk_mol.push_back(m); jk_i0.push_back(i + 1); jk_i1.push_back(hi); ++ncj;
                    hi = i + 1;
                    acc = 0;
                }
                acc += wk[i];
            }
            jk_mol.push_back(m); jk_i0.push_back(0); jk_i1.push_back(hi); ++ncj;
        }
        p->jkc0[m + 1] = p->jkc0[m] + ncj;
        G0[m + 1] = G0[m] + (int64_t)ncj * N * N;      // one N x N exchange partial per J/K CTA
        Jp0[m + 1] = Jp0[m] + (int64_t)(ncj + 1) * npp;
        p->grid0[m] = a_grid0[atom0[m]];
        const int64_t g_end = a_grid0[atom0[m + 1]];
        const int64_t npts = g_end - p->grid0[m];
        // points per XC CTA: the most populated AO-count bucket uses XC_CHUNK; minority
        // buckets (a few large molecules) use XC_CHUNK / 4 so their CTAs do not form a
        // long tail behind the main launch
        const int chunk = ((N + 15) / 16 - 1) == xc_main_bucket ? XC_CHUNK : XC_CHUNK / 4;
        const int ncx = (int)((npts + chunk - 1) / chunk);
        for (int c = 0; c < ncx; ++c) {
            xc_mol.push_back(m);
            xc_p0.push_back(p->grid0[m] + (int64_t)c * chunk);
            xc_p1.push_back(std::min(g_end, p->grid0[m] + (int64_t)(c + 1) * chunk));
        }
        p->xcc0[m + 1] = p->xcc0[m] + ncx;
        V0[m + 1] = V0[m] + (int64_t)ncx * N * N;
    }
    p->grid0[nm] = a_grid0[in->n_atom];
    TRACE("plan:ctas", tr);
    // XC CTAs grouped by AO-count bucket (NQ = 4 * ceil(N / 16))
    std::vector<int> xc_sorted;
    for (int bkt = 0; bkt < 6; ++bkt) {
        for (int c = 0; c < (int)xc_mol.size(); ++c)
            if ((p->nao[xc_mol[c]] + 15) / 16 - 1 == bkt) xc_sorted.push_back(c);
        p->xc_bucket_n[bkt] = (int)xc_sorted.size() - (bkt ? 0 : 0);
    }
    for (int bkt = 5; bkt > 0; --bkt) p->xc_bucket_n[bkt] -= p->xc_bucket_n[bkt - 1];
    // J/K CTAs grouped the same way (one kernel instance per AO-count bucket)
    std::vector<int> jk_sorted;
    for (int bkt = 0; bkt < 6; ++bkt) {
        const size_t before = jk_sorted.size();
        for (int c = 0; c < (int)jk_mol.size(); ++c)
            if ((p->nao[jk_mol[c]] + 15) / 16 - 1 == bkt) jk_sorted.push_back(c);
        p->jk_bucket_n[bkt] = (int)(jk_sorted.size() - before);
    }
    p->eri0 = eri0;
    // largest molecules first: the per-molecule SCF kernels run ~2 waves of one CTA per SM,
    // so longest-first keeps the second wave from ending on a large molecule
    std::vector<int> mol_order(nm);
    for (int m = 0; m < nm; ++m) mol_order[m] = m;
    std::stable_sort(mol_order.begin(), mol_order.end(), [&](int a, int c) { return p->nao[a] > p->nao[c]; });
    // J/K CTAs: largest work first within each bucket
    {
        std::vector<int64_t> work(jk_mol.size(), 0);
        for (size_t c = 0; c < jk_mol.size(); ++c)
            for (int i = jk_i0[c]; i < jk_i1[c]; ++i) {
                const int64_t A = i / 4 + 1;
                work[c] += (int64_t)(i + 1) * (A * (A + 1) / 2);
            }
        int off = 0;
        for (int bkt = 0; bkt < 6; ++bkt) {
            std::stable_sort(jk_sorted.begin() + off, jk_sorted.begin() + off + p->jk_bucket_n[bkt],
                             [&](int a, int c) { return work[a] > work[c]; });
            off += p->jk_bucket_n[bkt];
        }
    }
    TRACE("plan:sort", tr);
    const int64_t npts_tot = a_grid0[in->n_atom];
    const int njk = (int)jk_mol.size(), nxc = (int)xc_mol.size();
    const int64_t mat = p->mat0[nm];
    const int maxit = opts->max_iterations;

    // ---------------- layout
    Lay L;
    struct Up { size_t off; const void *src; size_t bytes; };
    std::vector<Up> ups;
    auto up = [&](size_t off, const void *src, size_t bytes) { ups.push_back({off, src, bytes}); };
    std::vector<int> m_atom0(atom0), m_shell0(shell0), m_pair0(pair0);
    std::vector<int> jkc0v(p->jkc0), xcc0v(p->xcc0);
    std::vector<int64_t> mat0v(p->mat0), npp0v(p->npp0), grid0v(p->grid0);
#define UP(field, T, vec, n)                       \
    size_t o_##field = L.add<T>(n);                \
    up(o_##field, (vec), sizeof(T) * (size_t)(n));
    UP(m_nao, int, p->nao.data(), nm)
    UP(m_nocc, int, in->mol_nocc, nm)
    UP(m_natom, int, in->mol_natom, nm)
    UP(m_atom0, int, m_atom0.data(), nm + 1)
    UP(m_nshell, int, in->mol_nshell, nm)
    UP(m_shell0, int, m_shell0.data(), nm + 1)
    UP(m_pair0, int, m_pair0.data(), nm + 1)
    UP(m_npl, int, npl.data(), 3 * nm)
    UP(m_mat0, int64_t, mat0v.data(), nm + 1)
    UP(m_npp0, int64_t, npp0v.data(), nm + 1)
    UP(m_eri0, int64_t, eri0.data(), nm + 1)
    UP(m_grid0, int64_t, grid0v.data(), nm + 1)
    UP(m_jkcta0, int, jkc0v.data(), nm + 1)
    UP(m_xccta0, int, xcc0v.data(), nm + 1)
    UP(m_G0, int64_t, G0.data(), nm + 1)
    UP(m_Jp0, int64_t, Jp0.data(), nm + 1)
    UP(m_V0, int64_t, V0.data(), nm + 1)
    UP(cls0, int64_t, cls0.data(), cls0.size())
    UP(a_z, int, in->atom_z, in->n_atom)
    UP(a_xyz, double, in->atom_xyz, 3 * (size_t)in->n_atom)
    UP(a_grid0, int64_t, a_grid0.data(), in->n_atom + 1)
    std::vector<int> zeros_atom(in->n_atom, 0);
    UP(a_tmpl0, int, in->n_tmpl ? in->atom_tmpl0 : zeros_atom.data(), in->n_atom)
    UP(a_tmpln, int, in->n_tmpl ? in->atom_tmpln : zeros_atom.data(), in->n_atom)
    UP(tmpl, double, in->tmpl_xyzw, 4 * (size_t)in->n_tmpl)
    UP(s_kind, int, in->shell_kind, in->n_shell)
    UP(s_ao, int, s_ao.data(), in->n_shell)
    UP(s_atom, int, s_atom_g.data(), in->n_shell)
    UP(s_exp, double, in->shell_exp, 3 * (size_t)in->n_shell)
    UP(s_cs, double, in->shell_cs, 3 * (size_t)in->n_shell)
    UP(s_cp, double, in->shell_cp, 3 * (size_t)in->n_shell)
    UP(p_sa, int, p_sa.data(), npair)
    UP(p_sb, int, p_sb.data(), npair)
    UP(jk_mol, int, jk_mol.data(), njk)
    UP(jk_i0, int, jk_i0.data(), njk)
    UP(jk_i1, int, jk_i1.data(), njk)
    UP(jk_sorted, int, jk_sorted.data(), njk)
    UP(mol_order, int, mol_order.data(), nm)
    UP(xc_mol, int, xc_mol.data(), nxc)
    UP(xc_p0, int64_t, xc_p0.data(), nxc)
    UP(xc_p1, int64_t, xc_p1.data(), nxc)
    UP(xc_sorted, int, xc_sorted.data(), nxc)
#undef UP
    p->in_bytes = (L.off + 255) & ~(size_t)255;
    p->work_off = L.add<char>(0);
    const size_t o_p_geo = L.add<double>(6 * (size_t)npair);
    const size_t o_pp = L.add<double>((size_t)PP_FIELDS * NPP * npair);
    const size_t o_p_q = L.add<double>(npair);
    const size_t o_qao = L.add<double>(p->npp0[nm]);
    const size_t o_gxyz = L.add<double>(3 * (size_t)npts_tot);
    const size_t o_gw = L.add<double>(npts_tot);
    size_t o_mats[14];
    for (int k = 0; k < 13; ++k) o_mats[k] = L.add<double>(mat);
    o_mats[13] = L.add<double>(2 * (size_t)mat);                    // scratch: two matrices
    const size_t o_Fring = L.add<double>((size_t)opts->diis_history * mat);
    const size_t o_Ering = L.add<double>((size_t)opts->diis_history * mat);
    const size_t o_Gp = L.add<double>(G0[nm]);
    const size_t o_Jp = L.add<double>(Jp0[nm]);
    const size_t o_Vp = L.add<double>(V0[nm]);
    const size_t o_Ep = L.add<double>(std::max(nxc, 1));
    const size_t o_enn = L.add<double>(nm);
    const size_t o_hist = L.add<double>((size_t)nm * maxit);
    const size_t o_comp = L.add<double>(5 * (size_t)nm);
    const size_t o_Bmat = L.add<double>((size_t)nm * opts->diis_history * opts->diis_history);
    const size_t o_eps = L.add<double>((size_t)nm * NMAX);
    const size_t o_dbg = L.add<long long>((size_t)nm * 16);
    size_t o_ints[9];
    for (int k = 0; k < 9; ++k) o_ints[k] = L.add<int>(nm);
    const int eri64 = !opts->precision || ERI64_F32;
    const int esz = eri64 ? 8 : 4;
    p->eri_off = L.add<char>((size_t)eri0[nm] * esz);
    p->eri_bytes = (size_t)eri0[nm] * esz;
    p->mem_bytes = (L.off + 255) & ~(size_t)255;
    // ---------------- allocate + upload
    // stream-ordered allocation from the device's default pool, retained across plans so a
    // stream of batches does not pay cudaMalloc/cudaFree each time
    {
        static bool pool_set[64] = {false};
        static std::mutex pool_mu;
        std::lock_guard<std::mutex> pool_lock(pool_mu);
        if (!pool_set[p->device]) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, p->device) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
                // no reuse of a block freed on another stream by making this stream wait for
                // that stream's pending work (the free of a batch still running elsewhere):
                // concurrent plans take their own blocks (the pool keeps them all)
                int no = 0;
                cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
            }
            pool_set[p->device] = true;
        }
    }
    TRACE("plan", tr);
    p->stream = st;
    {
        AuxSet a;
        if (!aux_take(p->device, a)) {
            dftb_plan_destroy(p);
            return fail(DFTB_ECUDA, "stream/event creation failed");
        }
        p->aux = a.s; p->fork = a.fork; p->join = a.join; p->fin = a.fin;
    }
    TRACE("streams", tr);
    // allocation rounded up to 64 MiB so the pool's blocks are interchangeable between the
    // slightly different batch sizes that follow each other through the pipeline
    const size_t alloc_bytes = (p->mem_bytes + ((size_t)64 << 20) - 1) & ~(((size_t)64 << 20) - 1);
    // allocation and upload on the plan's own aux stream, synchronized here: on the caller's
    // stream they would queue behind that stream's previous batch, and the synchronization
    // below would block plan creation until it finished (the labeling pipeline creates the
    // next batch's plan while the current one runs on the same stream)
    cudaError_t ce = cudaMallocAsync((void **)&p->mem, alloc_bytes, p->aux);
    TRACE("malloc", tr);
    if (ce != cudaSuccess) {
        p->mem = nullptr;
        dftb_plan_destroy(p);
        return fail(DFTB_ERESOURCE, std::string("device allocation of ") + std::to_string(p->mem_bytes >> 20) +
                                        " MiB failed: " + cudaGetErrorString(ce));
    }
    std::vector<unsigned char> blob(p->in_bytes, 0);
    for (auto &u : ups)
        if (u.bytes) std::memcpy(blob.data() + u.off, u.src, u.bytes);
    ce = cudaMemcpyAsync(p->mem, blob.data(), p->in_bytes, cudaMemcpyHostToDevice, p->aux);
    TRACE("copy", tr);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(p->aux);  // blob is pageable and local
    TRACE("sync", tr);
    if (ce != cudaSuccess) {
        dftb_plan_destroy(p);
        return fail(DFTB_ECUDA, std::string("upload: ") + cudaGetErrorString(ce));
    }
    // ---------------- device view
    DevBatch &d = p->d;
    unsigned char *M = p->mem;
#define PTR(T, o) reinterpret_cast<T *>(M + (o))
    d.n_mol = nm; d.n_atom = in->n_atom; d.n_shell = in->n_shell; d.n_pair = npair; d.n_pts = (int)npts_tot;
    d.prec = opts->precision ? 1 : 0;
    d.eri64 = eri64;
    d.m_nao = PTR(int, o_m_nao); d.m_nocc = PTR(int, o_m_nocc); d.m_natom = PTR(int, o_m_natom);
    d.m_atom0 = PTR(int, o_m_atom0); d.m_nshell = PTR(int, o_m_nshell); d.m_shell0 = PTR(int, o_m_shell0);
    d.m_pair0 = PTR(int, o_m_pair0); d.m_npl = PTR(int, o_m_npl);
    d.m_mat0 = PTR(int64_t, o_m_mat0); d.m_npp0 = PTR(int64_t, o_m_npp0); d.m_eri0 = PTR(int64_t, o_m_eri0);
    d.m_grid0 = PTR(int64_t, o_m_grid0); d.m_jkcta0 = PTR(int, o_m_jkcta0); d.m_xccta0 = PTR(int, o_m_xccta0);
    d.m_G0 = PTR(int64_t, o_m_G0); d.m_Jp0 = PTR(int64_t, o_m_Jp0); d.m_V0 = PTR(int64_t, o_m_V0);
    d.cls0 = PTR(int64_t, o_cls0);
    d.a_z = PTR(int, o_a_z); d.a_xyz = PTR(double, o_a_xyz); d.a_grid0 = PTR(int64_t, o_a_grid0);
    d.a_tmpl0 = PTR(int, o_a_tmpl0); d.a_tmpln = PTR(int, o_a_tmpln); d.tmpl = PTR(double, o_tmpl);
    d.s_kind = PTR(int, o_s_kind); d.s_ao = PTR(int, o_s_ao); d.s_atom = PTR(int, o_s_atom);
    d.s_exp = PTR(double, o_s_exp); d.s_cs = PTR(double, o_s_cs); d.s_cp = PTR(double, o_s_cp);
    d.p_sa = PTR(int, o_p_sa); d.p_sb = PTR(int, o_p_sb);
    d.p_geo = PTR(double, o_p_geo); d.pp = PTR(double, o_pp); d.p_q = PTR(double, o_p_q); d.qao = PTR(double, o_qao);
    d.jk_mol = PTR(int, o_jk_mol); d.jk_i0 = PTR(int, o_jk_i0); d.jk_i1 = PTR(int, o_jk_i1); d.n_jk_cta = njk;
    d.xc_mol = PTR(int, o_xc_mol); d.xc_p0 = PTR(int64_t, o_xc_p0); d.xc_p1 = PTR(int64_t, o_xc_p1);
    d.n_xc_cta = nxc;
    p->xc_bucket_ctas = PTR(int, o_xc_sorted);
    p->jk_bucket_ctas = PTR(int, o_jk_sorted);
    d.mol_order = PTR(int, o_mol_order);
    d.g_xyz = PTR(double, o_gxyz); d.g_w = PTR(double, o_gw);
    double **mats[14] = {&d.S, &d.T, &d.V, &d.H, &d.X, &d.C, &d.Cp, &d.rho, &d.rho_prev, &d.F, &d.J, &d.K, &d.Vxc,
                         &d.scratch};
    for (int k = 0; k < 14; ++k) *mats[k] = PTR(double, o_mats[k]);
    d.Fring = PTR(double, o_Fring); d.Ering = PTR(double, o_Ering);
    d.eri = M + p->eri_off;
    d.Gpart = PTR(double, o_Gp); d.Jpart = PTR(double, o_Jp); d.Vpart = PTR(double, o_Vp); d.Epart = PTR(double, o_Ep);
    d.enn = PTR(double, o_enn); d.hist = PTR(double, o_hist); d.comp = PTR(double, o_comp);
    d.Bmat = PTR(double, o_Bmat); d.eps = PTR(double, o_eps);
    d.nmo = PTR(int, o_ints[0]); d.ring_n = PTR(int, o_ints[1]); d.ring_head = PTR(int, o_ints[2]);
    d.done = PTR(int, o_ints[3]); d.conv = PTR(int, o_ints[4]); d.iters = PTR(int, o_ints[5]);
    d.status = PTR(int, o_ints[6]);
    d.cpv = PTR(int, o_ints[7]);
    d.puri = PTR(int, o_ints[8]);
#ifdef FORCE_FULL_EIG
    d.full_eig = 1;
#else
    d.full_eig = 0;
#endif
    d.max_it = maxit;
    d.dbg = PTR(long long, o_dbg);
#undef PTR
    ce = cudaMemsetAsync(p->mem + p->work_off, 0, p->mem_bytes - p->work_off, st);
    if (ce != cudaSuccess) {
        dftb_plan_destroy(p);
        return fail(DFTB_ECUDA, std::string("memset: ") + cudaGetErrorString(ce));
    }
    const double *boys = nullptr;
    int rc = ensure_boys(p->device, &boys);
    if (rc) { dftb_plan_destroy(p); return rc; }
    d.boys = boys;
    *out = p;
    return 0;
}

static int zero_work(dftb_plan *p, cudaStream_t st) {
    CK(cudaMemsetAsync(p->mem + p->work_off, 0, p->mem_bytes - p->work_off, st));
    CK(cudaMemsetAsync(p->d.hist, 0xFF, sizeof(double) * (size_t)p->d.n_mol * p->d.max_it, st));
    return 0;
}

static void mark(dftb_plan *p, int k, cudaStream_t st) {
    if (p->timing) cudaEventRecord(p->ev[k], st);
}

static int setup_stage(dftb_plan *p, cudaStream_t st, bool screened) {
    const DevBatch &d = p->d;
    int nl = 0;
    launch_pairs(d, st);
    launch_schwarz(d, p->pair_tot, st);
    const double eps = screened ? p->opts.screen_eps : 0.0;
    launch_eri(d, p->cls_tot, eps, 1e-3 * eps, st, &nl);
    p->launches += 2 + 3 + 1 + nl;
    CK(cudaGetLastError());
    return 0;
}

int dftb_plan_set_full_eig(dftb_plan *p, int enable) {
    if (!p) return fail(DFTB_EINVAL, "null plan");
    p->d.full_eig = enable != 0;
    return 0;
}

int dftb_plan_set_timing(dftb_plan *p, int enable) {
    if (!p) return fail(DFTB_EINVAL, "null plan");
    p->timing = enable != 0;
    if (p->timing && !p->ev[0])
        for (auto &e : p->ev) CK(cudaEventCreate(&e));
    return 0;
}

// fork: aux waits for everything issued on st so far; join: st waits for aux
static cudaError_t fork(dftb_plan *p, cudaStream_t st) {
    cudaError_t e = cudaEventRecord(p->fork, st);
    return e != cudaSuccess ? e : cudaStreamWaitEvent(p->aux, p->fork, 0);
}
static cudaError_t join(dftb_plan *p, cudaStream_t st) {
    cudaError_t e = cudaEventRecord(p->join, p->aux);
    return e != cudaSuccess ? e : cudaStreamWaitEvent(st, p->join, 0);
}

int dftb_plan_begin(dftb_plan *p, void *stream) {
    if (!p) return fail(DFTB_EINVAL, "null plan");
    cudaStream_t st = (cudaStream_t)stream;
    enq_begin(p, st);
    const DevBatch &d = p->d;
    p->launches = 0;
    enq_begin(p, st);
    int rc = zero_work(p, st);
    if (rc) return rc;
    mark(p, 0, st);
    // the one-electron integrals, grid, orthogonaliser and core guess do not depend on the
    // ERI stage: they run on the aux stream while the pair tables, Schwarz bounds and ERIs
    // run on the caller's stream (stage 1 = ERI stage, stage 2 = the wait for the rest)
    CK(fork(p, st));
    launch_onee(d, p->aux);
    launch_enn(d, p->aux);
    launch_grid(d, p->natom_max, p->aux);
    launch_orth(d, p->nmax, p->aux);
    const dftb_opts &o = p->opts;
    launch_post(d, p->nmax, -1, o.diis_start, o.diis_history, o.damping_factor, o.convergence_std, p->aux);
    p->launches += 5;
    rc = setup_stage(p, st, true);
    if (rc) return rc;
    mark(p, 1, st);
    CK(join(p, st));
    CK(cudaGetLastError());
    mark(p, 2, st);
    enq_end(p, st);
    enq_end(p, st);
    return 0;
}

int dftb_plan_iterate(dftb_plan *p, int32_t it, void *stream) {
    if (!p || it < 0 || it >= p->opts.max_iterations) return fail(DFTB_EINVAL, "bad iteration index");
    cudaStream_t st = (cudaStream_t)stream;
    const DevBatch &d = p->d;
    const dftb_opts &o = p->opts;
    enq_begin(p, st);
    // J/K (aux stream) and XC (caller's stream) both read rho and write separate partials:
    // fork/join so their CTAs share the SMs (FP64/XU-heavy vs FP32-heavy, smem fits both)
    CK(fork(p, st));
    const int njl = launch_jk(d, p->jk_bucket_ctas, p->jk_bucket_n, p->aux);
    const int nxl = launch_xc(d, p->xc_bucket_ctas, p->xc_bucket_n, p->nsh_max, st);
    CK(join(p, st));
    launch_post(d, p->nmax, it, o.diis_start, o.diis_history, o.damping_factor, o.convergence_std, st);
    p->launches += 1 + njl + nxl;
    CK(cudaGetLastError());
    enq_end(p, st);
    return 0;
}

int dftb_plan_run(dftb_plan *p, void *stream) {
    int rc = dftb_plan_begin(p, stream);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const DevBatch &d = p->d;
    const dftb_opts &o = p->opts;
    std::vector<int> done(d.n_mol);
    for (int it = 0; it < o.max_iterations; ++it) {
        rc = dftb_plan_iterate(p, it, stream);
        if (rc) return rc;
        if (o.convergence_std > 0.0 && it >= 4 && (it % 4 == 0)) {
            // convergence mode only: one small readback every 4 iterations to stop early
            CK(cudaMemcpyAsync(done.data(), d.done, sizeof(int) * d.n_mol, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            bool all = true;
            for (int v : done) all = all && v;
            if (all) break;
        }
    }
    mark(p, 3, st);
    enq_end(p, st);
    return 0;
}

// Scatter a canonical packed list (composite order not required) into the dense store
// of molecule `mol` (store zeroed first).  Used by build_jk on arbitrary PackedERI input.
int dftb_plan_eri_load(dftb_plan *p, int32_t mol, int64_t count, const uint16_t *i, const uint16_t *j,
                       const uint16_t *k, const uint16_t *l, const double *v, void *stream) {
    if (!p || mol < 0 || mol >= p->d.n_mol) return fail(DFTB_EINVAL, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    enq_begin(p, st);
    const int64_t npp = p->npp0[mol + 1] - p->npp0[mol];
    const int esz = p->d.eri64 ? 8 : 4;
    const int N = p->nao[mol];
    const int64_t n = eri_size(N);
    const int64_t e0 = p->eri0[mol];
    std::vector<unsigned char> host((size_t)n * esz, 0);
    for (int64_t e = 0; e < count; ++e) {
        if (i[e] >= N || j[e] >= N || k[e] >= N || l[e] >= N) return fail(DFTB_EINVAL, "index out of range for n_ao");
        const int64_t off = eri_pos(i[e], j[e], k[e], l[e]);
        if (esz == 8) reinterpret_cast<double *>(host.data())[off] = p->d.prec ? (double)(float)v[e] : v[e];
        else reinterpret_cast<float *>(host.data())[off] = (float)v[e];
    }
    CK(cudaMemcpyAsync(p->mem + p->eri_off + (size_t)e0 * esz, host.data(), host.size(), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    enq_end(p, st);
    return 0;
}

int dftb_plan_load_grid(dftb_plan *p, const double *pts, const double *w, int64_t n, void *stream) {
    if (!p || n != p->d.n_pts) return fail(DFTB_EINVAL, "grid size does not match the plan");
    cudaStream_t st = (cudaStream_t)stream;
    enq_begin(p, st);
    CK(cudaMemcpyAsync(p->d.g_xyz, pts, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(p->d.g_w, w, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    enq_end(p, st);
    return 0;
}

int dftb_plan_stage_times(const dftb_plan *p, double *ms, int n) {
    if (!p || !p->timing) return fail(DFTB_EINVAL, "timing not enabled");
    cudaEventSynchronize(p->ev[3]);
    for (int k = 0; k < n && k < 3; ++k) {
        float t = 0.f;
        cudaEventElapsedTime(&t, p->ev[k], p->ev[k + 1]);
        ms[k] = t;
    }
    return 0;
}

int dftb_plan_launch_count(const dftb_plan *p, int64_t *count) {
    if (!p) return fail(DFTB_EINVAL, "null plan");
    *count = p->launches;
    return 0;
}

int dftb_plan_info(const dftb_plan *p, int64_t *info, int n) {
    if (!p) return fail(DFTB_EINVAL, "null plan");
    int64_t v[20] = {p->d.n_mol, p->d.n_pair, p->d.n_pts, (int64_t)p->mem_bytes, (int64_t)p->eri_bytes,
                     p->cls_tot[0], p->cls_tot[1], p->cls_tot[2], p->cls_tot[3], p->cls_tot[4], p->cls_tot[5],
                     p->d.n_jk_cta, p->d.n_xc_cta, p->nmax, p->mat0[p->d.n_mol], p->launches,
                     (int64_t)p->in_bytes, p->pair_tot[0], p->pair_tot[1], p->pair_tot[2]};
    for (int k = 0; k < n && k < 20; ++k) info[k] = v[k];
    return 0;
}

int dftb_plan_fetch(dftb_plan *p, dftb_results *r, void *stream) {
    if (!p || !r) return fail(DFTB_EINVAL, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    const DevBatch &d = p->d;
    const int nm = d.n_mol, mi = d.max_it;
    std::vector<double> hist((size_t)nm * mi);
    std::vector<int> it(nm);
    // after dftb_plan_run: copy on the aux stream once this plan's work is done, so the wait
    // does not include later work the caller already queued on its stream
    if (p->fin_rec && p->aux) {
        CK(cudaStreamWaitEvent(p->aux, p->fin, 0));
        st = p->aux;
    }
    CK(cudaMemcpyAsync(hist.data(), d.hist, sizeof(double) * hist.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(it.data(), d.iters, sizeof(int) * nm, cudaMemcpyDeviceToHost, st));
    if (r->E_comp) CK(cudaMemcpyAsync(r->E_comp, d.comp, sizeof(double) * 5 * nm, cudaMemcpyDeviceToHost, st));
    if (r->converged) CK(cudaMemcpyAsync(r->converged, d.conv, sizeof(int) * nm, cudaMemcpyDeviceToHost, st));
    if (r->n_mo) CK(cudaMemcpyAsync(r->n_mo, d.nmo, sizeof(int) * nm, cudaMemcpyDeviceToHost, st));
    if (r->epsilon) CK(cudaMemcpyAsync(r->epsilon, d.eps, sizeof(double) * NMAX * nm, cudaMemcpyDeviceToHost, st));
    if (r->C) CK(cudaMemcpyAsync(r->C, d.C, sizeof(double) * p->mat0[nm], cudaMemcpyDeviceToHost, st));
    if (r->status) CK(cudaMemcpyAsync(r->status, d.status, sizeof(int) * nm, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (r->history) std::memcpy(r->history, hist.data(), sizeof(double) * hist.size());
    if (r->iterations) std::memcpy(r->iterations, it.data(), sizeof(int) * nm);
    if (r->E_total)
        for (int m = 0; m < nm; ++m) r->E_total[m] = it[m] > 0 ? hist[(size_t)m * mi + it[m] - 1] : NAN;
    return 0;
}

int dftb_plan_fetch_device(dftb_plan *p, const dftb_results_dev *r, void *stream) {
    if (!p || !r) return fail(DFTB_EINVAL, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    const DevBatch &d = p->d;
    const int nm = d.n_mol;
    if (p->fin_rec) CK(cudaStreamWaitEvent(st, p->fin, 0));   // this plan's queued work first
    const cudaMemcpyKind k = cudaMemcpyDeviceToDevice;
    if (r->E_total || r->history) launch_fetch_dev(d, r->E_total, r->history, st);
    if (r->iterations) CK(cudaMemcpyAsync(r->iterations, d.iters, sizeof(int) * nm, k, st));
    if (r->E_comp) CK(cudaMemcpyAsync(r->E_comp, d.comp, sizeof(double) * 5 * nm, k, st));
    if (r->converged) CK(cudaMemcpyAsync(r->converged, d.conv, sizeof(int) * nm, k, st));
    if (r->n_mo) CK(cudaMemcpyAsync(r->n_mo, d.nmo, sizeof(int) * nm, k, st));
    if (r->epsilon) CK(cudaMemcpyAsync(r->epsilon, d.eps, sizeof(double) * NMAX * nm, k, st));
    if (r->C) CK(cudaMemcpyAsync(r->C, d.C, sizeof(double) * p->mat0[nm], k, st));
    if (r->status) CK(cudaMemcpyAsync(r->status, d.status, sizeof(int) * nm, k, st));
    CK(cudaGetLastError());
    // the plan's stream-ordered free must also wait for these reads
    enq_begin(p, st);
    enq_end(p, st);
    return 0;
}

int dftb_scf_batch(const dftb_batch_in *in, const dftb_opts *opts, dftb_results *out, void *stream) {
    dftb_plan *p = nullptr;
    int rc = dftb_plan_create(in, opts, stream, &p);
    if (rc) return rc;
    rc = dftb_plan_run(p, stream);
    if (!rc) rc = dftb_plan_fetch(p, out, stream);
    dftb_plan_destroy(p);
    return rc;
}

// ------------------------------------------------------------------ operator-level stages
int dftb_plan_one_electron(dftb_plan *p, void *stream) {
    if (!p) return fail(DFTB_EINVAL, "null plan");
    cudaStream_t st = (cudaStream_t)stream;
    enq_begin(p, st);
    int rc = zero_work(p, st);
    if (rc) return rc;
    launch_pairs(p->d, st);
    launch_onee(p->d, st);
    launch_enn(p->d, st);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    enq_end(p, st);
    return 0;
}

int dftb_plan_eri(dftb_plan *p, int screened, void *stream) {
    if (!p) return fail(DFTB_EINVAL, "null plan");
    cudaStream_t st = (cudaStream_t)stream;
    enq_begin(p, st);
    int rc = zero_work(p, st);
    if (rc) return rc;
    rc = setup_stage(p, st, screened != 0);
    if (rc) return rc;
    CK(cudaStreamSynchronize(st));
    enq_end(p, st);
    return 0;
}

int dftb_plan_grid(dftb_plan *p, void *stream) {
    if (!p) return fail(DFTB_EINVAL, "null plan");
    cudaStream_t st = (cudaStream_t)stream;
    enq_begin(p, st);
    launch_grid(p->d, p->natom_max, st);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    enq_end(p, st);
    return 0;
}

static int upload_rho(dftb_plan *p, const double *rho_host, cudaStream_t st) {
    CK(cudaMemcpyAsync(p->d.rho, rho_host, sizeof(double) * p->mat0[p->d.n_mol], cudaMemcpyHostToDevice, st));
    return 0;
}

// requires dftb_plan_eri first (dense store present)
int dftb_plan_jk(dftb_plan *p, const double *rho_host, double *J_host, double *K_host, void *stream) {
    if (!p) return fail(DFTB_EINVAL, "null plan");
    cudaStream_t st = (cudaStream_t)stream;
    enq_begin(p, st);
    int rc = upload_rho(p, rho_host, st);
    if (rc) return rc;
    launch_jk(p->d, p->jk_bucket_ctas, p->jk_bucket_n, st);
    launch_reduce(p->d, 1, st);
    CK(cudaGetLastError());
    const size_t nb = sizeof(double) * p->mat0[p->d.n_mol];
    if (J_host) CK(cudaMemcpyAsync(J_host, p->d.J, nb, cudaMemcpyDeviceToHost, st));
    if (K_host) CK(cudaMemcpyAsync(K_host, p->d.K, nb, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    enq_end(p, st);
    return 0;
}

// requires dftb_plan_grid first
int dftb_plan_xc(dftb_plan *p, const double *rho_host, double *Vxc_host, double *Exc_host, void *stream) {
    if (!p) return fail(DFTB_EINVAL, "null plan");
    cudaStream_t st = (cudaStream_t)stream;
    enq_begin(p, st);
    int rc = upload_rho(p, rho_host, st);
    if (rc) return rc;
    launch_xc(p->d, p->xc_bucket_ctas, p->xc_bucket_n, p->nsh_max, st);
    launch_reduce(p->d, 2, st);
    CK(cudaGetLastError());
    if (Vxc_host) CK(cudaMemcpyAsync(Vxc_host, p->d.Vxc, sizeof(double) * p->mat0[p->d.n_mol], cudaMemcpyDeviceToHost, st));
    if (Exc_host) {
        std::vector<double> comp(5 * (size_t)p->d.n_mol);
        CK(cudaMemcpyAsync(comp.data(), p->d.comp, sizeof(double) * comp.size(), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int m = 0; m < p->d.n_mol; ++m) Exc_host[m] = comp[5 * m + 4];
    }
    CK(cudaStreamSynchronize(st));
    int bad = 0;
    std::vector<int> status(p->d.n_mol);
    CK(cudaMemcpyAsync(status.data(), p->d.status, sizeof(int) * p->d.n_mol, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int s : status) bad |= s & DFTB_ST_XC_NONFINITE;
    if (bad) return fail(DFTB_ENUMERIC, "non-finite functional output (density underflow mishandled)");
    enq_end(p, st);
    return 0;
}

int dftb_plan_eval_ao(dftb_plan *p, int32_t mol, double *phi_host, double *grad_host, void *stream) {
    if (!p || mol < 0 || mol >= p->d.n_mol) return fail(DFTB_EINVAL, "bad molecule index");
    cudaStream_t st = (cudaStream_t)stream;
    enq_begin(p, st);
    const int64_t npts = p->grid0[mol + 1] - p->grid0[mol];
    const int N = p->nao[mol];
    double *buf = nullptr;
    CK(cudaMallocAsync((void **)&buf, sizeof(double) * 4 * npts * N, st));
    launch_eval_ao(p->d, mol, buf, st);
    CK(cudaGetLastError());
    if (phi_host) CK(cudaMemcpyAsync(phi_host, buf, sizeof(double) * npts * N, cudaMemcpyDeviceToHost, st));
    if (grad_host)
        CK(cudaMemcpyAsync(grad_host, buf + npts * N, sizeof(double) * 3 * npts * N, cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(buf, st));
    CK(cudaStreamSynchronize(st));
    enq_end(p, st);
    return 0;
}

int dftb_plan_roothaan(dftb_plan *p, const double *F_host, double *C_host, double *eps_host, int32_t *nmo_host,
                       void *stream) {
    if (!p) return fail(DFTB_EINVAL, "null plan");
    cudaStream_t st = (cudaStream_t)stream;
    enq_begin(p, st);
    // S must be present (dftb_plan_one_electron or dftb_plan_set "S"); X from S
    CK(cudaMemsetAsync(p->d.status, 0, sizeof(int) * p->d.n_mol, st));
    launch_orth(p->d, p->nmax, st);
    CK(cudaMemcpyAsync(p->d.F, F_host, sizeof(double) * p->mat0[p->d.n_mol], cudaMemcpyHostToDevice, st));
    launch_roothaan(p->d, p->nmax, st);
    CK(cudaGetLastError());
    if (C_host) CK(cudaMemcpyAsync(C_host, p->d.C, sizeof(double) * p->mat0[p->d.n_mol], cudaMemcpyDeviceToHost, st));
    if (eps_host) CK(cudaMemcpyAsync(eps_host, p->d.eps, sizeof(double) * NMAX * p->d.n_mol, cudaMemcpyDeviceToHost, st));
    if (nmo_host) CK(cudaMemcpyAsync(nmo_host, p->d.nmo, sizeof(int) * p->d.n_mol, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    enq_end(p, st);
    return 0;
}

int dftb_plan_eri_compact(dftb_plan *p, int32_t mol, double eps, const double *qsp_host, int64_t *count,
                          uint16_t *oi, uint16_t *oj, uint16_t *ok, uint16_t *ol, double *ov, void *stream) {
    if (!p || mol < 0 || mol >= p->d.n_mol || !count) return fail(DFTB_EINVAL, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    enq_begin(p, st);
    const int N = p->nao[mol];
    const int64_t npp = (int64_t)N * (N + 1) / 2;
    double *qsp = nullptr;
    int64_t *rc_ = nullptr;
    CK(cudaMallocAsync((void **)&qsp, sizeof(double) * npp, st));
    CK(cudaMallocAsync((void **)&rc_, sizeof(int64_t) * (npp + 1), st));
    CK(cudaMemcpyAsync(qsp, qsp_host, sizeof(double) * npp, cudaMemcpyHostToDevice, st));
    launch_compact_count(p->d, mol, eps, qsp, rc_, st);
    std::vector<int64_t> cnt(npp);
    CK(cudaMemcpyAsync(cnt.data(), rc_, sizeof(int64_t) * npp, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<int64_t> off(npp + 1, 0);
    for (int64_t r = 0; r < npp; ++r) off[r + 1] = off[r] + cnt[r];
    *count = off[npp];
    if (oi && oj && ok && ol && ov && off[npp] > 0) {
        const int64_t n = off[npp];
        uint16_t *di = nullptr;
        double *dv = nullptr;
        CK(cudaMallocAsync((void **)&di, sizeof(uint16_t) * 4 * n, st));
        CK(cudaMallocAsync((void **)&dv, sizeof(double) * n, st));
        CK(cudaMemcpyAsync(rc_, off.data(), sizeof(int64_t) * (npp + 1), cudaMemcpyHostToDevice, st));
        launch_compact_write(p->d, mol, eps, qsp, rc_, di, di + n, di + 2 * n, di + 3 * n, dv, st);
        CK(cudaMemcpyAsync(oi, di, sizeof(uint16_t) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(oj, di + n, sizeof(uint16_t) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(ok, di + 2 * n, sizeof(uint16_t) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(ol, di + 3 * n, sizeof(uint16_t) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(ov, dv, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaFreeAsync(di, st));
        CK(cudaFreeAsync(dv, st));
    }
    CK(cudaFreeAsync(qsp, st));
    CK(cudaFreeAsync(rc_, st));
    CK(cudaStreamSynchronize(st));
    enq_end(p, st);
    return 0;
}

int dftb_plan_get(dftb_plan *p, const char *which, int32_t mol, double *host, int64_t n, void *stream) {
    if (!p || !which || mol < 0 || mol >= p->d.n_mol) return fail(DFTB_EINVAL, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const DevBatch &d = p->d;
    const std::string w(which);
    const int64_t mo = p->mat0[mol], mn = p->mat0[mol + 1] - mo;
    const double *src = nullptr;
    int64_t cnt = 0;
    if (w == "S") { src = d.S + mo; cnt = mn; }
    else if (w == "T") { src = d.T + mo; cnt = mn; }
    else if (w == "V") { src = d.V + mo; cnt = mn; }
    else if (w == "H") { src = d.H + mo; cnt = mn; }
    else if (w == "X") { src = d.X + mo; cnt = mn; }
    else if (w == "F") { src = d.F + mo; cnt = mn; }
    else if (w == "J") { src = d.J + mo; cnt = mn; }
    else if (w == "K") { src = d.K + mo; cnt = mn; }
    else if (w == "Vxc") { src = d.Vxc + mo; cnt = mn; }
    else if (w == "rho") { src = d.rho + mo; cnt = mn; }
    else if (w == "C") { src = d.C + mo; cnt = mn; }
    else if (w == "qao") { src = d.qao + p->npp0[mol]; cnt = p->npp0[mol + 1] - p->npp0[mol]; }
    else if (w == "points") { src = d.g_xyz + 3 * p->grid0[mol]; cnt = 3 * (p->grid0[mol + 1] - p->grid0[mol]); }
    else if (w == "weights") { src = d.g_w + p->grid0[mol]; cnt = p->grid0[mol + 1] - p->grid0[mol]; }
    else if (w == "enn") { src = d.enn + mol; cnt = 1; }
    else if (w == "dbg") { src = (const double *)(d.dbg + 16 * mol); cnt = 16; }
    else if (w == "eri") {
        // returned unpadded, in canonical composite order (row P, Q <= P)
        const int64_t npp = p->npp0[mol + 1] - p->npp0[mol];
        const int esz = d.eri64 ? 8 : 4;
        const int N = p->nao[mol];
        cnt = npp * (npp + 1) / 2;
        if (n < cnt) return fail(DFTB_EINVAL, "host buffer too small");
        std::vector<unsigned char> tmp((size_t)eri_size(N) * esz);
        CK(cudaMemcpyAsync(tmp.data(), (unsigned char *)d.eri + (size_t)p->eri0[mol] * esz, tmp.size(),
                           cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        int64_t o = 0;
        for (int ii = 0; ii < N; ++ii)
            for (int jj = 0; jj <= ii; ++jj)
                for (int kk = 0; kk <= ii; ++kk)
                    for (int ll = 0; ll <= (kk == ii ? jj : kk); ++ll, ++o) {
                        const int64_t src = eri_row(ii, jj) + eri_ket(kk, ll);
                        host[o] = esz == 8 ? reinterpret_cast<double *>(tmp.data())[src]
                                           : (double)reinterpret_cast<float *>(tmp.data())[src];
                    }
        return 0;
    } else {
        return fail(DFTB_EINVAL, "unknown buffer " + w);
    }
    if (n < cnt) return fail(DFTB_EINVAL, "host buffer too small");
    CK(cudaMemcpyAsync(host, src, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return 0;
}

int dftb_plan_set(dftb_plan *p, const char *which, int32_t mol, const double *host, int64_t n, void *stream) {
    if (!p || !which || mol < 0 || mol >= p->d.n_mol) return fail(DFTB_EINVAL, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const std::string w(which);
    const int64_t mo = p->mat0[mol], mn = p->mat0[mol + 1] - mo;
    double *dst = nullptr;
    if (w == "S") dst = p->d.S + mo;
    else if (w == "F") dst = p->d.F + mo;
    else if (w == "rho") dst = p->d.rho + mo;
    else if (w == "H") dst = p->d.H + mo;
    else return fail(DFTB_EINVAL, "unknown buffer " + w);
    if (n != mn) return fail(DFTB_EINVAL, "size mismatch");
    CK(cudaMemcpyAsync(dst, host, sizeof(double) * mn, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    return 0;
}

int dftb_b3lyp(const double *n, const double *sigma, int64_t npts, double *exc, double *vrho, double *vsigma,
               void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (npts <= 0) return 0;
    double *buf = nullptr;
    CK(cudaMallocAsync((void **)&buf, sizeof(double) * 5 * npts, st));
    CK(cudaMemcpyAsync(buf, n, sizeof(double) * npts, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(buf + npts, sigma, sizeof(double) * npts, cudaMemcpyHostToDevice, st));
    launch_b3lyp(buf, buf + npts, npts, buf + 2 * npts, buf + 3 * npts, buf + 4 * npts, st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(exc, buf + 2 * npts, sizeof(double) * npts, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(vrho, buf + 3 * npts, sizeof(double) * npts, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(vsigma, buf + 4 * npts, sizeof(double) * npts, cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(buf, st));
    CK(cudaStreamSynchronize(st));
    for (int64_t k = 0; k < npts; ++k)
        if (!std::isfinite(exc[k]) || !std::isfinite(vrho[k]) || !std::isfinite(vsigma[k]))
            return fail(DFTB_ENUMERIC, "non-finite functional output (density underflow mishandled)");
    return 0;
}

int dftb_diis(const double *F, const double *E, int32_t m, int32_t n, double *out, void *stream) {
    if (m < 1 || m > DIIS_MAX || n < 1) return fail(DFTB_EINVAL, "diis: need 1 <= m <= 64 entries");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t nn = (size_t)n * n;
    double *buf = nullptr;
    CK(cudaMallocAsync((void **)&buf, sizeof(double) * (2 * m + 1) * nn, st));
    CK(cudaMemcpyAsync(buf, F, sizeof(double) * m * nn, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(buf + m * nn, E, sizeof(double) * m * nn, cudaMemcpyHostToDevice, st));
    launch_diis_single(buf, buf + m * nn, m, n, buf + 2 * m * nn, st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, buf + 2 * m * nn, sizeof(double) * nn, cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(buf, st));
    CK(cudaStreamSynchronize(st));
    return 0;
}

int dftb_plan_kernel_times(dftb_plan *p, int32_t reps, double *ms_jk, double *ms_xc, void *stream) {
    if (!p || reps < 1 || !ms_jk) return fail(DFTB_EINVAL, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    enq_begin(p, st);
    const DevBatch &d = p->d;
    // the kernels skip molecules whose SCF has finished: clear the flags for the timing
    // and restore them afterwards
    std::vector<int> done(d.n_mol);
    CK(cudaMemcpyAsync(done.data(), d.done, sizeof(int) * d.n_mol, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaMemsetAsync(d.done, 0, sizeof(int) * d.n_mol, st));
    cudaEvent_t e[3];
    for (auto &x : e) CK(cudaEventCreate(&x));
    const bool xc = ms_xc != nullptr;     // null: J/K only (no grid needed)
    launch_jk(d, p->jk_bucket_ctas, p->jk_bucket_n, st);                 // warm
    if (xc) launch_xc(d, p->xc_bucket_ctas, p->xc_bucket_n, p->nsh_max, st);
    CK(cudaEventRecord(e[0], st));
    for (int r = 0; r < reps; ++r) launch_jk(d, p->jk_bucket_ctas, p->jk_bucket_n, st);
    CK(cudaEventRecord(e[1], st));
    if (xc)
        for (int r = 0; r < reps; ++r) launch_xc(d, p->xc_bucket_ctas, p->xc_bucket_n, p->nsh_max, st);
    CK(cudaEventRecord(e[2], st));
    CK(cudaEventSynchronize(e[2]));
    float a = 0.f, c = 0.f;
    CK(cudaEventElapsedTime(&a, e[0], e[1]));
    CK(cudaEventElapsedTime(&c, e[1], e[2]));
    *ms_jk = a / reps;
    if (xc) *ms_xc = c / reps;
    for (auto &x : e) cudaEventDestroy(x);
    CK(cudaMemcpyAsync(d.done, done.data(), sizeof(int) * d.n_mol, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    enq_end(p, st);
    return 0;
}

int dftb_plan_post_time(dftb_plan *p, int32_t reps, double *ms, void *stream) {
    if (!p || reps < 1 || !ms) return fail(DFTB_EINVAL, "bad arguments");
    if (p->opts.max_iterations < 2) return fail(DFTB_EINVAL, "needs max_iterations >= 2");
    cudaStream_t st = (cudaStream_t)stream;
    enq_begin(p, st);
    const DevBatch &d = p->d;
    const dftb_opts &o = p->opts;
    const int it = o.max_iterations - 2;        // a non-final iteration: the purification path
    CK(cudaMemsetAsync(d.done, 0, sizeof(int) * d.n_mol, st));
    launch_post(d, p->nmax, it, o.diis_start, o.diis_history, o.damping_factor, o.convergence_std, st);   // warm
    cudaEvent_t e[2];
    for (auto &x : e) CK(cudaEventCreate(&x));
    CK(cudaEventRecord(e[0], st));
    for (int r = 0; r < reps; ++r) {
        CK(cudaMemsetAsync(d.done, 0, sizeof(int) * d.n_mol, st));
        launch_post(d, p->nmax, it, o.diis_start, o.diis_history, o.damping_factor, o.convergence_std, st);
    }
    CK(cudaEventRecord(e[1], st));
    CK(cudaEventSynchronize(e[1]));
    float a = 0.f;
    CK(cudaEventElapsedTime(&a, e[0], e[1]));
    *ms = a / reps;
    for (auto &x : e) cudaEventDestroy(x);
    CK(cudaGetLastError());
    enq_end(p, st);
    return 0;
}

int dftb_fma_peak(int fp64, double *tflops, void *stream) {
    *tflops = fma_peak(fp64, (cudaStream_t)stream);
    CK(cudaGetLastError());
    return 0;
}

#pragma GCC visibility pop
}  // extern "C"
