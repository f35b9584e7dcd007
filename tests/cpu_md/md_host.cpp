// TEST HARNESS (not product code): runs the device integral math of
// paper_2311_01135_b200/csrc/md.cuh on the CPU so tests can check it against the
// oracle without a GPU.  Built by tests/cpu_md/build.sh into tests/cpu_md/_md_host.so.
#define __host__
#define __device__
#define __forceinline__ inline
#include <stdint.h>
#include <math.h>
#include <vector>
#include "../../paper_2311_01135_b200/csrc/md.cuh"

using namespace dftb;

static int64_t tri64(int64_t i) { return i * (i + 1) / 2; }
static int64_t pidx64(int i, int j) { return i >= j ? tri64(i) + j : tri64(j) + i; }

struct Shell { int kind, ao; double xyz[3], e[3], cs[3], cp[3]; };

static void pair_record(const Shell &a, const Shell &b, std::vector<double> &pp, int64_t np, int64_t pr) {
    double rab2 = 0;
    for (int d = 0; d < 3; ++d) rab2 += (a.xyz[d] - b.xyz[d]) * (a.xyz[d] - b.xyz[d]);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double p = a.e[i] + b.e[j], K = exp(-(a.e[i] * b.e[j] / p) * rab2);
            int k = 3 * i + j;
            auto put = [&](int f, double v) { pp[((int64_t)f * 9 + k) * np + pr] = v; };
            put(PF_P, p);
            for (int d = 0; d < 3; ++d) put(PF_X + d, (a.e[i] * a.xyz[d] + b.e[j] * b.xyz[d]) / p);
            put(PF_H, 0.5 / p);
            put(PF_CSS, a.cs[i] * b.cs[j] * K);
            put(PF_CSP, a.cs[i] * b.cp[j] * K);
            put(PF_CPS, a.cp[i] * b.cs[j] * K);
            put(PF_CPP, a.cp[i] * b.cp[j] * K);
            put(PF_BOUND, fmax(fabs(a.cs[i]), fabs(a.cp[i])) * fmax(fabs(b.cs[j]), fabs(b.cp[j])) * K);
        }
}

template <int KA, int KB, int KC, int KD, int KC0, int NKS>
static void run_slice(const PPView &V, int64_t P, int64_t Q, const Shell &a, const Shell &b,
                      const Shell &c, const Shell &d, const double *tab, double prim_cut, double *dense,
                      int64_t n) {
    constexpr int NA = KA ? 4 : 1, NB = KB ? 4 : 1, ND = KD ? 4 : 1;
    double out[NA * NB][NKS];
    for (int x = 0; x < NA * NB; ++x)
        for (int y = 0; y < NKS; ++y) out[x][y] = 0.0;
    eri_quartet<KA, KB, KC, KD, KC0, NKS>(V, P, Q, a.xyz, b.xyz, c.xyz, d.xyz, tab, prim_cut, out);
    for (int x = 0; x < NA * NB; ++x)
        for (int y = 0; y < NKS; ++y) {
            int kc = KC0 + y;
            int i = a.ao + x / NB, j = b.ao + x % NB, k = c.ao + kc / ND, l = d.ao + kc % ND;
            int64_t Pi = pidx64(i, j), Qi = pidx64(k, l);
            if (Pi < Qi) { int64_t t = Pi; Pi = Qi; Qi = t; }
            dense[tri64(Pi) + Qi] = out[x][y];
        }
}

template <int KA, int KB, int KC, int KD>
static void run_all(const PPView &V, int64_t P, int64_t Q, const Shell *s, const double *tab,
                    double cut, double *dense, int64_t n, int sa, int sb, int sc, int sd) {
    constexpr int NKET = (KC ? 4 : 1) * (KD ? 4 : 1);
    // use the un-split instantiation for small kets, 1-component slices otherwise
    if constexpr (NKET == 16) {
#define S1(c) run_slice<KA, KB, KC, KD, c, 1>(V, P, Q, s[sa], s[sb], s[sc], s[sd], tab, cut, dense, n);
        S1(0) S1(1) S1(2) S1(3) S1(4) S1(5) S1(6) S1(7) S1(8) S1(9) S1(10) S1(11) S1(12) S1(13) S1(14) S1(15)
    } else if constexpr (NKET == 4 && KA + KB == 2) {
        S1(0) S1(1) S1(2) S1(3)
#undef S1
    } else {
        run_slice<KA, KB, KC, KD, 0, NKET>(V, P, Q, s[sa], s[sb], s[sc], s[sd], tab, cut, dense, n);
    }
}

extern "C" {

void md_boys_table(double *tab) { boys_table_host(tab); }

// Dense 8-fold ERI store for one molecule (unscreened unless eps > 0), plus S, T, V.
// Shell arrays: kind, ao, xyz[3*nsh], exp/cs/cp[3*nsh]; nuclei natom, axyz, az.
void md_molecule(int nsh, const int *kind, const int *ao, const double *xyz, const double *ex,
                 const double *cs, const double *cp, int n_ao, int natom, const double *axyz,
                 const int *az, double prim_cut, double *dense, double *S, double *T, double *Vm) {
    std::vector<double> full(431 * 16), tab((size_t)(kBoysLMax + 1) * kBoysNT * 8);
    boys_table_host(full.data());
    boys_slices_host(full.data(), tab.data());
    std::vector<Shell> sh(nsh);
    for (int s = 0; s < nsh; ++s) {
        sh[s].kind = kind[s];
        sh[s].ao = ao[s];
        for (int d = 0; d < 3; ++d) {
            sh[s].xyz[d] = xyz[3 * s + d];
            sh[s].e[d] = ex[3 * s + d];
            sh[s].cs[d] = cs[3 * s + d];
            sh[s].cp[d] = cp[3 * s + d];
        }
    }
    // canonical pair orientation: L shell first, else higher index first
    std::vector<int> pa, pb;
    for (int a = 0; a < nsh; ++a)
        for (int b = 0; b <= a; ++b) {
            int x = a, y = b;
            if (sh[x].kind < sh[y].kind) { int t = x; x = y; y = t; }
            pa.push_back(x);
            pb.push_back(y);
        }
    int64_t np = pa.size();
    std::vector<double> pp((int64_t)10 * 9 * np);
    for (int64_t p = 0; p < np; ++p) pair_record(sh[pa[p]], sh[pb[p]], pp, np, p);
    PPView V{pp.data(), np};
    for (int64_t P = 0; P < np; ++P)
        for (int64_t Q = 0; Q <= P; ++Q) {
            int64_t bp = P, kp = Q;
            int kb = sh[pa[bp]].kind + sh[pb[bp]].kind, kk = sh[pa[kp]].kind + sh[pb[kp]].kind;
            if (kk > kb) { int64_t t = bp; bp = kp; kp = t; }
            int a = pa[bp], b = pb[bp], c = pa[kp], d = pb[kp];
            int code = sh[a].kind * 8 + sh[b].kind * 4 + sh[c].kind * 2 + sh[d].kind;
            switch (code) {
                case 15: run_all<1, 1, 1, 1>(V, bp, kp, sh.data(), tab.data(), prim_cut, dense, n_ao, a, b, c, d); break;
                case 14: run_all<1, 1, 1, 0>(V, bp, kp, sh.data(), tab.data(), prim_cut, dense, n_ao, a, b, c, d); break;
                case 12: run_all<1, 1, 0, 0>(V, bp, kp, sh.data(), tab.data(), prim_cut, dense, n_ao, a, b, c, d); break;
                case 10: run_all<1, 0, 1, 0>(V, bp, kp, sh.data(), tab.data(), prim_cut, dense, n_ao, a, b, c, d); break;
                case 8: run_all<1, 0, 0, 0>(V, bp, kp, sh.data(), tab.data(), prim_cut, dense, n_ao, a, b, c, d); break;
                case 0: run_all<0, 0, 0, 0>(V, bp, kp, sh.data(), tab.data(), prim_cut, dense, n_ao, a, b, c, d); break;
                default: break;
            }
        }
    for (int64_t p = 0; p < np; ++p) {
        const Shell &a = sh[pa[p]], &b = sh[pb[p]];
        double s4[4][4], t4[4][4], v4[4][4];
        onee_pair(a.kind, b.kind, a.e, a.cs, a.cp, b.e, b.cs, b.cp, a.xyz, b.xyz, natom, axyz, az,
                  tab.data(), s4, t4, v4);
        int na = a.kind ? 4 : 1, nb = b.kind ? 4 : 1;
        for (int x = 0; x < na; ++x)
            for (int y = 0; y < nb; ++y) {
                int i = a.ao + x, j = b.ao + y;
                S[i * n_ao + j] = S[j * n_ao + i] = s4[x][y];
                T[i * n_ao + j] = T[j * n_ao + i] = t4[x][y];
                Vm[i * n_ao + j] = Vm[j * n_ao + i] = v4[x][y];
            }
    }
}
}

#include "../../paper_2311_01135_b200/csrc/b3lyp.cuh"
extern "C" void md_b3lyp(int64_t n, const double *rho, const double *sig, double *exc, double *vr, double *vs) {
    for (int64_t i = 0; i < n; ++i) {
        XCOut o = b3lyp_point(rho[i], sig[i]);
        exc[i] = o.exc; vr[i] = o.vrho; vs[i] = o.vsigma;
    }
}
