// Shared device-side definitions for the qm1b_b200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>
#include <mutex>
#include <set>
#include <utility>

#include "../../include/qm1b_b200.h"

#define HD __host__ __device__ __forceinline__

namespace dftb {

constexpr int NMAX = DFTB_NMAX;
constexpr int NPRIM = DFTB_NPRIM;
constexpr int NPP = NPRIM * NPRIM;   // primitive pairs per shell pair
constexpr int BOYS_NCOL = 16;        // F_m columns, m = 0..15
constexpr int BOYS_NT = 431;         // T = 0.0 .. 43.0 step 0.1
constexpr int PP_FIELDS = 10;        // p, Px, Py, Pz, 1/(2p), c_ss, c_sp, c_ps, c_pp, bound
constexpr int DIIS_MAX = 64;   // largest DIIS ring (diis_history, capped by max_iterations on the host)
constexpr int NCLS = 6;              // quartet classes (LL|LL) (LL|LS) (LL|SS) (LS|LS) (LS|SS) (SS|SS)

HD int64_t tri(int64_t i) { return i * (i + 1) / 2; }
HD int64_t pidx(int i, int j) { return i >= j ? tri(i) + j : tri(j) + i; }
// ERI store layout ("ket-tiled rows").  Row P = (i, j), i >= j, holds the kets (k, l),
// k >= l, (k, l) <= (i, j) as the lower-triangular 4x4 tiles of its symmetric ket matrix
// restricted to k, l <= i: tile (a, b), a >= b, a <= i/4, sits at tile index tri(a) + b,
// 16 elements [k%4][l%4].  Slots with l > k inside diagonal tiles, with k > i, or with
// k == i and l > j are zero (they belong to other rows).  All i + 1 rows of slab i have the
// same length 16 * tri(i/4 + 1), so a row starts on a 64-byte (f32) / 128-byte (f64)
// boundary and the J/K kernel can read whole tiles with 16-byte vector loads.
// Inside a tile the four rows are rotated by eri_tile_rot(tile index): logical row r sits in
// 4-element slot (r + rot) & 3.  A J/K thread that owns tile tau reads its rows in logical
// order from slots (r + rot) & 3, so the 8 lanes of a quarter warp (8 consecutive tiles,
// 64 bytes apart) hit 8 different 16-byte bank groups instead of 2 (a 4-way conflict).
HD int64_t eri_rowlen(int i) {
    const int64_t A = (i >> 2) + 1;
    return 8 * A * (A + 1);
}
HD int64_t eri_slab0(int i) {                 // elements in all rows with first index < i
    const int64_t a = i >> 2;
    const int64_t h = a * (a - 1) / 2;
    const int64_t full = 8 * (16 * h * h + 58 * ((a - 1) * a * (2 * a - 1) / 6) + 62 * h + 20 * a);
    return full + eri_rowlen(i) * (tri(i) - tri(4 * a));
}
HD int64_t eri_row(int i, int j) { return eri_slab0(i) + (int64_t)j * eri_rowlen(i); }
HD int eri_tile_rot(int tau) { return (tau >> 1) & 3; }
HD int eri_tile_slot(int tau, int r) { return (r + eri_tile_rot(tau)) & 3; }    // 4-element slot of logical row r
HD int eri_ket(int k, int l) {   // k >= l
    const int tau = (int)(tri(k >> 2) + (l >> 2));
    return 16 * tau + 4 * eri_tile_slot(tau, k & 3) + (l & 3);
}
// offset of (ij|kl) in a molecule's store (any index order)
HD int64_t eri_pos(int i, int j, int k, int l) {
    if (i < j) { const int t = i; i = j; j = t; }
    if (k < l) { const int t = k; k = l; l = t; }
    if (tri(i) + j < tri(k) + l) { int t = i; i = k; k = t; t = j; j = l; l = t; }
    return eri_row(i, j) + eri_ket(k, l);
}
HD int64_t eri_size(int N) { return eri_slab0(N); }

// Opt a kernel in to the device's full dynamic shared memory, once per (kernel, device).
// The attribute is process-global state: setting it per launch to a batch-dependent size
// raced between the pipeline's host threads (one plan per thread, batches with different
// AO counts): a thread could launch after another had lowered the limit ("invalid argument" /
// "too many resources requested for launch").  A launch still reserves only its own size.
inline void smem_optin(const void *fn) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    if (!done.insert({fn, dev}).second) return;
    cudaFuncAttributes a;
    int optin = 0;
    cudaFuncGetAttributes(&a, fn);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)a.sharedSizeBytes);
}

// Device-resident view of one batch.  Every pointer is a device pointer owned by
// the plan (plan.cu).  Index conventions: "global" = over the whole batch,
// "local" = within one molecule.
struct DevBatch {
    int n_mol, n_atom, n_shell, n_pair, n_pts;
    int prec;                 // 0 f64, 1 f32 (ERI values + XC arithmetic)
    int eri64;                // ERI store element type: 1 = f64 (f32 build: f32-rounded values)
    // molecules
    const int *m_nao, *m_nocc, *m_natom, *m_atom0, *m_nshell, *m_shell0, *m_pair0;
    const int *m_npl;         // [n_mol*3] pair counts LL, LS, SS
    const int64_t *m_mat0;    // prefix of nao^2
    const int64_t *m_npp0;    // prefix of nao(nao+1)/2
    const int64_t *m_eri0;    // prefix of npp(npp+1)/2
    const int64_t *m_grid0;   // prefix of grid points
    const int *m_jkcta0;      // prefix of J/K CTAs
    const int *m_xccta0;      // prefix of XC CTAs
    const int64_t *m_G0;      // prefix of tri(nao)*nao  (K partial rows)
    const int64_t *m_Jp0;     // prefix of (ncta_jk+1)*npp (J partials)
    const int64_t *m_V0;      // prefix of ncta_xc*nao^2 (Vxc partials)
    const int64_t *cls0;      // [NCLS*(n_mol+1)] quartet-count prefixes per class
    // atoms (global)
    const int *a_z;
    const double *a_xyz;
    const int64_t *a_grid0;
    const int *a_tmpl0, *a_tmpln;
    const double *tmpl;       // [n_tmpl*4]
    // shells (global)
    const int *s_kind, *s_ao, *s_atom;
    const double *s_exp, *s_cs, *s_cp;
    // shell pairs (global); canonical orientation: L before S, else higher index first
    const int *p_sa, *p_sb;
    double *p_geo;            // [6][n_pair] A, B
    double *pp;               // [PP_FIELDS][NPP][n_pair]
    double *p_q;              // [n_pair] Schwarz bound sqrt(max (ab|ab))
    double *qao;              // [sum npp] sqrt((ij|ij))
    // J/K CTA table
    const int *jk_mol, *jk_i0, *jk_i1;
    const int *mol_order;     // molecules by N descending: launch order of the per-molecule kernels
    int n_jk_cta;
    // XC CTA table
    const int *xc_mol;
    const int64_t *xc_p0, *xc_p1;
    int n_xc_cta;
    // grid
    double *g_xyz;            // [n_pts*3]
    double *g_w;              // [n_pts]
    // matrices (each sum nao^2 doubles)
    double *S, *T, *V, *H, *X, *C, *Cp, *rho, *rho_prev, *F, *J, *K, *Vxc, *scratch;
    double *Fring, *Ering;    // [diis_history][sum nao^2]
    // ERI store (f64 or f32)
    void *eri;
    // partials
    double *Gpart, *Jpart, *Vpart, *Epart;
    // per-molecule scalars
    double *enn, *hist, *comp, *Bmat, *eps;
    int *nmo, *ring_n, *ring_head, *done, *conv, *iters, *status;
    int *cpv;                 // [n_mol] Cp holds the previous iteration's eigenvectors (warm start valid)
    int *puri;                // [n_mol] purification sweeps of the last non-final iteration (diagnostics)
    int full_eig;             // 1: eigendecomposition every iteration (host callback path)
    const double *boys;       // [kBoysLMax + 1][BOYS_NT][8] per-order slices (md.cuh)
    int max_it;
    long long *dbg;           // [n_mol*16] phase cycle counters (diagnostics)
};

// Warp / block reductions (deterministic: fixed shuffle tree).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide sum; `red` is >= 32 doubles of shared memory. All threads get the result.
__device__ __forceinline__ double block_sum(double v, double *red) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    if (w == 0) {
        t = lane < nw ? red[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) red[0] = t;
    }
    __syncthreads();
    t = red[0];
    __syncthreads();
    return t;
}
// two block maxima with one set of barriers (red: >= 64 doubles)
__device__ __forceinline__ void block_max2(double &a, double &b, double *red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    a = warp_max(a);
    b = warp_max(b);
    __syncthreads();
    if (lane == 0) { red[w] = a; red[32 + w] = b; }
    __syncthreads();
    if (w == 0) {
        double x = lane < nw ? red[lane] : 0.0, y = lane < nw ? red[32 + lane] : 0.0;
        x = warp_max(x);
        y = warp_max(y);
        if (lane == 0) { red[0] = x; red[32] = y; }
    }
    __syncthreads();
    a = red[0];
    b = red[32];
    __syncthreads();
}

__device__ __forceinline__ double block_max(double v, double *red) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    if (w == 0) {
        t = lane < nw ? red[lane] : 0.0;
        t = warp_max(t);
        if (lane == 0) red[0] = t;
    }
    __syncthreads();
    t = red[0];
    __syncthreads();
    return t;
}

// binary search: largest m with prefix[m] <= g  (prefix has n+1 entries, prefix[0] = 0)
__device__ __forceinline__ int find_mol(const int64_t *prefix, int n, int64_t g) {
    int lo = 0, hi = n;  // invariant prefix[lo] <= g < prefix[hi]
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (__ldg(prefix + mid) <= g) lo = mid; else hi = mid;
    }
    return lo;
}

}  // namespace dftb
