// Per-molecule setup kernels: nuclear repulsion, S/T/V, molecular grid (Becke).
//
// Reference: molio.nuclear_repulsion (molio.py:78-87), integrals.one_electron
// (integrals.py:115-132 -> _one_electron_kernel, _kernels.py:229-343),
// xc.build_grid (xc.py:123-162 -> _becke_kernel, _kernels.py:622-647).
#include "common.cuh"
#include "md.cuh"

namespace dftb {

__device__ __forceinline__ int find_int(const int *prefix, int n, int g) {
    int lo = 0, hi = n;
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (prefix[mid] <= g) lo = mid; else hi = mid;
    }
    return lo;
}

// E_nn = sum_{a<b} Za Zb / r_ab, pairs summed in the reference's (a, b>a) order.
__global__ void k_enn(DevBatch b) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= b.n_mol) return;
    const int a0 = b.m_atom0[m], na = b.m_natom[m];
    double e = 0.0;
    for (int x = 0; x < na; ++x)
        for (int y = x + 1; y < na; ++y) {
            const double *p = b.a_xyz + 3 * (a0 + x), *q = b.a_xyz + 3 * (a0 + y);
            const double dx = p[0] - q[0], dy = p[1] - q[1], dz = p[2] - q[2];
            e += (double)(b.a_z[a0 + x] * b.a_z[a0 + y]) / sqrt(dx * dx + dy * dy + dz * dz);
        }
    b.enn[m] = e;
}

// S, T, V (and H = T + V) for one fused shell pair per thread, both triangles written.
__global__ void __launch_bounds__(128) k_onee(DevBatch b) {
    const int pr = blockIdx.x * blockDim.x + threadIdx.x;
    if (pr >= b.n_pair) return;
    const int m = find_int(b.m_pair0, b.n_mol, pr);
    const int sa = b.p_sa[pr], sb = b.p_sb[pr];
    const int a0 = b.m_atom0[m];
    const double *A = b.a_xyz + 3 * b.s_atom[sa], *B = b.a_xyz + 3 * b.s_atom[sb];
    double S[4][4], T[4][4], V[4][4];
    onee_pair(b.s_kind[sa], b.s_kind[sb], b.s_exp + 3 * sa, b.s_cs + 3 * sa, b.s_cp + 3 * sa,
              b.s_exp + 3 * sb, b.s_cs + 3 * sb, b.s_cp + 3 * sb, A, B, b.m_natom[m],
              b.a_xyz + 3 * a0, b.a_z + a0, b.boys, S, T, V);
    const int N = b.m_nao[m];
    const int64_t o = b.m_mat0[m];
    const int na = b.s_kind[sa] ? 4 : 1, nb = b.s_kind[sb] ? 4 : 1;
    const int ia = b.s_ao[sa], ib = b.s_ao[sb];
    for (int x = 0; x < na; ++x)
        for (int y = 0; y < nb; ++y) {
            const int64_t u = o + (int64_t)(ia + x) * N + ib + y, w = o + (int64_t)(ib + y) * N + ia + x;
            b.S[u] = b.S[w] = S[x][y];
            b.T[u] = b.T[w] = T[x][y];
            b.V[u] = b.V[w] = V[x][y];
            b.H[u] = b.H[w] = V[x][y] + T[x][y];
        }
}

// Grid points + Becke-partitioned weights; one CTA per atom.  dynamic smem:
// natom_max*(natom_max) inverse distances + natom_max*3 coordinates.
constexpr int GRID_MAX_ATOMS = 96;

__global__ void __launch_bounds__(256) k_grid(DevBatch b) {
    extern __shared__ double gsm[];
    const int atom = blockIdx.x;
    // molecule of this atom
    int lo = 0, hi = b.n_mol;
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (b.m_atom0[mid] <= atom) lo = mid; else hi = mid;
    }
    const int m = lo, a0 = b.m_atom0[m], na = b.m_natom[m], own = atom - a0;
    double *cx = gsm, *inv = gsm + 3 * na;
    for (int t = threadIdx.x; t < 3 * na; t += blockDim.x) cx[t] = b.a_xyz[3 * a0 + t];
    __syncthreads();
    for (int t = threadIdx.x; t < na * na; t += blockDim.x) {
        const int x = t / na, y = t % na;
        double v = 0.0;
        if (x != y) {
            const double dx = cx[3 * x] - cx[3 * y], dy = cx[3 * x + 1] - cx[3 * y + 1], dz = cx[3 * x + 2] - cx[3 * y + 2];
            v = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
        }
        inv[t] = v;
    }
    __syncthreads();
    const int n = b.a_tmpln[atom];
    const double *tp = b.tmpl + 4 * (int64_t)b.a_tmpl0[atom];
    const int64_t g0 = b.a_grid0[atom];
    const double C0 = cx[3 * own], C1 = cx[3 * own + 1], C2 = cx[3 * own + 2];
    double d[GRID_MAX_ATOMS];
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        const double x = C0 + tp[4 * t], y = C1 + tp[4 * t + 1], z = C2 + tp[4 * t + 2];
        double w = tp[4 * t + 3];
        if (na > 1) {
            for (int a = 0; a < na; ++a) {
                const double dx = x - cx[3 * a], dy = y - cx[3 * a + 1], dz = z - cx[3 * a + 2];
                d[a] = sqrt(dx * dx + dy * dy + dz * dz);
            }
            double tot = 0.0, pown = 0.0;
            for (int a = 0; a < na; ++a) {
                double cell = 1.0;
                for (int c = 0; c < na; ++c) {
                    if (c == a) continue;
                    double f = (d[a] - d[c]) * inv[a * na + c];
                    f = 1.5 * f - 0.5 * f * f * f;
                    f = 1.5 * f - 0.5 * f * f * f;
                    f = 1.5 * f - 0.5 * f * f * f;
                    cell *= 0.5 * (1.0 - f);
                }
                tot += cell;
                if (a == own) pown = cell;
            }
            w *= tot > 0.0 ? pown / tot : 0.0;
        }
        if (w < 0.0) {
            if (w < -1e-14) atomicOr(b.status + m, DFTB_ST_NEG_WEIGHT);
            w = 0.0;
        }
        b.g_xyz[3 * (g0 + t)] = x;
        b.g_xyz[3 * (g0 + t) + 1] = y;
        b.g_xyz[3 * (g0 + t) + 2] = z;
        b.g_w[g0 + t] = w;
    }
}

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

void launch_enn(const DevBatch &b, cudaStream_t s) {
    k_enn<<<nblk(b.n_mol, 64), 64, 0, s>>>(b);
}
void launch_onee(const DevBatch &b, cudaStream_t s) {
    if (b.n_pair) k_onee<<<nblk(b.n_pair, 128), 128, 0, s>>>(b);
}
void launch_grid(const DevBatch &b, int max_atoms, cudaStream_t s) {
    const size_t sm = sizeof(double) * ((size_t)max_atoms * max_atoms + 3 * max_atoms);
    smem_optin((const void *)k_grid);
    if (b.n_atom) k_grid<<<b.n_atom, 256, sm, s>>>(b);
}

}  // namespace dftb
