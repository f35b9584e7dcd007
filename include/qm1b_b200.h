/*
 * qm1b_b200 — C ABI of the B200-native batched RKS B3LYP/STO-3G label generator.
 *
 * This is the drop-in boundary for the reference's SCF driver path
 * (/root/reference/pkg/src/deskdft).  The reference is pure Python + numba, so
 * there is no native FFI to mirror verbatim; the entry points below are the
 * batched, plain-C equivalents of the reference's operator boundaries, each
 * citing the reference interface it replaces:
 *
 *   dftb_scf_batch / dftb_plan_run  <- deskdft.scf.scf          (scf.py:139-210)
 *   dftb_plan_one_electron          <- deskdft.integrals.one_electron (integrals.py:115-132)
 *   dftb_plan_eri                   <- deskdft.integrals.eri_packed   (integrals.py:135-196)
 *   dftb_plan_eri_compact           <- eri_packed's screening + canonical order (:147-191)
 *   dftb_plan_jk                    <- deskdft.integrals.build_jk     (integrals.py:199-218)
 *   dftb_plan_grid                  <- deskdft.xc.build_grid          (xc.py:123-162)
 *   dftb_plan_xc                    <- deskdft.xc.xc_matrix           (xc.py:320-350)
 *   dftb_plan_eval_ao               <- deskdft.xc.eval_ao             (xc.py:165-194)
 *   dftb_b3lyp                      <- deskdft.xc.b3lyp               (xc.py:277-306)
 *   dftb_plan_roothaan              <- deskdft.scf.solve_roothaan     (scf.py:86-98)
 *   dftb_diis                       <- deskdft.scf.diis_step          (scf.py:101-132)
 *
 * Conventions: all arrays passed in dftb_batch_in / dftb_results are HOST
 * memory (dftb_results_dev: device memory owned by the caller); the plan owns every device buffer it allocates (freed by
 * dftb_plan_destroy).  Functions taking a `stream` enqueue work on that CUDA
 * stream (cudaStream_t passed as void*; NULL = legacy default stream).
 * Every function returns 0 on success or a DFTB_E* code; dftb_last_error()
 * gives the message (thread-local).  Units: Bohr, Hartree.
 */
#ifndef QM1B_B200_H
#define QM1B_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFTB_NMAX 96          /* max AOs per molecule on the device path */
#define DFTB_NPRIM 3          /* primitives per contracted shell (STO-3G) */

enum {
    DFTB_OK = 0,
    DFTB_EINVAL = 1,          /* bad arguments (maps to DeskDFTError / DimensionError) */
    DFTB_ERESOURCE = 2,       /* N_ao or memory above limits (ResourceLimitError) */
    DFTB_ECUDA = 3,           /* CUDA runtime failure (DeviceError) */
    DFTB_ENUMERIC = 4         /* overlap not PD, negative weight, non-finite XC (DeskDFTError) */
};

/* per-molecule status bits returned in dftb_results.status */
#define DFTB_ST_OVERLAP_NOT_PD   1
#define DFTB_ST_NEG_WEIGHT       2
#define DFTB_ST_XC_NONFINITE     4
#define DFTB_ST_NO_ORBITALS      8
#define DFTB_ST_SINGULAR        16   /* no overlap eigenvalue above the 1e-7 linear-dependence cut */

typedef struct dftb_plan dftb_plan;

/* A batch of molecules, concatenated (host memory).  Shells are FUSED: kind 0 =
 * S (1 AO), kind 1 = L (s,px,py,pz sharing 3 exponents).  Shells are listed in
 * atom order so AO numbering equals the reference's (basis.py:223-276). */
typedef struct {
    int32_t n_mol;
    int32_t n_atom;            /* total atoms */
    int32_t n_shell;           /* total fused shells */
    const int32_t *mol_natom;  /* [n_mol] */
    const int32_t *mol_nshell; /* [n_mol] */
    const int32_t *mol_nocc;   /* [n_mol] doubly occupied orbitals */
    const int32_t *atom_z;     /* [n_atom] */
    const double *atom_xyz;    /* [n_atom*3] Bohr */
    const int32_t *shell_kind; /* [n_shell] 0 = S, 1 = L */
    const int32_t *shell_atom; /* [n_shell] atom index within its molecule */
    const double *shell_exp;   /* [n_shell*3] */
    const double *shell_cs;    /* [n_shell*3] s-component coefficients (normalised) */
    const double *shell_cp;    /* [n_shell*3] p-component coefficients (0 for S) */
    /* atom-centred quadrature templates (xc.py:123-162 without the Becke factor):
     * tmpl_xyzw[4*k] = (r*ux, r*uy, r*uz, w_r*r^2*w_ang); atom a uses
     * tmpl[atom_tmpl0[a] .. atom_tmpl0[a]+atom_tmpln[a]).  May be empty (no grid). */
    int32_t n_tmpl;
    const double *tmpl_xyzw;
    const int32_t *atom_tmpl0; /* [n_atom] */
    const int32_t *atom_tmpln; /* [n_atom] */
} dftb_batch_in;

typedef struct {
    int32_t precision;         /* 0 = f64 build, 1 = f32 build (SCFOptions.precision) */
    int32_t max_iterations;    /* >= 5 (scf.py:60-62) */
    double convergence_std;    /* std(last 5 E) threshold; 0 = fixed iteration count */
    int32_t diis_history;      /* 1..64: DIIS ring slots (the Python layer passes min(diis_history, max_iterations)) */
    int32_t diis_start;
    double damping_factor;
    double screen_eps;         /* Schwarz threshold; primitive cut = 1e-3 * eps */
} dftb_opts;

/* Results (host memory, caller-allocated; any pointer may be NULL to skip). */
typedef struct {
    double *E_total;           /* [n_mol] */
    double *E_comp;            /* [n_mol*5]: E_nn, E_core, E_coulomb, E_exx, E_xc */
    double *history;           /* [n_mol*max_iterations], unused tail = NaN */
    int32_t *iterations;       /* [n_mol] */
    int32_t *converged;        /* [n_mol] */
    int32_t *n_mo;             /* [n_mol] orbitals kept after the linear-dependence drop */
    double *epsilon;           /* [n_mol*DFTB_NMAX], ascending, first n_mo valid */
    double *C;                 /* [sum_m n_ao(m)*n_ao(m)], row-major n_ao x n_ao, first n_mo columns valid */
    int32_t *status;           /* [n_mol] DFTB_ST_* bits */
} dftb_results;

const char *dftb_last_error(void);
const char *dftb_version(void);
int dftb_device_count(int *count);

/* One-shot: upload, run the whole batched SCF on the device, download results. */
int dftb_scf_batch(const dftb_batch_in *in, const dftb_opts *opts, dftb_results *out, void *stream);

/* Plan lifecycle (device-resident inputs; used by the benchmark's `value` arm). */
int dftb_plan_create(const dftb_batch_in *in, const dftb_opts *opts, void *stream, dftb_plan **plan);
int dftb_plan_destroy(dftb_plan *plan);   /* frees after the plan's queued work, stream-ordered */
int dftb_plan_run(dftb_plan *plan, void *stream);              /* setup + SCF loop */
int dftb_plan_begin(dftb_plan *plan, void *stream);            /* setup + core guess only */
int dftb_plan_iterate(dftb_plan *plan, int32_t it, void *stream); /* one SCF iteration */
/* Blocks until this plan's last dftb_plan_run has completed (not any later work queued on
 * `stream` by other plans) and copies the results to host memory on the plan's own stream. */
int dftb_plan_fetch(dftb_plan *plan, dftb_results *out, void *stream);
/* Results into CALLER-OWNED DEVICE buffers (e.g. PyTorch tensors), same layouts as
 * dftb_results; NULL members are skipped.  Enqueued on `stream` after this plan's queued
 * work (stream-ordered; no host synchronisation, the caller's memory is never freed).
 * Replaces the host copy of scf()'s SCFResult fields (scf.py:202-210) for device consumers. */
typedef struct {
    double *E_total;           /* [n_mol] */
    double *E_comp;            /* [n_mol*5] */
    double *history;           /* [n_mol*max_iterations], unused tail = NaN */
    int32_t *iterations;       /* [n_mol] */
    int32_t *converged;        /* [n_mol] */
    int32_t *n_mo;             /* [n_mol] */
    double *epsilon;           /* [n_mol*DFTB_NMAX] */
    double *C;                 /* [sum_m n_ao(m)^2] */
    int32_t *status;           /* [n_mol] */
} dftb_results_dev;
int dftb_plan_fetch_device(dftb_plan *plan, const dftb_results_dev *out, void *stream);
int dftb_plan_info(const dftb_plan *plan, int64_t *info, int n_info);  /* sizes, see plan.cu */

/* Operator-level stages (each enqueues device work; results fetched with dftb_plan_get). */
int dftb_plan_one_electron(dftb_plan *plan, void *stream);    /* S, T, V */
int dftb_plan_eri(dftb_plan *plan, int screened, void *stream);/* dense 8-fold store */
int dftb_plan_grid(dftb_plan *plan, void *stream);             /* points + Becke weights */
int dftb_plan_jk(dftb_plan *plan, const double *rho_host, double *J_host, double *K_host, void *stream);
int dftb_plan_xc(dftb_plan *plan, const double *rho_host, double *Vxc_host, double *Exc_host, void *stream);
int dftb_plan_eval_ao(dftb_plan *plan, int32_t mol, double *phi_host, double *grad_host, void *stream);
/* Roothaan solve for F_host given the plan's S (set by dftb_plan_one_electron or dftb_plan_set). */
int dftb_plan_roothaan(dftb_plan *plan, const double *F_host, double *C_host, double *eps_host,
                       int32_t *n_mo_host, void *stream);
/* Reference-semantics screening of the dense store into the canonical list of
 * molecule `mol` (composite order).  With out arrays NULL, returns the count in *count. */
int dftb_plan_eri_compact(dftb_plan *plan, int32_t mol, double screen_eps, const double *q_split_pair_host,
                          int64_t *count, uint16_t *i, uint16_t *j, uint16_t *k, uint16_t *l,
                          double *v, void *stream);
/* Overwrite an internal per-molecule N x N buffer ("S", "F", "rho", "H") from host memory. */
int dftb_plan_set(dftb_plan *plan, const char *which, int32_t mol, const double *host, int64_t n, void *stream);
/* Scatter a canonical (i>=j, k>=l) packed list into molecule `mol`'s dense store. */
int dftb_plan_eri_load(dftb_plan *plan, int32_t mol, int64_t count, const uint16_t *i, const uint16_t *j,
                       const uint16_t *k, const uint16_t *l, const double *v, void *stream);
/* Overwrite the grid of the batch (points [n_pts*3], weights [n_pts]) — n_pts must equal the plan's. */
int dftb_plan_load_grid(dftb_plan *plan, const double *points, const double *weights, int64_t n_pts, void *stream);
/* Copy an internal per-molecule buffer to host: which = "S","T","V","X","points","weights",
 * "qao","eri" (dense store, values as double), "rho","F". */
int dftb_plan_get(dftb_plan *plan, const char *which, int32_t mol, double *host, int64_t n, void *stream);

/* Standalone pointwise / small kernels on host arrays (device round trip). */
int dftb_b3lyp(const double *n, const double *sigma, int64_t npts, double *exc, double *vrho,
               double *vsigma, void *stream);
int dftb_diis(const double *F, const double *E, int32_t m, int32_t n, double *out, void *stream);

/* Timing helpers used by bench.py: per-stage device time (ms) of the last run,
 * and the count of kernels launched by the last dftb_plan_run. */
int dftb_plan_stage_times(const dftb_plan *plan, double *ms, int n);
int dftb_plan_launch_count(const dftb_plan *plan, int64_t *count);
int dftb_plan_set_timing(dftb_plan *plan, int enable);
/* enable != 0: every SCF iteration diagonalises F' and stores C (the host iteration_callback
 * path, scf.py:188-189, observes C each iteration).  Default 0: iterations before the last form
 * the density projector by trace-correcting purification and only the last one (or the one
 * that converges) diagonalises - the returned orbitals and eigenvalues are the same. */
int dftb_plan_set_full_eig(dftb_plan *plan, int enable);
/* Measured-peak helper: FP64 / FP32 FMA throughput microbenchmark (TFLOP/s). */
int dftb_fma_peak(int fp64, double *tflops, void *stream);
/* Kernel-level timing for roofline reporting: re-runs the J/K digestion and the XC
 * kernels (pure functions of the device-resident density; they only rewrite their own
 * partials) `reps` times between CUDA events on `stream` and returns the average time of
 * one J/K launch set and of one XC launch set (ms).  Requires a completed dftb_plan_run, or
 * (ms_xc == NULL: J/K only) a dense store from dftb_plan_eri and a density from dftb_plan_jk. */
int dftb_plan_kernel_times(dftb_plan *plan, int32_t reps, double *ms_jk, double *ms_xc, void *stream);
/* Kernel-level timing of the post kernel (Fock, energies, DIIS, density projector) re-run as a
 * non-final SCF iteration on the resident state.  Advances the plan's SCF state: call it
 * only after the results were fetched. */
int dftb_plan_post_time(dftb_plan *plan, int32_t reps, double *ms, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* QM1B_B200_H */
