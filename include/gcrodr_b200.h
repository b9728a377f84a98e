/*
 * gcrodr_b200.h -- C ABI of the B200-native GCRO-DR-IR solver.
 *
 * The reference (irkit, /root/reference/pkg/src/irkit) is a pure-Python
 * package; its "boundary" is the Python API.  This C ABI is
 * what a binding for that API calls (see INTEGRATION.md for the ctypes
 * binding the drop-in package uses).  Every entry point below replaces a
 * reference function; the citation is given next to each declaration.
 *
 * Conventions
 *   - Matrices are row-major (numpy C order) float64 carriers.
 *   - Host pointers unless the argument name ends in _dev.
 *   - Every call returns gb_status; numerical failures that the reference
 *     reports in-band (zero pivots, x0 overflow, missing reference solution)
 *     are reported through out-parameters, not as errors.
 *   - stream: a cudaStream_t cast to void* (NULL = legacy default stream).
 */
#ifndef GCRODR_B200_H
#define GCRODR_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* formats -- irkit.precision.Format (precision.py:54-60) */
#define GB_HALF 0
#define GB_SINGLE 1
#define GB_DOUBLE 2
#define GB_QUAD 3

/* methods -- irkit.refine.Method (refine.py:56-61) */
#define GB_SIR 0
#define GB_GMRES_IR 1
#define GB_SGMRES_IR 2
#define GB_RGMRES_IR 3
#define GB_RSGMRES_IR 4

typedef enum {
  GB_OK = 0,
  GB_ERR_ARG = 1,         /* ValueError in the reference */
  GB_ERR_UNSUPPORTED = 2, /* valid in the reference, not built here */
  GB_ERR_CUDA = 3,
  GB_ERR_STATE = 4        /* call order violated */
} gb_status;

/* Resolved RefineConfig (refine.py:100-134): the caller resolves the
 * defaults (m = min(n, 40) when 0, tau by u, max_cycles = ceil(10 n / m),
 * extra precision by method) exactly as the reference does. */
typedef struct {
  int uf, u, ur;         /* PrecisionTriple */
  int method;            /* GB_* method */
  int m, k;              /* restart length, recycle dimension */
  double tau;            /* inner relative tolerance */
  int max_cycles;        /* GmresConfig/GcrodrConfig.resolved_max_cycles */
  int reorthogonalize;   /* RefineConfig.reorthogonalize */
  int extra_precision;   /* operator at u^2 (1) or u (0) */
  int grid_ctas;         /* CTAs cooperating on one system; 0 = auto */
  int lu_mode;           /* 0 = exact (reference arithmetic) */
  int explicit_residual; /* GmresConfig.restart_residual / GcrodrConfig.cycle_residual
                           * != "recurrence": s - A~ x recomputed at each restart
                           * (gmres.py:292-295, gcrodr.py:301-304, 376-379) */
} gb_options;

/* One refinement step (refine.py:362-407 loop body) */
typedef struct {
  double nu;         /* ||r||_inf at the top of the step */
  int inner_iters;   /* sum of Arnoldi steps (GmresOutcome.total_iterations) */
  int ncycles;       /* restart / deflated cycles */
  int status;        /* 1 converged, 2 stagnated, 4 breakdown, 256 nu == 0, 512 nu non-finite */
  int applies;       /* operator applications */
  int keff;          /* recycle dimension carried out */
  int pad;
  double ferr;       /* forward error vs xref (NaN without xref) */
  double nbe, cbe;   /* backward errors after the update */
} gb_step_info;

typedef struct gb_solver gb_solver;

/* library */
const char* gb_version(void);
const char* gb_last_error(void);
int gb_device_count(void);

/* solver context: device workspaces for one system of order n */
gb_status gb_solver_create(gb_solver** out, int n, const gb_options* opt, void* stream);
gb_status gb_solver_destroy(gb_solver* s);

/* refine.py:285-300 -- A, b rounded to u, ||A||_inf, ||b||_inf */
gb_status gb_set_system(gb_solver* s, const double* a, const double* b);
/* same with float64 inputs already resident in device memory */
gb_status gb_set_system_device(gb_solver* s, const double* a_dev, const double* b_dev);

/* densela.lu_factor (densela.py:124-168) on fl_u(A) rounded to u_f.
 * zero_col = first exact zero pivot (-1 if none), growth = max|U|/max|A| */
gb_status gb_factorize(gb_solver* s, int* zero_col, double* growth);

/* refine.py:317-321 -- x0 = lu_solve(F, b, u_f) stored in u; x0_reset = 1
 * when the substitution overflowed and x0 was reset to 0 */
gb_status gb_initial_solution(gb_solver* s, int* x0_reset);

/* refine._reference_solution (refine.py:236-258); ok = 0 -> None */
gb_status gb_reference_solution(gb_solver* s, int* ok);

/* one refinement step: residual-scaled correction solve, update, errors */
gb_status gb_refine_step(gb_solver* s, gb_step_info* info);

/* per-cycle Arnoldi steps and k_eff of the last step */
gb_status gb_last_cycles(gb_solver* s, int* iters, int* keff, int cap, int* ncycles);

/* current solution x (u-valued) into a float64 host array */
gb_status gb_get_solution(gb_solver* s, double* x);
gb_status gb_get_reference(gb_solver* s, double* xref);
gb_status gb_get_factors(gb_solver* s, double* lu_packed, long long* perm);

/* kernel-level entry points mirroring densela (one vector, host buffers):
 * apply_preconditioned (densela.py:268-299), precond_rhs (314-333),
 * residual (340-361), lu_solve (235-261).  fmt = context format. */
gb_status gb_apply_preconditioned(gb_solver* s, const double* v, double* w, int fmt);
gb_status gb_precond_rhs(gb_solver* s, const double* r, double* out, int fmt);
gb_status gb_residual(gb_solver* s, const double* x, double* r, int fmt);
gb_status gb_lu_solve(gb_solver* s, const double* b, double* x);

/* The inner solver alone, as the refinement loop calls it: gmres_solve
 * (gmres.py:235-311) for the GMRES methods, gcrodr_solve (gcrodr.py:221-419)
 * for the recycling ones, on the right-hand side r (rounded to u; the loop
 * passes fl_u(r / ||r||_inf), refine.py:366-378) with this solver's m, k,
 * tau, max_cycles.  d = the solution of U^-1 L^-1 A d = U^-1 L^-1 r, info =
 * iterations / cycles / status / applies / k_eff (per-cycle counts through
 * gb_last_cycles).  The recycle space is the context's: it is carried from
 * the previous step or inner solve (recycle_in) and kept for the next one
 * (the returned RecycleSpace); reset_recycle = 1 starts cold (recycle_in =
 * None). */
gb_status gb_debug_inner_solve(gb_solver* s, const double* r, int reset_recycle, double* d, gb_step_info* info);

/* check_convergence's device part (refine.py:194-208): r = b - A x at u_r
 * (r may be NULL), nbe = ||r||_inf / (||A||_inf ||x||_inf + ||b||_inf), cbe =
 * max_i |r_i| / (|A| |x| + |b|)_i over the finite ratios. */
gb_status gb_backward_errors(gb_solver* s, const double* x, double* r, double* nbe, double* cbe);

/* measurement: device time (ms) of one kernel-level launch of `what`
 * (0 apply_preconditioned, 1 precond_rhs, 2 residual in u_r, 3 lu_solve),
 * averaged over `reps` back-to-back launches on device-resident data (the
 * vector of the last kernel-level call).  No reference counterpart. */
gb_status gb_time_op(gb_solver* s, int what, int reps, double* ms_per_launch);

/* diagnostics: arm a phase-timer log of `cap` (tag, globaltimer ns) entries
 * for subsequent launches; with out != NULL first copy the current log
 * (1 + 2*cap words: count, then pairs) out.  cap = 0 disarms. */
gb_status gb_debug_phaselog(gb_solver* s, int cap, unsigned long long* out);

/* diagnostics: the Hessenberg matrix H of the last Arnoldi cycle, (m+1) x m
 * column-major fp64 (arnoldi_cycle's H, gmres.py:123-215); for per-cycle
 * parity checks run the step with max_cycles = 1.  No reference counterpart. */
gb_status gb_debug_hessenberg(gb_solver* s, double* h);

/* diagnostics: lower the cycle cap of subsequent steps to `cycles`
 * (1 <= cycles <= the max_cycles the solver was created with).  Mirrors
 * calling gmres_solve / gcrodr_solve with a smaller GmresConfig.max_cycles
 * (gmres.py:51-54, gcrodr.py:86-89): per-cycle parity checks run one cycle
 * at a time, the bench truncates its warm-up solves with it. */
gb_status gb_debug_set_max_cycles(gb_solver* s, int cycles);

/* number of kernels this library has launched (process-wide) */
long long gb_launch_count(void);

/* timing helper: device time (ms) of the last gb_refine_step / gb_factorize */
double gb_last_step_ms(gb_solver* s);
double gb_last_factor_ms(gb_solver* s);

/* blocked tensor-mode LU (lu_mode = 1, n >= 2048; lu_factor, densela.py:148-168
 * restated as a blocked GEPP): device times of the last factorisation,
 * out[0] = ms in the rank-1024 tcgen05 trailing updates, out[1] = their flop
 * count (2 M N K summed), out[2] = ms in U12 = L11^-1 A12, out[3] = ms in the
 * panel factorisations and row interchanges.  Zeros in exact mode. */
gb_status gb_lu_tc_stats(gb_solver* s, double* out);

/* Batched mode (config 3): `count` independent systems of order n, one CTA
 * per system, the whole refinement loop (refine.py:277-421) on the device.
 * a: count x n x n, b: count x n (float64, host or device per on_device).
 * Outputs per system (host arrays): converged, steps, reason (0 none,
 * 1 IMaxExceeded, 2 InnerStagnation, 3 ErrorGrowth), inner[count*i_max],
 * nbe[count*i_max], ferr[count*i_max], x[count*n], growth[count],
 * flags[count] (1 x0_reset, 2 no_reference_solution, 4 lu_failed). */
typedef struct {
  int* converged;
  int* steps;
  int* reason;
  int* inner;
  double* nbe;
  double* ferr;
  double* x;
  double* growth;
  int* flags;
} gb_batch_out;

gb_status gb_solve_batched(int count, int n, const gb_options* opt, int i_max, double c_conv,
                           const double* a, const double* b, int on_device, gb_batch_out* out,
                           double* device_ms, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GCRODR_B200_H */
