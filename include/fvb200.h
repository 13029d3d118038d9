/*
 * fvb200.h -- C ABI of the B200-native finite-volume stage hot path.
 *
 * The reference (`conslaw`, /root/reference/pkg/src/conslaw) is pure Python
 * and has no FFI; each entry point below replaces one reference function on
 * the hot path.  The Python host layer
 * (paper_1912_07645_b200/*.py) binds these with ctypes and mirrors the
 * reference's API on top; INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - Fields are float64, component-major SoA, x fastest: the reference
 *    Field.data layout (grid.py:3-6, 81-88).  A field is described by a base
 *    pointer and an fvb_layout (element strides + offset of interior cell
 *    (0,0,0) of component 0), so padded (ghosted) and interior-only buffers
 *    both work.  Ghost cells are read from memory only on axes whose
 *    boundary is FVB_BC_HALO; periodic/outflow ghosts are resolved in-kernel
 *    (identical values to fill_boundary, grid.py:147-175).
 *  - All device pointers are owned by the caller; the library owns only the
 *    context scratch.  Calls are stream-ordered on the context's stream.
 *  - Every function returns an fvb status; details via fvb_last_error.
 */
#ifndef FVB200_H
#define FVB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: map 1:1 onto the reference exceptions (errors.py:4-46) */
#define FVB_OK 0
#define FVB_E_CONFIG 1      /* ConfigError */
#define FVB_E_UNPHYSICAL 2  /* UnphysicalStateError */
#define FVB_E_SIMULATION 3  /* SimulationError */
#define FVB_E_STATIC 4      /* StaticFieldError */
#define FVB_E_PROTOCOL 5    /* ProtocolError */
#define FVB_E_CUDA 6        /* CUDA runtime failure */

/* error detail (fvb_run_info.errsub) */
#define FVB_SUB_NONE 0
#define FVB_SUB_INIT_UNPHYSICAL 1   /* solver.py:211-212 */
#define FVB_SUB_STAGE_UNPHYSICAL 2  /* solver.py:90-93 (cell = z*ny*nx+y*nx+x) */
#define FVB_SUB_NONFINITE 3         /* solver.py:231-238 (cell = comp-major flat) */
#define FVB_SUB_POST_UNPHYSICAL 4   /* solver.py:239-242 */
#define FVB_SUB_HLLC_DEGENERATE 5   /* numerics.py:166-167 */
#define FVB_SUB_SPEED_UNPHYSICAL 6  /* equations.py:118-119 via wave_speed_maxima */
#define FVB_SUB_REMOTE 7            /* another rank of a decomposed run failed (parallel.py:470-472) */

enum { FVB_EQ_EULER = 0, FVB_EQ_BURGERS = 1, FVB_EQ_ADVECTION = 2 };
enum { FVB_FLUX_RUSANOV = 0, FVB_FLUX_HLLC = 1 };
enum { FVB_RECON_NONE = 0, FVB_RECON_WENO2 = 1, FVB_RECON_WENO3 = 2 };
enum { FVB_BC_PERIODIC = 0, FVB_BC_OUTFLOW = 1, FVB_BC_HALO = 2 };
/* T_END: run_simulation (solver.py:199-246); FIXED: run_parallel n_steps;
 * PAR_T_END: run_parallel without n_steps (parallel.py:490-520: t_end loop,
 * finiteness-only post-step check) */
enum { FVB_MODE_T_END = 0, FVB_MODE_FIXED = 1, FVB_MODE_PAR_T_END = 2 };
enum { FVB_ARITH_EXACT = 0, FVB_ARITH_FAST = 1 };

/* SchemeConfig + GridSpec + EquationModel (solver.py:36-44, grid.py:39-50,
 * equations.py:27-31) flattened. */
typedef struct fvb_scheme {
  int32_t dim;        /* 1..3 */
  int32_t ncomp;      /* dim+2 (Euler) or 1 */
  int32_t eq;         /* FVB_EQ_* */
  int32_t flux;       /* FVB_FLUX_* */
  int32_t recon;      /* FVB_RECON_* */
  int32_t rk_order;   /* 1..3 */
  int32_t arith;      /* FVB_ARITH_EXACT (bitwise == reference) or FAST */
  int32_t ghost;      /* ghost width present in memory (HALO axes) */
  int32_t bc[3];      /* FVB_BC_* per axis, x first */
  int32_t pad;
  int64_t cells[3];   /* x first; unused axes = 1 */
  double deltas[3];   /* cell sizes (grid.py:68-75) */
  double gamma;
  double weno_eps;
  double cfl;
  double t_end;
  double adv[3];      /* advection speeds */
} fvb_scheme;

/* Element strides of a field buffer. */
typedef struct fvb_layout {
  int64_t origin;     /* offset of interior (0,0,0), component 0 */
  int64_t sy, sz;     /* row / plane stride */
  int64_t sc;         /* component stride */
  int64_t si;         /* instance stride (batched ensembles) */
} fvb_layout;

/* Per-instance result of fvb_run. */
typedef struct fvb_run_info {
  double t;
  double dt;
  int64_t steps;
  int32_t err;
  int32_t errsub;
  int64_t errcell;
} fvb_run_info;

typedef struct fvb_ctx fvb_ctx;

/* context: device + stream (cudaStream_t as void*, NULL = legacy default) */
int fvb_ctx_create(int device, void* stream, fvb_ctx** out);
int fvb_ctx_destroy(fvb_ctx* ctx);
int fvb_ctx_set_stream(fvb_ctx* ctx, void* stream);
int fvb_last_error(const fvb_ctx* ctx, char* buf, size_t n);
int fvb_sync(fvb_ctx* ctx);
int fvb_version(void);

/* grid.py:167-175 fill_boundary: write periodic/outflow ghosts in memory
 * (sequential x, y, z passes so corners fill transitively). */
int fvb_fill_ghosts(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay,
                    double* u, int ninst);

/* solver.py:128-136 wave_speed_maxima: per-axis max over the interior.
 * h_max: host array of dim doubles per instance. Raises (returns)
 * FVB_E_UNPHYSICAL if any interior state is unphysical (check=True). */
int fvb_wave_speed_maxima(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay,
                          const double* u, int ninst, double* h_max);

/* solver.py:82-113 spatial_residual: L(u) for the interior into `out`
 * (same layout as u, interior cells only written). */
int fvb_spatial_residual(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay,
                         const double* u, double* out, int ninst);

/* solver.py:176-196 ssp_rk_step with a host dt: un is advanced in place
 * using scratch buffers w1, w2 (same layout). */
int fvb_ssp_rk_step(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay,
                    double* un, double* w1, double* w2, int ninst, double dt);

/* solver.py:199-246 run_simulation (mode FVB_MODE_T_END, max_steps<0 = none)
 * or parallel.py:479-521's n_steps loop (FVB_MODE_FIXED, max_steps = n).
 * bufs[0] holds u^0 on entry; the final field is in bufs[info.steps%2] for
 * rk_order 1, else bufs[0].  bufs[1], bufs[2]: scratch.  h_log (optional):
 * host array of ninst*log_cap (t, dt) pairs (ring: step s at (s-1)%log_cap).  graph_steps: steps per
 * CUDA-graph batch (0 = default). */
int fvb_run(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, double* bufs[3],
            int ninst, int mode, int64_t max_steps, double* h_log, int64_t log_cap,
            int graph_steps, fvb_run_info* h_info);

/* Asynchronous variant for timing: enqueue exactly n_steps FIXED-mode steps
 * (no host sync, no dt cap), continuing from the context's device state.
 * fvb_run_begin resets the state (t=0, initial wave-speed pass). */
int fvb_run_begin(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, double* bufs[3],
                  int ninst, int mode, int64_t max_steps);
int fvb_run_steps(fvb_ctx* ctx, int64_t n_steps);
int fvb_run_end(fvb_ctx* ctx, fvb_run_info* h_info, double* h_log, int64_t log_cap);
/* read the per-instance state of the active run (blocking); h_done optional */
int fvb_run_poll(fvb_ctx* ctx, fvb_run_info* h_info, int32_t* h_done);
/* enable the on-device (t, dt) step log for the next fvb_run_begin:
 * per_instance entries for each of ninst instances (0 disables) */
int fvb_run_set_log(fvb_ctx* ctx, int64_t per_instance, int ninst);
/* copy the step-log ring of the active run: entry (inst, (step-1) % per_instance)
 * holds (t, dt) of that step; h_log has 2*ninst*per_instance doubles */
int fvb_run_read_log(fvb_ctx* ctx, double* h_log, int64_t per_instance);
/* parallel.py:430-521 on one device: the ninst instances of the next
 * fvb_run_begin are the subdomains of ONE run on a Cartesian rank grid
 * (ranks[3], x fastest, parallel.py:45-89).  Axes with ranks > 1 must be
 * FVB_BC_HALO in the scheme; a face-only halo kernel fills their ghosts
 * before every stage (periodic[k]: wrap at the world edge, else outflow).
 * All instances share one step state (global dt = max over subdomains,
 * parallel.py:498-501).  ranks = NULL clears. */
int fvb_run_set_topology(fvb_ctx* ctx, const int32_t* ranks, const int32_t* periodic);
/* Process-per-GPU decomposition (parallel.py:479-521 over NCCL): with
 * external reduce on, the next fvb_run_begin computes the local wave-speed
 * maxima but does not finalise; the caller drives the step stage by stage:
 *   for s in stages: fill HALO ghosts of the stage input (fvb_halo_pack /
 *   send-recv / fvb_halo_unpack); fvb_run_stage(ctx, s)
 *   fvb_run_export(ctx, d_buf)        d_buf[dim+2]: maxima, hard-error, unphysical
 *   all-reduce(MAX) d_buf across ranks
 *   fvb_run_finalize(ctx, d_buf, 1)   (post = 0 after fvb_run_begin)
 * Stage inputs: stage s of RK2/3 reads bufs[s]; RK1 reads bufs[steps % 2]. */
int fvb_run_set_external_reduce(fvb_ctx* ctx, int on);
int fvb_run_stage(fvb_ctx* ctx, int stage);
/* the same stage restricted to march-axis cells [row_lo, row_hi) (dim >= 2):
 * the inner box runs while the march-axis halos are in flight, the shell
 * slabs after they land (overlapped_residual, parallel.py:288-361); pass
 * last_part = 1 on the final call of a stage */
int fvb_run_stage_rows(fvb_ctx* ctx, int stage, int64_t row_lo, int64_t row_hi, int last_part);
/* the same stage restricted to the cell box [lo[k], hi[k]) (x, y, z; dim
 * entries): the overlap schedule of a decomposition split along several
 * axes (parallel.py:288-361) -- the inner box runs while every split axis's
 * halos are in flight, then the disjoint shell slabs. */
int fvb_run_stage_box(fvb_ctx* ctx, int stage, const int64_t* lo, const int64_t* hi, int last_part);
/* fused halo exchange (parallel.py:201-254 without the message step): with
 * the march axis (y in 2D, z in 3D) split, lo[k] / hi[k] are the low / high
 * neighbour's copies of bufs[k] -- peer memory over NVLink (CUDA IPC /
 * symmetric memory), identical layout.  Every stage then also stores its
 * first / last g march rows into the neighbour's ghost rows of the buffer it
 * writes; the caller orders stages across ranks (a device barrier after each
 * stage).  lo or hi may be NULL (world edge).  External-reduce runs, one
 * subdomain per context. */
int fvb_run_set_peers(fvb_ctx* ctx, double* const* lo, double* const* hi);
int fvb_run_export(fvb_ctx* ctx, double* d_out);
int fvb_run_finalize(fvb_ctx* ctx, const double* d_global, int post);
/* kernel launches issued by the last fvb_run / fvb_run_steps calls */
int64_t fvb_launch_count(const fvb_ctx* ctx);

/* uq.py:135-148 MomentAccumulator.merge of one sample (count 1, m2 0) into
 * (mean, m2) holding `count_before` samples; u: field in `lay`, mean/m2:
 * dense (ncomp, *interior) arrays. */
int fvb_moments_push(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay,
                     const double* u, int inst, double* mean, double* m2, int64_t count_before);
/* the same for instances inst .. inst+nbatch-1 merged in that order (one
 * read + write of mean / m2 per batch; bitwise equal to nbatch pushes) */
int fvb_moments_push_batch(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, const double* u, int inst,
                           int nbatch, double* mean, double* m2, int64_t count_before);

/* uq.py:135-148 merge of two accumulators (Chan) for the cross-GPU reduce:
 * (mean_a, m2_a, count_a) <- merge with (mean_b, m2_b, count_b), n values. */
int fvb_moments_merge(fvb_ctx* ctx, double* mean_a, double* m2_a, int64_t count_a,
                      const double* mean_b, const double* m2_b, int64_t count_b, int64_t n);

/* uq.py:254-262 StructureFunctionAccumulator.update: per-sample sums for
 * h = 0..H of mean over positions/axes of |u(x+h e_j) - u(x)|^p (periodic),
 * added into d_sums (device, H+1 doubles) in the reference's order. */
int fvb_structure_push(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay,
                       const double* u, int inst, int comp, double p, int H, double* d_sums);

/* iodsl/expr.py:338-386 eval_init on the device: evaluate
 * the per-component initial-data programs (stack bytecode compiled from the
 * reference's expression AST by initdev.py; d_code / d_consts on the
 * device, comp_off[ncomp+1] on the host) at every cell centre (origin[dim]
 * + (i + 0.5) delta) of `ninst` samples (random vectors d_vecs, nrand per
 * sample), convert primitive Euler data to conserved, and write the padded
 * batch buffer `out` (ninst instances, ghosts zeroed).  d_bad[ninst *
 * (ncomp + 2)] receives the lowest flat cell of: a non-finite component c,
 * a non-positive primitive state (slot ncomp), an unphysical state (slot
 * ncomp + 1); ~0 when none.  sin / cos / exp / pow are CUDA's: rounding-level
 * parity with numpy, IEEE + - * / sqrt bitwise. */
int fvb_init_eval(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, const double* origin,
                  const int32_t* d_code, const int32_t* comp_off, const double* d_consts, int max_depth,
                  int primitive, const double* d_vecs, int nrand, int ninst, double* out,
                  unsigned long long* d_bad);

/* parallel.py:185-254 halo slabs: pack the g-thick interior slab next to
 * face (axis, side) into a contiguous buffer / unpack a received slab into
 * the ghost region of that face.  Slabs span the full padded extent of the
 * other axes (corners propagate in sequential-axis mode). */
int fvb_halo_pack(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, const double* u,
                  int axis, int side, double* buf);
int fvb_halo_unpack(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, double* u,
                    int axis, int side, const double* buf);
int64_t fvb_halo_count(const fvb_scheme* s, int axis);

/* numerics.py:133-196 rusanov_flux / hllc_flux (FLUX_FUNCTIONS, the
 * reference's flux registry seam, numerics.py:199-206) on n face pairs:
 * uL, uR, F are (ncomp, n) component-major device arrays.  Uses s->dim,
 * ncomp, eq, flux, gamma, adv, arith.  FVB_E_UNPHYSICAL for a degenerate
 * HLLC wave fan (numerics.py:166-167), FVB_E_CONFIG for HLLC on a scalar law
 * (numerics.py:150-151). */
int fvb_face_flux(fvb_ctx* ctx, const fvb_scheme* s, int axis, const double* uL, const double* uR, int64_t n,
                  double* F);
/* numerics.py:64-87 weno_weights + weno_face_value, elementwise over n
 * stencils (um, uc, up): w0, w1 (nullable) and the downwind face value
 * (nullable).  s->recon selects WENO2/WENO3 ideal weights, s->weno_eps the
 * epsilon; exact arithmetic follows the reference op by op. */
int fvb_weno(fvb_ctx* ctx, const fvb_scheme* s, const double* um, const double* uc, const double* up, int64_t n,
             double* w0, double* w1, double* face);

#ifdef __cplusplus
}
#endif
#endif /* FVB200_H */
