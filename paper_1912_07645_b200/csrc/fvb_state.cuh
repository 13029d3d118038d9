// Device-resident step state and the step-finalisation logic shared by the
// stage kernels and the standalone wave-speed kernel.
//
// One FvbState per instance (a batched MC ensemble runs one instance per
// sample).  The loop control replicates run_simulation (solver.py:219-245)
// and run_parallel's n_steps mode (parallel.py:490-520) exactly, on device,
// so no host round trip is needed per step.
#pragma once
#include <cstdint>
#include "../../include/fvb200.h"
#include "fvb_common.cuh"

namespace fvb {

constexpr long long kNone = 0x7fffffffffffffffLL;

struct FvbState {
  double t;                  // simulated time
  double dt;                 // dt of the step in flight (valid while !done)
  long long step;            // accepted steps
  int done;                  // no further step runs
  int err;                   // FVB_* status of the run (0 = ok)
  int errsub;                // FVB_SUB_* detail
  int pad0;
  long long errcell;         // flat index for messages (see host)
  unsigned long long smax[3];  // per-axis wave-speed maxima (IEEE bits, >= 0)
  long long bad_nonfinite;   // min ((c*nz+z)*ny+y)*nx+x over non-finite values
  long long bad_unphys;      // min (z*ny+y)*nx+x over unphysical cells
  long long stage_err;       // min over (stage<<42 | kind<<40 | cell)
  unsigned int blocks_done;  // last-block-done counter
  unsigned int pad1;
};

// Loop-control parameters (uniform over instances).
struct LoopCtl {
  int mode;          // FVB_MODE_T_END or FVB_MODE_FIXED
  int dim;
  double t_end;
  double cfl;
  long long max_steps;  // T_END: <0 = unlimited; FIXED: n_steps
  double deltas[3];
  double2* log;      // per instance ring: log[inst*log_cap + (step-1) % log_cap] = (t, dt)
  long long log_cap;
};

__device__ __forceinline__ double bits_to_d(unsigned long long b) { return __longlong_as_double((long long)b); }

// Single-thread step finalisation.  post=true: called once a step's last
// stage completed; post=false: called after the initial wave-speed pass.
__device__ inline void finalize_step(FvbState* st, const LoopCtl& L, int inst, bool post,
                                     bool init_check) {
  volatile FvbState* vs = st;
  bool stop = false;
  if (post) {
    const double dt = vs->dt;
    const double t = vs->t + dt;                 // solver.py:230
    const long long step = vs->step + 1;          // solver.py:229
    vs->t = t;
    vs->step = step;
    if (L.log && L.log_cap > 0) L.log[inst * L.log_cap + (step - 1) % L.log_cap] = make_double2(t, dt);
    const long long se = vs->stage_err;
    const long long nf = vs->bad_nonfinite;
    const long long up = vs->bad_unphys;
    if (se != kNone) {
      const int kind = (int)((se >> 40) & 3);
      vs->err = kind == 0 ? FVB_E_SIMULATION : FVB_E_UNPHYSICAL;
      vs->errsub = kind == 0 ? FVB_SUB_STAGE_UNPHYSICAL : FVB_SUB_HLLC_DEGENERATE;
      vs->errcell = se & ((1LL << 40) - 1);
      stop = true;
    } else if (nf != kNone) {                       // solver.py:231-238
      vs->err = FVB_E_SIMULATION;
      vs->errsub = FVB_SUB_NONFINITE;
      vs->errcell = nf;
      stop = true;
    } else if (L.mode == FVB_MODE_T_END && up != kNone) {  // solver.py:239-242
      vs->err = FVB_E_SIMULATION;
      vs->errsub = FVB_SUB_POST_UNPHYSICAL;
      vs->errcell = up;
      stop = true;
    }
  } else if (vs->bad_unphys != kNone) {
    if (L.mode == FVB_MODE_T_END && init_check) {  // solver.py:211-212
      vs->err = FVB_E_SIMULATION;
      vs->errsub = FVB_SUB_INIT_UNPHYSICAL;
    } else {                                       // wave_speed_maxima check=True
      vs->err = FVB_E_UNPHYSICAL;
      vs->errsub = FVB_SUB_SPEED_UNPHYSICAL;
    }
    vs->errcell = vs->bad_unphys;
    stop = true;
  }
  const bool t_control = L.mode != FVB_MODE_FIXED;
  if (!stop && post && L.mode != FVB_MODE_T_END && vs->bad_unphys != kNone) {
    // run_parallel checks only finiteness after a step (parallel.py:518-519);
    // the next iteration's wave_speed_maxima(check=True) raises
    // (equations.py:118-119) -- if there is a next iteration
    const bool more = t_control ? (vs->t < L.t_end && !(L.t_end - vs->t <= 1e-14 * L.t_end))
                                : (vs->step < L.max_steps);
    if (more) {
      vs->err = FVB_E_UNPHYSICAL;
      vs->errsub = FVB_SUB_SPEED_UNPHYSICAL;
      vs->errcell = vs->bad_unphys;
      stop = true;
    }
  }
  double rem = 0.0;
  if (!stop) {
    const double t = vs->t;
    if (t_control) {
      if (!(t < L.t_end)) stop = true;             // solver.py:219 / parallel.py:495
      rem = L.t_end - t;                           // solver.py:220
      if (!stop && rem <= 1e-14 * L.t_end) stop = true;
      if (!stop && L.max_steps >= 0 && vs->step >= L.max_steps) stop = true;
    } else {
      if (vs->step >= L.max_steps) stop = true;    // parallel.py:491-493
    }
  }
  if (!stop) {
    double denom = 0.0;                            // solver.py:141-143
    for (int k = 0; k < L.dim; ++k) denom += bits_to_d(vs->smax[k]) / L.deltas[k];
    if (denom == 0.0) {
      vs->err = FVB_E_STATIC;
      vs->errsub = FVB_SUB_NONE;
      stop = true;
    } else {
      double dt = L.cfl / denom;
      if (t_control) dt = (rem < dt) ? rem : dt;  // min(dt, remaining)
      vs->dt = dt;
    }
  }
  if (stop) vs->done = 1;
  for (int k = 0; k < 3; ++k) vs->smax[k] = 0ull;
  vs->bad_nonfinite = kNone;
  vs->bad_unphys = kNone;
  vs->stage_err = kNone;
  vs->blocks_done = 0u;
  __threadfence();
}

// Cross-rank step finalisation (process-per-GPU decomposition): the caller
// all-reduces (MAX) what export wrote -- [maxima (dim), hard error, unphysical]
// -- and every rank finalises with the same global values, so t, dt and the
// stop decision agree on all ranks (parallel.py:498-501).
__device__ inline void export_step(const FvbState* st, int dim, double* out) {
  const volatile FvbState* vs = st;
  for (int k = 0; k < dim; ++k) out[k] = bits_to_d(vs->smax[k]);
  out[dim] = (vs->stage_err != kNone || vs->bad_nonfinite != kNone) ? 1.0 : 0.0;
  out[dim + 1] = vs->bad_unphys != kNone ? 1.0 : 0.0;
}

__device__ inline void finalize_global(FvbState* st, const LoopCtl& L, const double* g, bool post) {
  volatile FvbState* vs = st;
  // steps enqueued past the end (the host polls only every few steps) leave
  // the finished state untouched, like the no-op stage kernels before them
  if (vs->done) return;
  for (int k = 0; k < L.dim; ++k) vs->smax[k] = (unsigned long long)__double_as_longlong(g[k]);
  const bool local_hard = vs->stage_err != kNone || vs->bad_nonfinite != kNone;
  if (g[L.dim] != 0.0 && !local_hard) {  // another rank failed this step
    if (post) {
      vs->t = vs->t + vs->dt;
      vs->step = vs->step + 1;
    }
    vs->err = FVB_E_SIMULATION;
    vs->errsub = FVB_SUB_REMOTE;
    vs->errcell = -1;
    vs->done = 1;
    return;
  }
  if (g[L.dim + 1] != 0.0 && vs->bad_unphys == kNone) vs->bad_unphys = kNone - 1;  // remote cell
  finalize_step(st, L, 0, post, true);
}

// Kernel parameters of one stage launch (identical in both arithmetic modes).
struct StageParams {
  const double* us;   // stage input u^(s) (stencil reads)
  const double* un;   // u^n (pointwise, RK combination)
  double* out;        // stage output (may alias un)
  FvbState* st;       // per-instance state (dt, done, error slots)
  int64_t n[3];
  int bc[3];
  int g;
  int64_t origin, sy, sz, sc, si;
  double dd[3];       // deltas
  double id[3];       // 1/delta
  int divd[3];        // 1: divide by delta (exact mode, delta not a power of 2)
  Phys P;
  int kind;           // 0: L  1: us+dt*L  2: RK2 final  3: RK3 stage 2  4: RK3 final
  int final_stage;    // 1: post-step checks + wave-speed maxima + finalize
  int check_input;    // 1: stage-start physical check of u^(s) (solver.py:90-93); 0 when the
                      //    previous step's post-check already covered it (stage 1 of a run)
  int stage_idx;      // stage number within the step (error ordering)
  int chunks;         // chunks along the march axis
  int H;              // rows per chunk
  int64_t row_lo;     // march-axis cell range computed by this launch: [row_lo, row_hi)
  int64_t row_hi;     // (inner box / shell slabs of the overlap schedule, parallel.py:288-361)
  int64_t x_lo, x_hi; // in-plane cell ranges of this launch (x; y in 3D): the inner box / shells of
  int64_t y_lo, y_hi; // a split in-plane axis.  Honoured by the ring, pair and 3D all-interior kernels.
  double* peer_lo;    // fused halo exchange (decomposed run, march axis split): the low / high
  double* peer_hi;    // neighbour's copy of `out` (peer memory, interior origin); cells of the first /
  int64_t peer_shift; // last g march rows are also stored there, shifted by n_march * march stride
  int64_t n_march;
  unsigned nblocks;   // blocks per state (finalize counter)
  int shared_state;   // 1: all instances are subdomains of one run (one FvbState)
  int defer_finalize; // 1: leave maxima/flags in the state; the caller reduces them
                      //    across ranks and calls fvb_run_finalize
  int ni;             // instances per block (2D ring kernel, scalar laws); 0/1 = one
  int variant;        // 1D/2D kernel: 0 = warp strip, 1 = shared-memory tile
  LoopCtl ctl;
};

// Device initial-data program (fvb_aux.cu init_eval_kernel, initdev.py)
struct InitArgs {
  const int* code;     // all components' programs back to back; word = op | (arg << 8)
  const double* k;     // constants
  int off[9];          // program c = code[off[c] .. off[c+1])
  int ncomp, dim, primitive, euler, nrand;
  double origin[3], delta[3], gamma;
  int64_t n[3];
};

}  // namespace fvb
