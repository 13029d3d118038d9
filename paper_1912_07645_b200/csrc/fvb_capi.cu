// C ABI of the B200 finite-volume hot path (include/fvb200.h).
//
// Owns: the context (device, stream, scratch, error text), the
// device-resident run loop (CUDA-graph batches of whole SSP-RK steps with dt,
// t and the stop flag kept in device memory), and the dispatch into the two
// compiled arithmetic modes (namespace exact: bitwise == reference; fast).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/fvb200.h"
#include "fvb_state.cuh"

namespace fvb {
namespace exact {
int launch_face_flux(int dim, int eq, int flux, const Phys& P, int axis, const double* uL, const double* uR,
                     int64_t n, double* F, unsigned long long* err, cudaStream_t s);
int launch_weno(int recon, double eps, const double* um, const double* uc, const double* up, int64_t n, double* w0,
                double* w1, double* face, cudaStream_t s);
int launch_stage(int dim, int eq, int flux, int recon, const StageParams& p, dim3 grid, cudaStream_t s);
int launch_speed(int dim, int eq, const StageParams& p, int finalize, dim3 grid, cudaStream_t s);
void stage_block(int dim, int eq, int variant, int& nt, int& nty);
}  // namespace exact
namespace fast {
int launch_face_flux(int dim, int eq, int flux, const Phys& P, int axis, const double* uL, const double* uR,
                     int64_t n, double* F, unsigned long long* err, cudaStream_t s);
int launch_weno(int recon, double eps, const double* um, const double* uc, const double* up, int64_t n, double* w0,
                double* w1, double* face, cudaStream_t s);
int launch_stage(int dim, int eq, int flux, int recon, const StageParams& p, dim3 grid, cudaStream_t s);
int launch_speed(int dim, int eq, const StageParams& p, int finalize, dim3 grid, cudaStream_t s);
void stage_block(int dim, int eq, int variant, int& nt, int& nty);
}  // namespace fast
// fvb_aux.cu
int launch_fill_axis(const fvb_scheme& s, const fvb_layout& L, double* u, int ninst, int axis, cudaStream_t st);
int launch_halo(const fvb_scheme& s, const fvb_layout& L, double* u, int axis, int side, double* buf,
                int unpack, cudaStream_t st);
int64_t halo_count(const fvb_scheme& s, int axis);
int launch_moments_push(const fvb_scheme& s, const fvb_layout& L, const double* u, int inst, int nbatch, double* mean,
                        double* m2, int64_t count_before, cudaStream_t st);
int launch_moments_merge(double* ma, double* m2a, int64_t ca, const double* mb, const double* m2b, int64_t cb,
                         int64_t n, cudaStream_t st);
int launch_structure(const fvb_scheme& s, const fvb_layout& L, const double* u, int inst, int comp, double p,
                     int H, double* d_sums, double* d_partials, int nblocks, cudaStream_t st);
int structure_blocks(const fvb_scheme& s);
int launch_init_eval(const InitArgs& A, const fvb_layout& L, const double* vecs, int ninst, double* out,
                     unsigned long long* bad, cudaStream_t st);
int launch_halo_instances(const fvb_scheme& s, const fvb_layout& L, double* u, int ninst, const int* ranks,
                          const int* periodic, cudaStream_t st);
int launch_export(const FvbState* st, int dim, double* out, cudaStream_t s);
int launch_finalize_global(FvbState* st, const LoopCtl& L, const double* g, int post, cudaStream_t s);
}  // namespace fvb

using fvb::FvbState;
using fvb::LoopCtl;
using fvb::StageParams;

struct RunPlan {
  fvb_scheme s;
  fvb_layout L;
  double* bufs[3];
  int ninst;
  int mode;
  int64_t max_steps;
  int64_t steps_enqueued;
  StageParams stage[3];  // per stage of a step (RK1 uses [0] with ping-pong)
  int nstages;
  dim3 grid;
  int active;
  int external;      // cross-rank reduce driven by the caller (fvb_run_stage/export/finalize)
  int topo;          // instances are the subdomains of one decomposed run
  int ranks[3];
  int periodic[3];
  double* peer[2][3];  // fused halo exchange: the low / high march-axis neighbour's bufs[k] (peer memory)
  int peer_on;
};

struct fvb_ctx {
  int device;
  cudaStream_t stream;      // stream all work is issued on
  cudaStream_t own_stream;  // created when the caller passes the legacy NULL stream

  char msg[1024];
  FvbState* d_state;  // run state, one per instance
  int state_cap;
  FvbState* d_scratch_state;  // for single-shot calls
  double2* d_log;
  int64_t log_cap_alloc;  // allocated (t,dt) entries
  int64_t log_stride;     // entries per instance for the current run (0 = no log)
  double* d_partials;
  int64_t partials_cap;
  RunPlan plan;
  int topo_pending;
  int external_pending;
  int topo_ranks[3];
  int topo_periodic[3];
  cudaGraphExec_t graph;
  int graph_steps;
  int graph_parity_ok;
  int64_t launches;
};

static int set_err(fvb_ctx* ctx, int code, const char* fmt, ...) {
  if (ctx) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(ctx->msg, sizeof(ctx->msg), fmt, ap);
    va_end(ap);
  }
  return code;
}

#define CUDA_TRY(ctx, call)                                                              \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return set_err(ctx, FVB_E_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

static int check_launch(fvb_ctx* ctx, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(ctx, FVB_E_CUDA, "%s launch failed: %s", what, cudaGetErrorString(e));
  return FVB_OK;
}

static int validate(fvb_ctx* ctx, const fvb_scheme* s) {
  if (!s) return set_err(ctx, FVB_E_CONFIG, "null scheme");
  if (s->dim < 1 || s->dim > 3) return set_err(ctx, FVB_E_CONFIG, "dim must be 1, 2 or 3, got %d", s->dim);
  if (s->eq < 0 || s->eq > 2) return set_err(ctx, FVB_E_CONFIG, "unknown equation kind %d", s->eq);
  const int nc = s->eq == FVB_EQ_EULER ? s->dim + 2 : 1;
  if (s->ncomp != nc) return set_err(ctx, FVB_E_CONFIG, "ncomp %d does not match the equation (%d)", s->ncomp, nc);
  if (s->flux == FVB_FLUX_HLLC && s->eq != FVB_EQ_EULER)
    return set_err(ctx, FVB_E_CONFIG, "HLLC flux requires the Euler equations");
  if (s->rk_order < 1 || s->rk_order > 3)
    return set_err(ctx, FVB_E_CONFIG, "rk_order must be 1, 2 or 3, got %d", s->rk_order);
  const int radius = s->recon == FVB_RECON_NONE ? 1 : 2;
  for (int k = 0; k < 3; ++k) {
    if (k >= s->dim) continue;
    if (s->cells[k] < 1) return set_err(ctx, FVB_E_CONFIG, "all cell counts must be >= 1");
    if (s->bc[k] == FVB_BC_PERIODIC && s->cells[k] < radius)
      return set_err(ctx, FVB_E_CONFIG, "periodic axis %d needs cells >= %d", k, radius);
    if (s->bc[k] == FVB_BC_HALO && s->ghost < radius)
      return set_err(ctx, FVB_E_CONFIG, "ghost_width %d too small for reconstruction radius %d", s->ghost, radius);
  }
  return FVB_OK;
}

// Instance count and extent checks shared by the stage entry points: the
// single-shot calls use a 4096-entry scratch state, and the 2D ring kernel
// addresses one instance (all components, plus the batched instances of a
// block) with 32-bit element offsets.
static int validate_instances(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, int ninst, bool scratch) {
  if (ninst < 1) return set_err(ctx, FVB_E_CONFIG, "ninst must be >= 1");
  if (scratch && ninst > 4096) return set_err(ctx, FVB_E_CONFIG, "too many instances (%d > 4096)", ninst);
  if (lay && s->dim == 3 && (s->cells[0] + 2 * s->ghost) * (s->cells[1] + 2 * s->ghost) * (s->cells[2] + 2 * s->ghost) >= (int64_t(1) << 31))
    return set_err(ctx, FVB_E_CONFIG, "3D instance component exceeds the 32-bit kernel offsets (2^31 cells)");
  if (lay && s->dim == 2) {
    const int64_t g = s->ghost;
    const int64_t span = (int64_t)(s->ncomp - 1) * lay->sc + (s->cells[1] + 2 * g) * lay->sy + s->cells[0] + 2 * g;
    const int64_t batch = s->ncomp == 1 ? 3 * lay->si : 0;  // up to 4 instances per block (scalar laws)
    if (span + batch >= (int64_t(1) << 31))
      return set_err(ctx, FVB_E_CONFIG, "2D instance of %lld elements exceeds the 32-bit kernel offsets",
                     (long long)(span + batch));
  }
  return FVB_OK;
}

static bool is_pow2(double d) {
  int e;
  const double m = std::frexp(d, &e);
  return m == 0.5;
}

// Fill the geometry / physics part of a StageParams.
static StageParams base_params(const fvb_scheme& s, const fvb_layout& L) {
  StageParams p;
  std::memset(&p, 0, sizeof(p));
  for (int k = 0; k < 3; ++k) {
    p.n[k] = k < s.dim ? s.cells[k] : 1;
    p.bc[k] = k < s.dim ? s.bc[k] : FVB_BC_PERIODIC;
    p.dd[k] = k < s.dim ? s.deltas[k] : 1.0;
    p.id[k] = 1.0 / p.dd[k];
    p.divd[k] = is_pow2(p.dd[k]) ? 0 : 1;
  }
  p.g = s.ghost;
  p.origin = L.origin;
  p.sy = L.sy;
  p.sz = L.sz;
  p.sc = L.sc;
  p.si = L.si;
  p.P.gamma = s.gamma;
  p.P.gm1 = s.gamma - 1.0;
  p.P.eps = s.weno_eps;
  for (int k = 0; k < 3; ++k) p.P.adv[k] = s.adv[k];
  p.check_input = 1;
  p.ctl.dim = s.dim;
  p.ctl.cfl = s.cfl;
  p.ctl.t_end = s.t_end;
  for (int k = 0; k < 3; ++k) p.ctl.deltas[k] = p.dd[k];
  return p;
}

static int sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
  return n;
}

// Resident blocks per SM of the stage kernel `p` selects (register and
// shared-memory limits of the compiled kernel, queried from the runtime).
// One grid serves every stage of a step, so take the most constrained of
// the stage shapes (first / middle / final stage).
static int stage_occupancy(const fvb_scheme& s, const StageParams& p) {
  static const int shapes[4][2] = {{1, 0}, {3, 0}, {4, 1}, {1, 1}};  // (kind, final_stage)
  int best = 0;
  for (const auto& sh : shapes) {
    StageParams q = p;
    q.H = std::max(q.H, 16);
    q.kind = sh[0];
    q.final_stage = sh[1];
    const int n = s.arith == FVB_ARITH_FAST
                      ? fvb::fast::launch_stage(s.dim, s.eq, s.flux, s.recon, q, dim3(0, 0, 0), 0)
                      : fvb::exact::launch_stage(s.dim, s.eq, s.flux, s.recon, q, dim3(0, 0, 0), 0);
    if (n > 0) best = best == 0 ? n : std::min(best, n);
  }
  return best;
}

// Grid of the stage kernel; fills chunks / H / nblocks.  xr / yr: optional
// in-plane cell ranges [lo, hi) (x; y in 3D) of this launch.
static dim3 stage_grid(const fvb_scheme& s, StageParams& p, int ninst, int64_t row_lo = 0, int64_t row_hi = -1,
                       const int64_t* xr = nullptr, const int64_t* yr = nullptr, int force_variant = -1) {
  int nt, nty;
  const char* kv = getenv("FVB_KERNEL");
  // 2D default: the pair kernel (two x-columns per thread, DESIGN.md
  // section 3) in fast mode, the cp.async ring kernel in exact mode.
  // FVB_KERNEL=ring / pair / tile / strip select explicitly.
  p.variant = (s.dim == 2 && s.arith == FVB_ARITH_FAST) ? 3 : 2;
  if (kv && std::strcmp(kv, "ring") == 0) p.variant = 2;
  // 3D default: the all-interior-rows ring kernel in fast mode; exact mode
  // keeps the round-1 ring3 kernel (measured faster with the IEEE sequences)
  if (s.dim == 3 && p.variant == 2 && s.arith == FVB_ARITH_FAST) p.variant = 4;
  if (kv && std::strcmp(kv, "ring3i") == 0 && s.dim == 3) p.variant = 4;
  if (kv && std::strcmp(kv, "ring3") == 0) p.variant = 2;
  if (kv && std::strcmp(kv, "strip") == 0) p.variant = 0;
  if (kv && std::strcmp(kv, "tile") == 0) p.variant = 1;
  if (kv && std::strcmp(kv, "pair") == 0) p.variant = 3;
  if (s.dim == 1 && p.variant >= 2) p.variant = 1;
  if (p.variant == 3 && s.dim != 2) p.variant = 2;  // pair kernel: 2D only
  if (force_variant >= 0) p.variant = force_variant;
  if (s.arith == FVB_ARITH_FAST) fvb::fast::stage_block(s.dim, s.eq, p.variant, nt, nty);
  else fvb::exact::stage_block(s.dim, s.eq, p.variant, nt, nty);
  p.x_lo = xr ? xr[0] : 0;
  p.x_hi = xr ? xr[1] : p.n[0];
  p.y_lo = yr ? yr[0] : 0;
  p.y_hi = yr ? yr[1] : p.n[1];
  const int64_t strips = std::max<int64_t>(1, (p.x_hi - p.x_lo + (nt - 2) - 1) / (nt - 2));
  // batched scalar ensembles on the 2D ring kernel: two instances per block
  p.ni = 1;
  if (s.dim == 2 && p.variant == 2 && s.ncomp == 1 && ninst % 2 == 0 && !p.shared_state) {
    const char* e = getenv("FVB_RING_NI");
    const int want = e ? atoi(e) : 2;
    p.ni = (want == 4 && ninst % 4 == 0) ? 4 : (want == 1 ? 1 : 2);
  }
  const int nig = ninst / p.ni;  // instance groups along grid z
  dim3 g(1, 1, 1);
  g.x = (unsigned)strips;
  int64_t H = 1, chunks = 1;
  if (s.dim >= 2) {
    const int64_t n_march = p.n[s.dim - 1];
    if (row_hi < 0) row_hi = n_march;
    p.row_lo = row_lo;
    p.row_hi = row_hi;
    const int64_t nm = std::max<int64_t>(1, row_hi - row_lo);
    int64_t ytiles = 1;
    if (s.dim == 3) ytiles = std::max<int64_t>(1, (p.y_hi - p.y_lo + (nty - 2) - 1) / (nty - 2));
    // resident blocks per SM (register-limited) and waves of blocks: one
    // wave keeps the march long (fewer redundant halo rows per chunk)
    int64_t per_sm = s.dim == 3 ? 2 : (p.variant == 0 ? 4 : 512 / nt);  // 16 warps/SM at 128 registers
    {
      const int occ = stage_occupancy(s, p);  // what the compiled kernel actually fits
      if (occ > 0) per_sm = occ;
    }
    int64_t waves = 1;
    if (const char* e = getenv("FVB_BLOCKS_PER_SM")) per_sm = std::max(1, atoi(e));
    if (const char* e = getenv("FVB_WAVES")) waves = std::max(1, atoi(e));
    const int64_t slots = (int64_t)sm_count() * per_sm;
    if (getenv("FVB_DEBUG_GRID")) fprintf(stderr, "fvb stage grid: %lld resident blocks per SM\n", (long long)per_sm);
    const int64_t base = strips * ytiles * nig;
    int64_t want_chunks = 1;
    if (getenv("FVB_WAVES")) {
      want_chunks = (slots * waves + base - 1) / base;
    } else {
      // march chunks: minimise (waves of resident blocks) x (rows per chunk +
      // the 2 extra rows a chunk marches), i.e. wave quantisation against
      // redundant halo rows (3D 256^3: 387 tiles on 296 slots -> 3 chunks)
      int64_t best = -1;
      for (int64_t c = 1; c <= std::max<int64_t>(1, nm / 4); ++c) {
        const int64_t w = (base * c + slots - 1) / slots;
        const int64_t cost = w * ((nm + c - 1) / c + 2);
        if (best < 0 || cost < best) { best = cost; want_chunks = c; }
        if (w > 64) break;
      }
    }
    want_chunks = std::max<int64_t>(1, std::min<int64_t>(want_chunks, nm));
    H = (nm + want_chunks - 1) / want_chunks;
    const char* env = getenv("FVB_MARCH_ROWS");
    if (env && atoi(env) > 0) H = atoi(env);
    // the per-block row-offset table lives in shared memory: cap the march
    // length (more chunks instead) so it stays small at any grid size
    H = std::max<int64_t>(4, std::min<int64_t>(std::min<int64_t>(H, nm), 2048));
    chunks = (nm + H - 1) / H;
    if (s.dim == 2) {
      g.y = (unsigned)chunks;
      g.z = nig;
    } else {
      g.y = (unsigned)ytiles;
      g.z = (unsigned)(chunks * ninst);
    }
  } else {
    g.z = ninst;
    p.row_lo = 0;
    p.row_hi = 1;
  }
  p.H = (int)H;
  p.chunks = (int)chunks;
  if (getenv("FVB_DEBUG_GRID"))
    fprintf(stderr, "fvb stage grid: dim %d variant %d grid (%u,%u,%u) H %lld chunks %lld sms %d\n", s.dim, p.variant,
            g.x, g.y, g.z, (long long)H, (long long)chunks, sm_count());
  p.nblocks = (unsigned)(g.x * g.y * (s.dim == 3 ? chunks : 1) * (s.dim == 2 ? chunks : 1));
  if (s.dim == 2) p.nblocks = (unsigned)(g.x * chunks);
  if (s.dim == 3) p.nblocks = (unsigned)(g.x * g.y * chunks);
  if (s.dim == 1) p.nblocks = g.x;
  return g;
}

static int do_stage(fvb_ctx* ctx, const fvb_scheme& s, const StageParams& p, dim3 grid) {
  int r = s.arith == FVB_ARITH_FAST ? fvb::fast::launch_stage(s.dim, s.eq, s.flux, s.recon, p, grid, ctx->stream)
                                    : fvb::exact::launch_stage(s.dim, s.eq, s.flux, s.recon, p, grid, ctx->stream);
  if (r != 0) return set_err(ctx, FVB_E_CONFIG, "unsupported scheme combination");
  ctx->launches++;
  return check_launch(ctx, "stage_kernel");
}

static int do_speed(fvb_ctx* ctx, const fvb_scheme& s, const StageParams& p, int finalize, int ninst) {
  const int64_t ncell = p.n[0] * p.n[1] * p.n[2];
  int64_t blocks = (ncell + 255) / 256;
  blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)sm_count() * 8 / std::max(1, ninst) + 1));
  dim3 grid((unsigned)blocks, ninst, 1);
  int r = s.arith == FVB_ARITH_FAST ? fvb::fast::launch_speed(s.dim, s.eq, p, finalize, grid, ctx->stream)
                                    : fvb::exact::launch_speed(s.dim, s.eq, p, finalize, grid, ctx->stream);
  if (r != 0) return set_err(ctx, FVB_E_CONFIG, "unsupported dim");
  ctx->launches++;
  return check_launch(ctx, "speed_kernel");
}

static void init_state_host(FvbState& h) {
  std::memset(&h, 0, sizeof(h));
  h.bad_nonfinite = fvb::kNone;
  h.bad_unphys = fvb::kNone;
  h.stage_err = fvb::kNone;
}

static int ensure_state(fvb_ctx* ctx, int ninst) {
  if (ninst <= ctx->state_cap) return FVB_OK;
  if (ctx->d_state) cudaFree(ctx->d_state);
  ctx->d_state = nullptr;
  CUDA_TRY(ctx, cudaMalloc(&ctx->d_state, sizeof(FvbState) * ninst));
  ctx->state_cap = ninst;
  return FVB_OK;
}

static int reset_states(fvb_ctx* ctx, FvbState* d, int ninst, double dt) {
  std::vector<FvbState> h(ninst);
  for (auto& x : h) {
    init_state_host(x);
    x.dt = dt;
  }
  CUDA_TRY(ctx, cudaMemcpyAsync(d, h.data(), sizeof(FvbState) * ninst, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return FVB_OK;
}

static void destroy_graph(fvb_ctx* ctx) {
  if (ctx->graph) cudaGraphExecDestroy(ctx->graph);
  ctx->graph = nullptr;
}

static int ensure_log(fvb_ctx* ctx, int64_t n) {
  if (n <= ctx->log_cap_alloc) return FVB_OK;
  if (ctx->d_log) cudaFree(ctx->d_log);
  ctx->d_log = nullptr;
  CUDA_TRY(ctx, cudaMalloc(&ctx->d_log, sizeof(double2) * n));
  ctx->log_cap_alloc = n;
  return FVB_OK;
}

extern "C" {

int fvb_version(void) { return 1; }

int fvb_ctx_create(int device, void* stream, fvb_ctx** out) {
  if (!out) return FVB_E_CONFIG;
  fvb_ctx* ctx = new fvb_ctx;
  std::memset(ctx, 0, sizeof(*ctx));
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    *out = ctx;
    return set_err(ctx, FVB_E_CUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
  }
  // CUDA graphs cannot be captured on the legacy NULL stream.  A blocking
  // stream created here is implicitly ordered with NULL-stream work (torch's
  // default stream), so callers see ordinary stream semantics.
  e = cudaStreamCreate(&ctx->own_stream);
  if (e != cudaSuccess) {
    *out = ctx;
    return set_err(ctx, FVB_E_CUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
  }
  ctx->stream = stream ? (cudaStream_t)stream : ctx->own_stream;
  e = cudaMalloc(&ctx->d_scratch_state, sizeof(FvbState) * 4096);
  if (e != cudaSuccess) {
    *out = ctx;
    return set_err(ctx, FVB_E_CUDA, "cudaMalloc: %s", cudaGetErrorString(e));
  }
  *out = ctx;
  return FVB_OK;
}

int fvb_ctx_destroy(fvb_ctx* ctx) {
  if (!ctx) return FVB_OK;
  destroy_graph(ctx);
  if (ctx->d_state) cudaFree(ctx->d_state);
  if (ctx->d_scratch_state) cudaFree(ctx->d_scratch_state);
  if (ctx->d_log) cudaFree(ctx->d_log);
  if (ctx->d_partials) cudaFree(ctx->d_partials);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
  return FVB_OK;
}

int fvb_ctx_set_stream(fvb_ctx* ctx, void* stream) {
  cudaStream_t s = stream ? (cudaStream_t)stream : ctx->own_stream;
  if (ctx->stream != s) destroy_graph(ctx);
  ctx->stream = s;
  return FVB_OK;
}

int fvb_last_error(const fvb_ctx* ctx, char* buf, size_t n) {
  if (!ctx || !buf || n == 0) return FVB_E_CONFIG;
  std::snprintf(buf, n, "%s", ctx->msg);
  return FVB_OK;
}

int fvb_sync(fvb_ctx* ctx) {
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return FVB_OK;
}

int64_t fvb_launch_count(const fvb_ctx* ctx) { return ctx ? ctx->launches : 0; }

int fvb_fill_ghosts(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, double* u, int ninst) {
  int r = validate(ctx, s);
  if (r) return r;
  for (int axis = 0; axis < s->dim; ++axis) {
    if (s->bc[axis] == FVB_BC_PERIODIC && s->cells[axis] < s->ghost)
      return set_err(ctx, FVB_E_CONFIG, "periodic axis %d needs cells >= ghost_width (%lld < %d)", axis,
                     (long long)s->cells[axis], s->ghost);
    if (s->bc[axis] == FVB_BC_HALO) continue;
    fvb::launch_fill_axis(*s, *lay, u, ninst, axis, ctx->stream);
    ctx->launches++;
    r = check_launch(ctx, "fill_axis");
    if (r) return r;
  }
  return FVB_OK;
}

int fvb_wave_speed_maxima(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, const double* u, int ninst,
                          double* h_max) {
  int r = validate(ctx, s);
  if (r) return r;
  r = validate_instances(ctx, s, lay, ninst, true);
  if (r) return r;
  r = reset_states(ctx, ctx->d_scratch_state, ninst, 0.0);
  if (r) return r;
  StageParams p = base_params(*s, *lay);
  p.us = u;
  p.st = ctx->d_scratch_state;
  r = do_speed(ctx, *s, p, 0, ninst);
  if (r) return r;
  std::vector<FvbState> h(ninst);
  CUDA_TRY(ctx, cudaMemcpyAsync(h.data(), ctx->d_scratch_state, sizeof(FvbState) * ninst, cudaMemcpyDeviceToHost,
                                ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < ninst; ++i) {
    for (int k = 0; k < s->dim; ++k) {
      double d;
      std::memcpy(&d, &h[i].smax[k], 8);
      h_max[i * s->dim + k] = d;
    }
    if (h[i].bad_unphys != fvb::kNone)
      return set_err(ctx, FVB_E_UNPHYSICAL, "unphysical state at cell %lld (instance %d)",
                     (long long)h[i].bad_unphys, i);
  }
  return FVB_OK;
}

static int stage_error(fvb_ctx* ctx, const FvbState& h, int inst) {
  if (h.stage_err == fvb::kNone) return FVB_OK;
  const int kind = (int)((h.stage_err >> 40) & 3);
  const long long cell = h.stage_err & ((1LL << 40) - 1);
  if (kind == 0)
    return set_err(ctx, FVB_E_SIMULATION, "unphysical state in interior cell #%lld (instance %d)", cell, inst);
  return set_err(ctx, FVB_E_UNPHYSICAL, "degenerate HLLC wave fan (sL >= sR)");
}

int fvb_spatial_residual(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, const double* u, double* out,
                         int ninst) {
  int r = validate(ctx, s);
  if (r) return r;
  r = validate_instances(ctx, s, lay, ninst, true);
  if (r) return r;
  r = reset_states(ctx, ctx->d_scratch_state, ninst, 0.0);
  if (r) return r;
  StageParams p = base_params(*s, *lay);
  p.us = u;
  p.un = u;
  p.out = out;
  p.st = ctx->d_scratch_state;
  p.kind = 0;
  dim3 g = stage_grid(*s, p, ninst);
  r = do_stage(ctx, *s, p, g);
  if (r) return r;
  std::vector<FvbState> h(ninst);
  CUDA_TRY(ctx, cudaMemcpyAsync(h.data(), ctx->d_scratch_state, sizeof(FvbState) * ninst, cudaMemcpyDeviceToHost,
                                ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < ninst; ++i) {
    r = stage_error(ctx, h[i], i);
    if (r) return r;
  }
  return FVB_OK;
}

// Stage parameters of one SSP-RK step over buffers b (solver.py:164-173).
static int build_step(const fvb_scheme& s, const fvb_layout& L, double* const b[3], StageParams base,
                      StageParams out[3]) {
  const int rk = s.rk_order;
  for (int i = 0; i < 3; ++i) out[i] = base;
  if (rk == 1) {
    out[0].us = b[0]; out[0].un = b[0]; out[0].out = b[1]; out[0].kind = 1; out[0].final_stage = 1;
    out[0].stage_idx = 0;
    return 1;
  }
  if (rk == 2) {
    out[0].us = b[0]; out[0].un = b[0]; out[0].out = b[1]; out[0].kind = 1; out[0].stage_idx = 0;
    out[1].us = b[1]; out[1].un = b[0]; out[1].out = b[0]; out[1].kind = 2; out[1].final_stage = 1;
    out[1].stage_idx = 1;
    return 2;
  }
  out[0].us = b[0]; out[0].un = b[0]; out[0].out = b[1]; out[0].kind = 1; out[0].stage_idx = 0;
  out[1].us = b[1]; out[1].un = b[0]; out[1].out = b[2]; out[1].kind = 3; out[1].stage_idx = 1;
  out[2].us = b[2]; out[2].un = b[0]; out[2].out = b[0]; out[2].kind = 4; out[2].final_stage = 1;
  out[2].stage_idx = 2;
  return 3;
}

int fvb_ssp_rk_step(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, double* un, double* w1, double* w2,
                    int ninst, double dt) {
  int r = validate(ctx, s);
  if (r) return r;
  r = validate_instances(ctx, s, lay, ninst, true);
  if (r) return r;
  r = reset_states(ctx, ctx->d_scratch_state, ninst, dt);
  if (r) return r;
  StageParams base = base_params(*s, *lay);
  base.st = ctx->d_scratch_state;
  dim3 g = stage_grid(*s, base, ninst);
  double* b[3] = {un, w1, w2};
  StageParams st[3];
  const int ns = build_step(*s, *lay, b, base, st);
  for (int i = 0; i < ns; ++i) {
    st[i].final_stage = 0;  // ssp_rk_step has no post-step checks (solver.py:176-196)
    r = do_stage(ctx, *s, st[i], g);
    if (r) return r;
  }
  if (s->rk_order == 1) {
    // result is in w1: copy back into un (interior and ghosts alike)
    const int64_t total = (int64_t)ninst * (lay->si ? lay->si : (lay->sc * s->ncomp));
    CUDA_TRY(ctx, cudaMemcpyAsync(un, w1, sizeof(double) * total, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  std::vector<FvbState> h(ninst);
  CUDA_TRY(ctx, cudaMemcpyAsync(h.data(), ctx->d_scratch_state, sizeof(FvbState) * ninst, cudaMemcpyDeviceToHost,
                                ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < ninst; ++i) {
    r = stage_error(ctx, h[i], i);
    if (r) return r;
  }
  return FVB_OK;
}

// ---------------------------------------------------------------------------
// Device-resident run loop
// ---------------------------------------------------------------------------

static int do_halo(fvb_ctx* ctx, const double* us) {
  RunPlan& P = ctx->plan;
  if (!P.topo) return FVB_OK;
  if (fvb::launch_halo_instances(P.s, P.L, const_cast<double*>(us), P.ninst, P.ranks, P.periodic, ctx->stream))
    ctx->launches++;
  return check_launch(ctx, "halo_instances");
}

static int enqueue_step(fvb_ctx* ctx) {
  RunPlan& P = ctx->plan;
  if (P.s.rk_order == 1) {
    StageParams p = P.stage[0];
    const int par = (int)(P.steps_enqueued & 1);
    p.us = P.bufs[par];
    p.un = P.bufs[par];
    p.out = P.bufs[1 - par];
    int r = do_halo(ctx, p.us);
    if (r) return r;
    r = do_stage(ctx, P.s, p, P.grid);
    if (r) return r;
  } else {
    for (int i = 0; i < P.nstages; ++i) {
      int r = do_halo(ctx, P.stage[i].us);
      if (r) return r;
      r = do_stage(ctx, P.s, P.stage[i], P.grid);
      if (r) return r;
    }
  }
  P.steps_enqueued++;
  return FVB_OK;
}

int fvb_run_begin(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, double* bufs[3], int ninst, int mode,
                  int64_t max_steps) {
  int r = validate(ctx, s);
  if (r) return r;
  r = validate_instances(ctx, s, lay, ninst, false);
  if (r) return r;
  destroy_graph(ctx);
  r = ensure_state(ctx, ninst);
  if (r) return r;
  r = reset_states(ctx, ctx->d_state, ninst, 0.0);
  if (r) return r;
  RunPlan& P = ctx->plan;
  std::memset(&P, 0, sizeof(P));
  P.s = *s;
  P.L = *lay;
  for (int i = 0; i < 3; ++i) P.bufs[i] = bufs[i];
  P.ninst = ninst;
  P.mode = mode;
  P.max_steps = max_steps;
  P.topo = ctx->topo_pending;
  ctx->topo_pending = 0;
  P.external = ctx->external_pending;
  ctx->external_pending = 0;
  for (int k = 0; k < 3; ++k) {
    P.ranks[k] = ctx->topo_ranks[k];
    P.periodic[k] = ctx->topo_periodic[k];
  }
  if (P.topo) {
    int64_t nr = (int64_t)P.ranks[0] * P.ranks[1] * P.ranks[2];
    if (nr != ninst) return set_err(ctx, FVB_E_CONFIG, "topology has %lld ranks but %d instances", (long long)nr, ninst);
  }
  StageParams base = base_params(*s, *lay);
  base.st = ctx->d_state;
  base.shared_state = P.topo;
  base.ctl.mode = mode;
  base.ctl.max_steps = mode == FVB_MODE_FIXED ? max_steps : max_steps;
  base.ctl.log = ctx->log_stride > 0 ? ctx->d_log : nullptr;
  base.ctl.log_cap = ctx->log_stride;
  P.grid = stage_grid(*s, base, ninst);
  if (P.topo) base.nblocks *= (unsigned)ninst;  // one shared state counts every subdomain's blocks
  P.nstages = build_step(*s, *lay, P.bufs, base, P.stage);
  // stage 1 reads u^n, already checked by the initial pass / the previous
  // step's post-step check (physical, or wave_speed_maxima in run_parallel)
  P.stage[0].check_input = 0;
  if (P.external) P.stage[P.nstages - 1].defer_finalize = 1;
  P.active = 1;
  // initial wave-speed pass + first dt (solver.py:211-224)
  StageParams sp = base;
  sp.us = bufs[0];
  return do_speed(ctx, *s, sp, P.external ? 0 : 1, ninst);
}

int fvb_run_steps(fvb_ctx* ctx, int64_t n_steps) {
  RunPlan& P = ctx->plan;
  if (!P.active) return set_err(ctx, FVB_E_CONFIG, "fvb_run_steps without fvb_run_begin");
  const char* env = getenv("FVB_GRAPH_STEPS");
  int gs = ctx->graph_steps > 0 ? ctx->graph_steps : 16;
  if (env && atoi(env) >= 0) gs = atoi(env);
  if (P.s.rk_order == 1 && (gs & 1)) gs += 1;
  int64_t left = n_steps;
  if (P.s.rk_order == 1 && (P.steps_enqueued & 1) && left > 0) {
    int r = enqueue_step(ctx);
    if (r) return r;
    --left;
  }
  if (gs > 1 && left >= gs) {
    if (!ctx->graph) {
      cudaGraph_t graph;
      CUDA_TRY(ctx, cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
      const int64_t saved = P.steps_enqueued;
      const int64_t saved_l = ctx->launches;
      for (int i = 0; i < gs; ++i) {
        int r = enqueue_step(ctx);
        if (r) {
          cudaStreamEndCapture(ctx->stream, &graph);
          return r;
        }
      }
      P.steps_enqueued = saved;
      ctx->launches = saved_l;
      CUDA_TRY(ctx, cudaStreamEndCapture(ctx->stream, &graph));
      CUDA_TRY(ctx, cudaGraphInstantiate(&ctx->graph, graph, 0));
      cudaGraphDestroy(graph);
      ctx->graph_steps = gs;
    }
    while (left >= ctx->graph_steps) {
      CUDA_TRY(ctx, cudaGraphLaunch(ctx->graph, ctx->stream));
      P.steps_enqueued += ctx->graph_steps;
      ctx->launches += (int64_t)ctx->graph_steps * (P.s.rk_order == 1 ? 1 : P.nstages);
      left -= ctx->graph_steps;
    }
  }
  while (left > 0) {
    int r = enqueue_step(ctx);
    if (r) return r;
    --left;
  }
  return FVB_OK;
}

static int state_to_info(fvb_ctx* ctx, const FvbState& h, fvb_run_info* info) {
  info->t = h.t;
  info->dt = h.dt;
  info->steps = h.step;
  info->err = h.err;
  info->errsub = h.errsub;
  info->errcell = h.errcell;
  return FVB_OK;
}

int fvb_run_poll(fvb_ctx* ctx, fvb_run_info* h_info, int32_t* h_done) {
  RunPlan& P = ctx->plan;
  if (!P.active) return set_err(ctx, FVB_E_CONFIG, "fvb_run_poll without fvb_run_begin");
  std::vector<FvbState> h(P.ninst);
  CUDA_TRY(ctx, cudaMemcpyAsync(h.data(), ctx->d_state, sizeof(FvbState) * P.ninst, cudaMemcpyDeviceToHost,
                                ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < P.ninst; ++i) {
    if (h_info) state_to_info(ctx, h[i], h_info + i);
    if (h_done) h_done[i] = h[i].done;
  }
  return FVB_OK;
}

int fvb_run_read_log(fvb_ctx* ctx, double* h_log, int64_t per_instance) {
  RunPlan& P = ctx->plan;
  if (!P.active || ctx->log_stride <= 0) return set_err(ctx, FVB_E_CONFIG, "no active step log");
  if (per_instance != ctx->log_stride) return set_err(ctx, FVB_E_CONFIG, "log size mismatch");
  CUDA_TRY(ctx, cudaMemcpyAsync(h_log, ctx->d_log, sizeof(double2) * per_instance * P.ninst, cudaMemcpyDeviceToHost,
                                ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return FVB_OK;
}

int fvb_run_set_external_reduce(fvb_ctx* ctx, int on) {
  ctx->external_pending = on ? 1 : 0;
  return FVB_OK;
}

// Peer buffers of the stage's output (fused halo exchange, fvb_run_set_peers).
static void apply_peers(const RunPlan& P, StageParams& p) {
  p.peer_lo = p.peer_hi = nullptr;
  if (!P.peer_on) return;
  int k = -1;
  for (int i = 0; i < 3; ++i)
    if (P.bufs[i] == p.out) k = i;
  if (k < 0) return;
  const int march = P.s.dim - 1;
  p.n_march = P.s.cells[march];
  p.peer_shift = p.n_march * (P.s.dim == 2 ? P.L.sy : P.L.sz);
  if (P.peer[0][k]) p.peer_lo = P.peer[0][k] + P.L.origin;
  if (P.peer[1][k]) p.peer_hi = P.peer[1][k] + P.L.origin;
}

int fvb_run_set_peers(fvb_ctx* ctx, double* const* lo, double* const* hi) {
  RunPlan& P = ctx->plan;
  if (!P.active || !P.external) return set_err(ctx, FVB_E_CONFIG, "fvb_run_set_peers needs an external-reduce run");
  if (P.s.dim < 2) return set_err(ctx, FVB_E_CONFIG, "fused halo exchange needs a march axis (dim >= 2)");
  if (P.ninst != 1) return set_err(ctx, FVB_E_CONFIG, "fused halo exchange is per subdomain (ninst == 1)");
  if (P.s.bc[P.s.dim - 1] != FVB_BC_HALO)
    return set_err(ctx, FVB_E_CONFIG, "fused halo exchange: the march axis must be a halo (split) axis");
  for (int k = 0; k < 3; ++k) {
    P.peer[0][k] = lo ? lo[k] : nullptr;
    P.peer[1][k] = hi ? hi[k] : nullptr;
  }
  P.peer_on = (lo != nullptr) || (hi != nullptr);
  return FVB_OK;
}

int fvb_run_stage(fvb_ctx* ctx, int stage) {
  RunPlan& P = ctx->plan;
  if (!P.active || !P.external) return set_err(ctx, FVB_E_CONFIG, "fvb_run_stage needs an external-reduce run");
  if (stage < 0 || stage >= P.nstages) return set_err(ctx, FVB_E_CONFIG, "stage %d out of range", stage);
  StageParams p = P.stage[stage];
  if (P.s.rk_order == 1) {
    const int par = (int)(P.steps_enqueued & 1);
    p.us = P.bufs[par];
    p.un = P.bufs[par];
    p.out = P.bufs[1 - par];
  }
  apply_peers(P, p);
  int r = do_stage(ctx, P.s, p, P.grid);
  if (r) return r;
  if (stage == P.nstages - 1) P.steps_enqueued++;
  return FVB_OK;
}

int fvb_run_stage_rows(fvb_ctx* ctx, int stage, int64_t row_lo, int64_t row_hi, int last_part) {
  RunPlan& P = ctx->plan;
  if (!P.active || !P.external) return set_err(ctx, FVB_E_CONFIG, "fvb_run_stage_rows needs an external-reduce run");
  if (stage < 0 || stage >= P.nstages) return set_err(ctx, FVB_E_CONFIG, "stage %d out of range", stage);
  if (P.s.dim < 2) return set_err(ctx, FVB_E_CONFIG, "row ranges need a march axis (dim >= 2)");
  StageParams p = P.stage[stage];
  if (P.s.rk_order == 1) {
    const int par = (int)(P.steps_enqueued & 1);
    p.us = P.bufs[par];
    p.un = P.bufs[par];
    p.out = P.bufs[1 - par];
  }
  if (row_hi <= row_lo) return FVB_OK;
  dim3 g = stage_grid(P.s, p, P.ninst, row_lo, row_hi);
  apply_peers(P, p);
  int r = do_stage(ctx, P.s, p, g);
  if (r) return r;
  if (last_part && stage == P.nstages - 1) P.steps_enqueued++;
  return FVB_OK;
}

int fvb_run_stage_box(fvb_ctx* ctx, int stage, const int64_t* lo, const int64_t* hi, int last_part) {
  RunPlan& P = ctx->plan;
  if (!P.active || !P.external) return set_err(ctx, FVB_E_CONFIG, "fvb_run_stage_box needs an external-reduce run");
  if (stage < 0 || stage >= P.nstages) return set_err(ctx, FVB_E_CONFIG, "stage %d out of range", stage);
  if (P.s.dim < 2) return set_err(ctx, FVB_E_CONFIG, "cell boxes need a march axis (dim >= 2)");
  StageParams p = P.stage[stage];
  if (P.s.rk_order == 1) {
    const int par = (int)(P.steps_enqueued & 1);
    p.us = P.bufs[par];
    p.un = P.bufs[par];
    p.out = P.bufs[1 - par];
  }
  const int march = P.s.dim - 1;
  for (int k = 0; k < P.s.dim; ++k)
    if (lo[k] >= hi[k]) return FVB_OK;  // empty box
  const int64_t xr[2] = {lo[0], hi[0]};
  const int64_t yr[2] = {lo[1], hi[1]};
  dim3 g = stage_grid(P.s, p, P.ninst, lo[march], hi[march], xr, P.s.dim == 3 ? yr : nullptr);
  const bool partial_plane = lo[0] != 0 || hi[0] != P.s.cells[0] ||
                             (P.s.dim == 3 && (lo[1] != 0 || hi[1] != P.s.cells[1]));
  if (partial_plane && P.s.dim == 3 && p.variant == 2)
    // in-plane ranges: the 3D all-interior kernel (same arithmetic, bitwise
    // equal to ring3 in both modes) instead of ring3, which has none
    g = stage_grid(P.s, p, P.ninst, lo[march], hi[march], xr, yr, 4);
  const bool ranged = P.s.dim == 2 ? (p.variant == 2 || p.variant == 3) : p.variant == 4;
  if (partial_plane && !ranged)
    return set_err(ctx, FVB_E_CONFIG, "in-plane cell ranges need the ring / pair / 3D all-interior kernels");
  apply_peers(P, p);
  int r = do_stage(ctx, P.s, p, g);
  if (r) return r;
  if (last_part && stage == P.nstages - 1) P.steps_enqueued++;
  return FVB_OK;
}

int fvb_run_export(fvb_ctx* ctx, double* d_out) {
  RunPlan& P = ctx->plan;
  if (!P.active) return set_err(ctx, FVB_E_CONFIG, "no active run");
  fvb::launch_export(ctx->d_state, P.s.dim, d_out, ctx->stream);
  ctx->launches++;
  return check_launch(ctx, "export");
}

int fvb_run_finalize(fvb_ctx* ctx, const double* d_global, int post) {
  RunPlan& P = ctx->plan;
  if (!P.active) return set_err(ctx, FVB_E_CONFIG, "no active run");
  fvb::launch_finalize_global(ctx->d_state, P.stage[0].ctl, d_global, post, ctx->stream);
  ctx->launches++;
  return check_launch(ctx, "finalize");
}

int fvb_run_set_topology(fvb_ctx* ctx, const int32_t* ranks, const int32_t* periodic) {
  if (!ranks) {
    ctx->topo_pending = 0;
    return FVB_OK;
  }
  for (int k = 0; k < 3; ++k) {
    if (ranks[k] < 1) return set_err(ctx, FVB_E_CONFIG, "ranks per axis must be >= 1");
    ctx->topo_ranks[k] = ranks[k];
    ctx->topo_periodic[k] = periodic ? periodic[k] : 1;
  }
  ctx->topo_pending = 1;
  return FVB_OK;
}

int fvb_run_set_log(fvb_ctx* ctx, int64_t per_instance, int ninst) {
  if (per_instance <= 0) {
    ctx->log_stride = 0;
    return FVB_OK;
  }
  int r = ensure_log(ctx, per_instance * ninst);
  if (r) return r;
  ctx->log_stride = per_instance;
  return FVB_OK;
}

int fvb_run_end(fvb_ctx* ctx, fvb_run_info* h_info, double* h_log, int64_t log_cap) {
  RunPlan& P = ctx->plan;
  if (!P.active) return set_err(ctx, FVB_E_CONFIG, "fvb_run_end without fvb_run_begin");
  std::vector<FvbState> h(P.ninst);
  CUDA_TRY(ctx, cudaMemcpyAsync(h.data(), ctx->d_state, sizeof(FvbState) * P.ninst, cudaMemcpyDeviceToHost,
                                ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  int first_err = FVB_OK;
  for (int i = 0; i < P.ninst; ++i) {
    if (h_info) state_to_info(ctx, h[i], h_info + i);
    if (h[i].err && !first_err) first_err = h[i].err;
  }
  if (h_log && log_cap > 0 && ctx->d_log && ctx->log_stride > 0) {
    const int64_t cap = std::min<int64_t>(log_cap, ctx->log_stride);
    for (int i = 0; i < P.ninst; ++i) {
      CUDA_TRY(ctx, cudaMemcpyAsync(h_log + 2 * i * log_cap, ctx->d_log + i * ctx->log_stride,
                                    sizeof(double2) * cap, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  }
  P.active = 0;
  if (first_err) return set_err(ctx, first_err, "run failed (see run info)");
  return FVB_OK;
}

int fvb_run(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, double* bufs[3], int ninst, int mode,
            int64_t max_steps, double* h_log, int64_t log_cap, int graph_steps, fvb_run_info* h_info) {
  int r = ensure_log(ctx, log_cap > 0 ? log_cap * ninst : 0);
  if (r) return r;
  ctx->log_stride = (h_log && log_cap > 0) ? log_cap : 0;
  ctx->graph_steps = graph_steps;
  r = fvb_run_begin(ctx, s, lay, bufs, ninst, mode, max_steps);
  if (r) return r;
  RunPlan& P = ctx->plan;
  std::vector<FvbState> h(ninst);
  int64_t batch = graph_steps > 0 ? graph_steps : 16;
  for (;;) {
    CUDA_TRY(ctx, cudaMemcpyAsync(h.data(), ctx->d_state, sizeof(FvbState) * ninst, cudaMemcpyDeviceToHost,
                                  ctx->stream));
    CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    bool all_done = true;
    double est = 0;
    for (int i = 0; i < ninst; ++i) {
      if (!h[i].done) {
        all_done = false;
        if (mode == FVB_MODE_T_END && h[i].dt > 0) est = std::max(est, (s->t_end - h[i].t) / h[i].dt);
      }
    }
    if (all_done) break;
    int64_t n = batch;
    if (mode == FVB_MODE_FIXED) n = std::max<int64_t>(1, max_steps - P.steps_enqueued);
    else if (max_steps >= 0) n = std::max<int64_t>(1, std::min<int64_t>(n, max_steps - P.steps_enqueued));
    r = fvb_run_steps(ctx, n);
    if (r) return r;
  }
  r = fvb_run_end(ctx, h_info, h_log, log_cap);
  ctx->log_stride = 0;
  return r;
}

// ---------------------------------------------------------------------------
// UQ statistics and halo slabs (kernels in fvb_aux.cu)
// ---------------------------------------------------------------------------

int fvb_moments_push(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, const double* u, int inst,
                     double* mean, double* m2, int64_t count_before) {
  return fvb_moments_push_batch(ctx, s, lay, u, inst, 1, mean, m2, count_before);
}

int fvb_moments_push_batch(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, const double* u, int inst,
                           int nbatch, double* mean, double* m2, int64_t count_before) {
  if (nbatch < 1) return set_err(ctx, FVB_E_CONFIG, "nbatch must be >= 1");
  fvb::launch_moments_push(*s, *lay, u, inst, nbatch, mean, m2, count_before, ctx->stream);
  ctx->launches += (nbatch + 63) / 64;
  return check_launch(ctx, "moments_push");
}

int fvb_moments_merge(fvb_ctx* ctx, double* mean_a, double* m2_a, int64_t count_a, const double* mean_b,
                      const double* m2_b, int64_t count_b, int64_t n) {
  fvb::launch_moments_merge(mean_a, m2_a, count_a, mean_b, m2_b, count_b, n, ctx->stream);
  ctx->launches++;
  return check_launch(ctx, "moments_merge");
}

int fvb_structure_push(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, const double* u, int inst,
                       int comp, double p, int H, double* d_sums) {
  if (H < 0) return set_err(ctx, FVB_E_CONFIG, "max offset must be >= 0, got %d", H);
  const int nb = fvb::structure_blocks(*s);
  const int64_t need = (int64_t)nb * (H + 1) * s->dim;
  if (need > ctx->partials_cap) {
    if (ctx->d_partials) cudaFree(ctx->d_partials);
    ctx->d_partials = nullptr;
    CUDA_TRY(ctx, cudaMalloc(&ctx->d_partials, sizeof(double) * need));
    ctx->partials_cap = need;
  }
  fvb::launch_structure(*s, *lay, u, inst, comp, p, H, d_sums, ctx->d_partials, nb, ctx->stream);
  ctx->launches += 2;
  return check_launch(ctx, "structure_push");
}

int fvb_init_eval(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, const double* origin,
                  const int32_t* d_code, const int32_t* comp_off, const double* d_consts, int max_depth,
                  int primitive, const double* d_vecs, int nrand, int ninst, double* out,
                  unsigned long long* d_bad) {
  int r = validate(ctx, s);
  if (r) return r;
  if (max_depth < 1 || max_depth > 32)
    return set_err(ctx, FVB_E_CONFIG, "initial-data expression needs a stack of %d (device limit 32)", max_depth);
  if (ninst < 1) return set_err(ctx, FVB_E_CONFIG, "ninst must be >= 1");
  fvb::InitArgs A;
  std::memset(&A, 0, sizeof(A));
  A.code = d_code;
  A.k = d_consts;
  for (int c = 0; c <= s->ncomp; ++c) A.off[c] = comp_off[c];
  A.ncomp = s->ncomp;
  A.dim = s->dim;
  A.primitive = primitive;
  A.euler = s->eq == FVB_EQ_EULER;
  A.nrand = nrand;
  A.gamma = s->gamma;
  for (int k = 0; k < 3; ++k) {
    A.origin[k] = k < s->dim ? origin[k] : 0.0;
    A.delta[k] = k < s->dim ? s->deltas[k] : 1.0;
    A.n[k] = k < s->dim ? s->cells[k] : 1;
  }
  // make_field(grid, ncomp, 0.0): ghosts are zero; error slots start at "none"
  CUDA_TRY(ctx, cudaMemsetAsync(out, 0, sizeof(double) * lay->si * ninst, ctx->stream));
  CUDA_TRY(ctx, cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long) * ninst * (s->ncomp + 2), ctx->stream));
  fvb::launch_init_eval(A, *lay, d_vecs, ninst, out, d_bad, ctx->stream);
  ctx->launches++;
  return check_launch(ctx, "init_eval");
}

int fvb_halo_pack(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, const double* u, int axis, int side,
                  double* buf) {
  fvb::launch_halo(*s, *lay, const_cast<double*>(u), axis, side, buf, 0, ctx->stream);
  ctx->launches++;
  return check_launch(ctx, "halo_pack");
}

int fvb_halo_unpack(fvb_ctx* ctx, const fvb_scheme* s, const fvb_layout* lay, double* u, int axis, int side,
                    const double* buf) {
  fvb::launch_halo(*s, *lay, u, axis, side, const_cast<double*>(buf), 1, ctx->stream);
  ctx->launches++;
  return check_launch(ctx, "halo_unpack");
}

int64_t fvb_halo_count(const fvb_scheme* s, int axis) { return fvb::halo_count(*s, axis); }

}  // extern "C"

// ---------------------------------------------------------------------------
// numerics.py function-level entry points (the FLUX_FUNCTIONS seam)
// ---------------------------------------------------------------------------

int fvb_face_flux(fvb_ctx* ctx, const fvb_scheme* s, int axis, const double* uL, const double* uR, int64_t n,
                  double* F) {
  if (!s) return set_err(ctx, FVB_E_CONFIG, "null scheme");
  if (s->dim < 1 || s->dim > 3) return set_err(ctx, FVB_E_CONFIG, "dim must be 1, 2 or 3, got %d", s->dim);
  if (axis < 0 || axis >= s->dim) return set_err(ctx, FVB_E_CONFIG, "axis %d out of range", axis);
  if (s->flux == FVB_FLUX_HLLC && s->eq != FVB_EQ_EULER)
    return set_err(ctx, FVB_E_CONFIG, "HLLC flux is only defined for the Euler equations");
  fvb::Phys P;
  P.gamma = s->gamma;
  P.gm1 = s->gamma - 1.0;
  P.eps = s->weno_eps;
  for (int k = 0; k < 3; ++k) P.adv[k] = s->adv[k];
  // three scratch words (no single-shot call is in flight): degenerate flag,
  // first unphysical uL / uR face
  unsigned long long* d_err = reinterpret_cast<unsigned long long*>(ctx->d_scratch_state);
  const unsigned long long init[3] = {0ull, ~0ull, ~0ull};
  CUDA_TRY(ctx, cudaMemcpyAsync(d_err, init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
  const int r = s->arith == FVB_ARITH_FAST
                    ? fvb::fast::launch_face_flux(s->dim, s->eq, s->flux, P, axis, uL, uR, n, F, d_err, ctx->stream)
                    : fvb::exact::launch_face_flux(s->dim, s->eq, s->flux, P, axis, uL, uR, n, F, d_err, ctx->stream);
  if (r) return set_err(ctx, FVB_E_CONFIG, "unsupported equation/flux combination");
  ctx->launches++;
  int rc = check_launch(ctx, "face_flux");
  if (rc) return rc;
  unsigned long long h[3];
  CUDA_TRY(ctx, cudaMemcpyAsync(h, d_err, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  // the reference evaluates physical_flux(uL), physical_flux(uR), then the fan check
  if (h[1] != ~0ull) return set_err(ctx, FVB_E_UNPHYSICAL, "unphysical state: side L face %llu", h[1]);
  if (h[2] != ~0ull) return set_err(ctx, FVB_E_UNPHYSICAL, "unphysical state: side R face %llu", h[2]);
  if (h[0]) return set_err(ctx, FVB_E_UNPHYSICAL, "degenerate HLLC wave fan (sL >= sR)");
  return FVB_OK;
}

int fvb_weno(fvb_ctx* ctx, const fvb_scheme* s, const double* um, const double* uc, const double* up, int64_t n,
             double* w0, double* w1, double* face) {
  if (!s) return set_err(ctx, FVB_E_CONFIG, "null scheme");
  if (s->recon != FVB_RECON_WENO2 && s->recon != FVB_RECON_WENO3)
    return set_err(ctx, FVB_E_CONFIG, "weno_weights needs WENO2 or WENO3");
  const int r = s->arith == FVB_ARITH_FAST
                    ? fvb::fast::launch_weno(s->recon, s->weno_eps, um, uc, up, n, w0, w1, face, ctx->stream)
                    : fvb::exact::launch_weno(s->recon, s->weno_eps, um, uc, up, n, w0, w1, face, ctx->stream);
  if (r) return set_err(ctx, FVB_E_CONFIG, "unsupported reconstruction");
  ctx->launches++;
  return check_launch(ctx, "weno");
}
