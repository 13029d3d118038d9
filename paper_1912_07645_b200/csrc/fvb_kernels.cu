// Instantiates the stage / wave-speed kernels for one arithmetic mode.
// Built twice: -DFVB_FAST=0 -DFVB_NS=exact -fmad=false  (bitwise == reference)
//              -DFVB_FAST=1 -DFVB_NS=fast  -fmad=true
#include <algorithm>

#include "fvb_stage.cuh"

namespace fvb {
namespace FVB_NS {

// 3D: smem tile kernel (NT x NTY face cells); 1D/2D: warp-strip kernel
// (variant 0) or the smem tile kernel marching in y (variant 1)
template <int DIM> struct Blk;
template <> struct Blk<1> { static constexpr int NT = 128, NTY = 1; };
template <> struct Blk<2> { static constexpr int NT = 64, NTY = 1; };
#ifndef FVB_TILE3_NTY
#define FVB_TILE3_NTY 8
#endif
template <> struct Blk<3> { static constexpr int NT = 32, NTY = FVB_TILE3_NTY; };
constexpr int kStripWarps = 4;
#ifndef FVB_RING_NT
#define FVB_RING_NT 64
#endif
#ifndef FVB_RING_NT_SCALAR
#define FVB_RING_NT_SCALAR 32
#endif
// Euler: two-warp blocks; scalar laws: one-warp blocks whose x sweep runs on
// shuffles (measured: Euler 19.3 at 64 vs 19.0 at 32; Burgers 107.5 vs 114)
constexpr int kRingNT = FVB_RING_NT, kRingNTScalar = FVB_RING_NT_SCALAR;

// cells per block along x (reported as nt-2) and the y tile (nty-2, 3D only)
#if FVB_KDIM == 0
void stage_block(int dim, int eq, int variant, int& nt, int& nty) {
  if (dim == 1 && variant == 2) variant = 1;
  if (dim == 2 && variant == 2) { nt = eq == EQ_EULER ? kRingNT : kRingNTScalar; nty = 1; return; }
  if (dim == 2 && variant == 3) { nt = 2 * kPairNT; nty = 1; return; }  // 62 cells per one-warp block
  if (dim == 3 && variant == 2) { nt = kRing3NT; nty = kRing3NTY; return; }
  if (dim == 3 && variant == 4) { nt = kR3iNT; nty = kR3iNTY + 2; return; }  // 30 x 8 cells per block
  if (dim <= 2 && variant == 0) { nt = kStripCells * kStripWarps + 2; nty = 1; }
  else if (dim == 1) { nt = Blk<1>::NT; nty = 1; }
  else if (dim == 2) { nt = Blk<2>::NT; nty = 1; }
  else { nt = Blk<3>::NT; nty = Blk<3>::NTY; }
}
#endif

// Launch with programmatic stream serialisation (the kernel waits on
// griddepcontrol before its first dependent read), so a stage's CTAs are
// scheduled while the previous stage's last blocks drain.
// grid.x == 0 is an occupancy query: resident blocks per SM of the kernel
// that would be launched (fvb_capi.cu stage_grid sizes the grid with it)
template <typename K>
static int occupancy(K kern, dim3 block, int smem) {
  // raise (never lower) the opt-in limit: a later launch may need more
  // (the per-block offset table grows with the march length)
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, (int)(block.x * block.y), smem) != cudaSuccess) n = 0;
  return n;
}

template <typename K>
static int launch_pdl(K kern, dim3 grid, dim3 block, int smem, cudaStream_t s, const StageParams& p) {
  if (grid.x == 0) return occupancy(kern, block, smem);
  // wider ring blocks (-DFVB_RING_NT=96/128) need more than 48 KB
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
#if FVB_PDL
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, p);
#else
  kern<<<grid, block, smem, s>>>(p);
#endif
  return 0;
}

// opt a kernel into more than 48 KB of dynamic shared memory, once per device
template <typename K>
static void ensure_smem(K kern, int smem, unsigned& done_mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned bit = 1u << (dev & 31);
  if (smem > 48 * 1024 && !(done_mask & bit)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    done_mask |= bit;
  }
}

template <int EQ, int FLUX, int RECON, int KS, bool FIN>
static int launch_ring(const StageParams& p, dim3 grid, cudaStream_t s) {
  constexpr int NT = NComp<EQ, 2>::value == 1 ? kRingNTScalar : kRingNT;
  const int table = 4 * (p.H + kRingPD + 4);  // row-offset table (32-bit)
  if constexpr (NComp<EQ, 2>::value == 1) {
    if (p.ni == 2) {  // two instances per block (batched scalar ensembles)
      const int smem = ring_smem_bytes<EQ, RECON, NT, 2>() + table;
      return launch_pdl(ring_kernel<EQ, FLUX, RECON, NT, KS, FIN, 2>, grid, dim3(NT), smem, s, p);
    }
    if (p.ni == 4) {
      const int smem = ring_smem_bytes<EQ, RECON, NT, 4>() + table;
      return launch_pdl(ring_kernel<EQ, FLUX, RECON, NT, KS, FIN, 4>, grid, dim3(NT), smem, s, p);
    }
  }
  const int smem = ring_smem_bytes<EQ, RECON, NT>() + table;
  return launch_pdl(ring_kernel<EQ, FLUX, RECON, NT, KS, FIN>, grid, dim3(NT), smem, s, p);
}

template <int EQ, int FLUX, int RECON, int KS, bool FIN>
static int launch_pair(const StageParams& p, dim3 grid, cudaStream_t s) {
  const int smem = pair_smem_bytes<EQ>() + 4 * (p.H + kRingPD + 4);
  return launch_pdl(pair_kernel<EQ, FLUX, RECON, KS, FIN>, grid, dim3(kPairNT), smem, s, p);
}

template <int EQ, int FLUX, int RECON, int KS, bool FIN>
static int launch_ring3i(const StageParams& p, dim3 grid, cudaStream_t s) {
  const int smem = ring3i_smem_bytes<EQ>() + 4 * (p.H + 4);  // + plane-offset table
  auto kern = ring3i_kernel<EQ, FLUX, RECON, KS, FIN>;
  static unsigned done = 0;  // per instantiation
  ensure_smem(kern, 227 * 1024, done);
  if (grid.x == 0) return occupancy(kern, dim3(kR3iNT, kR3iNTY), smem);
  kern<<<grid, dim3(kR3iNT, kR3iNTY), smem, s>>>(p);
  return 0;
}

template <int DIM, int EQ, int FLUX, int RECON, bool FIN>
static int launch_fin(const StageParams& p, dim3 grid, cudaStream_t s) {
  if constexpr (DIM == 3) {
    if (p.variant == 4) {  // all-interior rows (default 3D)
      const int ks = p.kind == 0 ? 0 : (p.kind == 1 ? 1 : 2);
      if (FIN && ks == 0) return -1;
      if (ks == 0) return launch_ring3i<EQ, FLUX, RECON, (FIN ? 1 : 0), FIN>(p, grid, s);
      if (ks == 1) return launch_ring3i<EQ, FLUX, RECON, 1, FIN>(p, grid, s);
      return launch_ring3i<EQ, FLUX, RECON, 2, FIN>(p, grid, s);
    }
    if (p.variant == 2) {
      const int smem = ring3_smem_bytes<EQ>() + 8 * (p.H + 4);  // + plane-offset table
      auto kern = ring3_kernel<EQ, FLUX, RECON, FIN>;
      static unsigned done = 0;  // per instantiation
      ensure_smem(kern, 227 * 1024, done);  // a cap: the plane table grows with H
      if (grid.x == 0) return occupancy(kern, dim3(kRing3NT, kRing3NTY), smem);
      kern<<<grid, dim3(kRing3NT, kRing3NTY), smem, s>>>(p);
      return 0;
    }
  }
  if constexpr (DIM == 2) {
    if (p.variant == 3) {  // two x-columns per thread
      const int ks = p.kind == 0 ? 0 : (p.kind == 1 ? 1 : 2);
      if (FIN && ks == 0) return -1;
      if (ks == 0) return launch_pair<EQ, FLUX, RECON, (FIN ? 1 : 0), FIN>(p, grid, s);
      if (ks == 1) return launch_pair<EQ, FLUX, RECON, 1, FIN>(p, grid, s);
      return launch_pair<EQ, FLUX, RECON, 2, FIN>(p, grid, s);
    }
  }
  if constexpr (DIM == 2) {
    if (p.variant == 2) {
      // stage combination as a compile-time shape: residual only / u^s + dt L
      // / a u^n + b (u^s + dt L); the final stage never is the bare residual
      const int ks = p.kind == 0 ? 0 : (p.kind == 1 ? 1 : 2);
      if (FIN && ks == 0) return -1;
      if (ks == 0) return launch_ring<EQ, FLUX, RECON, (FIN ? 1 : 0), FIN>(p, grid, s);
      if (ks == 1) return launch_ring<EQ, FLUX, RECON, 1, FIN>(p, grid, s);
      return launch_ring<EQ, FLUX, RECON, 2, FIN>(p, grid, s);
    }
  }
  if (DIM <= 2 && p.variant == 0) {
    auto kern = strip_kernel<DIM, EQ, FLUX, RECON, kStripWarps, FIN>;
    if (grid.x == 0) return occupancy(kern, dim3(32 * kStripWarps), 0);
    kern<<<grid, 32 * kStripWarps, 0, s>>>(p);
    return 0;
  } else {
    constexpr int NT = Blk<DIM>::NT, NTY = Blk<DIM>::NTY;
    constexpr int smem = stage_smem_bytes<DIM, EQ, RECON, NT, NTY>();
    auto kern = stage_kernel<DIM, EQ, FLUX, RECON, NT, NTY, FIN>;
    static unsigned done = 0;  // per instantiation
    ensure_smem(kern, smem, done);
    if (grid.x == 0) return occupancy(kern, dim3(NT, NTY), smem);
    kern<<<grid, dim3(NT, NTY), smem, s>>>(p);
    return 0;
  }
}

// the last stage of a step (post-step checks, CFL maxima, finalisation) is
// a separate instantiation so the other stages carry none of its registers
template <int DIM, int EQ, int FLUX, int RECON>
static int launch_one(const StageParams& p, dim3 grid, cudaStream_t s) {
  return p.final_stage ? launch_fin<DIM, EQ, FLUX, RECON, true>(p, grid, s)
                       : launch_fin<DIM, EQ, FLUX, RECON, false>(p, grid, s);
}

template <int DIM>
static int launch_dim(int eq, int flux, int recon, const StageParams& p, dim3 grid, cudaStream_t s) {
#define FVB_CASE(E, F, R) \
  if (eq == E && flux == F && recon == R) return launch_one<DIM, E, F, R>(p, grid, s);
  FVB_CASE(EQ_EULER, FLUX_HLLC, RECON_NONE)
  FVB_CASE(EQ_EULER, FLUX_HLLC, RECON_WENO2)
  FVB_CASE(EQ_EULER, FLUX_HLLC, RECON_WENO3)
  FVB_CASE(EQ_EULER, FLUX_RUSANOV, RECON_NONE)
  FVB_CASE(EQ_EULER, FLUX_RUSANOV, RECON_WENO2)
  FVB_CASE(EQ_EULER, FLUX_RUSANOV, RECON_WENO3)
  FVB_CASE(EQ_BURGERS, FLUX_RUSANOV, RECON_NONE)
  FVB_CASE(EQ_BURGERS, FLUX_RUSANOV, RECON_WENO2)
  FVB_CASE(EQ_BURGERS, FLUX_RUSANOV, RECON_WENO3)
  FVB_CASE(EQ_ADVECTION, FLUX_RUSANOV, RECON_NONE)
  FVB_CASE(EQ_ADVECTION, FLUX_RUSANOV, RECON_WENO2)
  FVB_CASE(EQ_ADVECTION, FLUX_RUSANOV, RECON_WENO3)
#undef FVB_CASE
  return -1;
}

// One translation unit per dimension (FVB_KDIM = 1, 2, 3) so the six
// instantiation-heavy units compile in parallel; FVB_KDIM = 0 holds the
// dispatcher and the wave-speed kernels.
#if FVB_KDIM == 1
int launch_stage_d1(int eq, int flux, int recon, const StageParams& p, dim3 grid, cudaStream_t s) {
  return launch_dim<1>(eq, flux, recon, p, grid, s);
}
#elif FVB_KDIM == 2
int launch_stage_d2(int eq, int flux, int recon, const StageParams& p, dim3 grid, cudaStream_t s) {
  return launch_dim<2>(eq, flux, recon, p, grid, s);
}
#if FVB_BLOCK_TIMES && FVB_FAST
}  // namespace FVB_NS
}  // namespace fvb
// diagnostic (variant builds only): per-block [start, end] ns and SM of the
// last pair-kernel launch of each RK stage; out: 3 x 8192 x 3 uint64
extern "C" int fvb_debug_block_times(unsigned long long* out) {
  static unsigned long long t[3][8192][2];
  static unsigned sm[3][8192];
  if (cudaMemcpyFromSymbol(t, fvb::fast::g_bt, sizeof(t)) != cudaSuccess) return 6;
  if (cudaMemcpyFromSymbol(sm, fvb::fast::g_bt_sm, sizeof(sm)) != cudaSuccess) return 6;
  for (int k = 0; k < 3; ++k)
    for (int b = 0; b < 8192; ++b) {
      out[(k * 8192 + b) * 3 + 0] = t[k][b][0];
      out[(k * 8192 + b) * 3 + 1] = t[k][b][1];
      out[(k * 8192 + b) * 3 + 2] = sm[k][b];
    }
  return 0;
}
namespace fvb {
namespace FVB_NS {
#endif
#elif FVB_KDIM == 3
int launch_stage_d3(int eq, int flux, int recon, const StageParams& p, dim3 grid, cudaStream_t s) {
  return launch_dim<3>(eq, flux, recon, p, grid, s);
}
#else
int launch_stage_d1(int eq, int flux, int recon, const StageParams& p, dim3 grid, cudaStream_t s);
int launch_stage_d2(int eq, int flux, int recon, const StageParams& p, dim3 grid, cudaStream_t s);
int launch_stage_d3(int eq, int flux, int recon, const StageParams& p, dim3 grid, cudaStream_t s);
int launch_stage(int dim, int eq, int flux, int recon, const StageParams& p, dim3 grid, cudaStream_t s) {
  switch (dim) {
    case 1: return launch_stage_d1(eq, flux, recon, p, grid, s);
    case 2: return launch_stage_d2(eq, flux, recon, p, grid, s);
    case 3: return launch_stage_d3(eq, flux, recon, p, grid, s);
  }
  return -1;
}

#endif

#if FVB_KDIM == 0
// numerics.py:133-196 on arrays of face pairs (the FLUX_FUNCTIONS seam):
// the stage kernels' own device flux functions, one face per thread.
// err[0]: degenerate HLLC fan seen; err[1] / err[2]: lowest face index with
// an unphysical uL / uR state (physical_flux's check, equations.py:91-99).
template <int EQ, int FLUX, int DIM>
__global__ void face_flux_kernel(Phys P, int axis, const double* __restrict__ uL, const double* __restrict__ uR,
                                 int64_t n, double* __restrict__ F, unsigned long long* err) {
  constexpr int NC = NComp<EQ, DIM>::value;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double a[NC], b[NC], f[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      a[c] = uL[c * n + i];
      b[c] = uR[c * n + i];
    }
    unsigned eb = 0;
    if constexpr (EQ == EQ_EULER) {
      if (!((a[0] > kFloor) & (euler_pressure<DIM>(a, P) > kFloor))) atomicMin(err + 1, (unsigned long long)i);
      if (!((b[0] > kFloor) & (euler_pressure<DIM>(b, P) > kFloor))) atomicMin(err + 2, (unsigned long long)i);
      const EState L = euler_state<DIM>(a, axis, P);
      const EState R = euler_state<DIM>(b, axis, P);
      if constexpr (FLUX == FLUX_HLLC) hllc<DIM>(a, b, L, R, axis, P, f, eb, bits_equal_all<NC>(a, b));
      else rusanov<EQ, DIM>(a, b, L, R, axis, P, f);
    } else {
      EState d{};
      rusanov<EQ, DIM>(a, b, d, d, axis, P, f);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) F[c * n + i] = f[c];
    if (eb) atomicOr(err, 1ull);
  }
}

template <int RECON>
__global__ void weno_kernel(double eps, const double* __restrict__ um, const double* __restrict__ uc,
                            const double* __restrict__ up, int64_t n, double* w0, double* w1, double* face) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double m = um[i], c = uc[i], q = up[i];
    // numerics.py:64-87, operation by operation
    constexpr double d0 = RECON == RECON_WENO2 ? 0.5 : 1.0 / 3.0, d1 = RECON == RECON_WENO2 ? 0.5 : 2.0 / 3.0;
    const double D0 = c - m, D1 = q - c;
    const double e0 = eps + D0 * D0, e1 = eps + D1 * D1;
    const double a0 = d0 / (e0 * e0), a1 = d1 / (e1 * e1);
    const double tot = a0 + a1;
    const double x0 = a0 / tot, x1 = a1 / tot;
    if (w0) w0[i] = x0;
    if (w1) w1[i] = x1;
    if (face) face[i] = c + 0.5 * (x0 * D0 + x1 * D1);
  }
}

int launch_face_flux(int dim, int eq, int flux, const Phys& P, int axis, const double* uL, const double* uR,
                     int64_t n, double* F, unsigned long long* err, cudaStream_t s) {
  const int blocks = (int)std::min<int64_t>((n + 127) / 128, 148 * 16);
  if (n <= 0) return 0;
#define FVB_FF(E, FL, D) \
  if (eq == E && flux == FL && dim == D) { face_flux_kernel<E, FL, D><<<blocks, 128, 0, s>>>(P, axis, uL, uR, n, F, err); return 0; }
  FVB_FF(EQ_EULER, FLUX_HLLC, 1) FVB_FF(EQ_EULER, FLUX_HLLC, 2) FVB_FF(EQ_EULER, FLUX_HLLC, 3)
  FVB_FF(EQ_EULER, FLUX_RUSANOV, 1) FVB_FF(EQ_EULER, FLUX_RUSANOV, 2) FVB_FF(EQ_EULER, FLUX_RUSANOV, 3)
  FVB_FF(EQ_BURGERS, FLUX_RUSANOV, 1) FVB_FF(EQ_BURGERS, FLUX_RUSANOV, 2) FVB_FF(EQ_BURGERS, FLUX_RUSANOV, 3)
  FVB_FF(EQ_ADVECTION, FLUX_RUSANOV, 1) FVB_FF(EQ_ADVECTION, FLUX_RUSANOV, 2)
  FVB_FF(EQ_ADVECTION, FLUX_RUSANOV, 3)
#undef FVB_FF
  return -1;
}

int launch_weno(int recon, double eps, const double* um, const double* uc, const double* up, int64_t n, double* w0,
                double* w1, double* face, cudaStream_t s) {
  if (n <= 0) return 0;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  if (recon == RECON_WENO2) weno_kernel<RECON_WENO2><<<blocks, 256, 0, s>>>(eps, um, uc, up, n, w0, w1, face);
  else if (recon == RECON_WENO3) weno_kernel<RECON_WENO3><<<blocks, 256, 0, s>>>(eps, um, uc, up, n, w0, w1, face);
  else return -1;
  return 0;
}

template <int DIM>
static int launch_speed_dim(int eq, const StageParams& p, int fin, dim3 grid, cudaStream_t s) {
  if (eq == EQ_EULER) speed_kernel<DIM, EQ_EULER><<<grid, 256, 0, s>>>(p, fin);
  else if (eq == EQ_BURGERS) speed_kernel<DIM, EQ_BURGERS><<<grid, 256, 0, s>>>(p, fin);
  else speed_kernel<DIM, EQ_ADVECTION><<<grid, 256, 0, s>>>(p, fin);
  return 0;
}

int launch_speed(int dim, int eq, const StageParams& p, int fin, dim3 grid, cudaStream_t s) {
  switch (dim) {
    case 1: return launch_speed_dim<1>(eq, p, fin, grid, s);
    case 2: return launch_speed_dim<2>(eq, p, fin, grid, s);
    case 3: return launch_speed_dim<3>(eq, p, fin, grid, s);
  }
  return -1;
}
#endif

}  // namespace FVB_NS
}  // namespace fvb
