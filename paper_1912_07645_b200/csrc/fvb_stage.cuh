// Fused finite-volume stage kernel: WENO2/3 (or piecewise-constant) face
// reconstruction + positivity fallback + Rusanov/HLLC flux + flux
// difference + SSP-RK stage combination + (last stage) post-step checks and
// the CFL wave-speed reduction, in ONE pass over the field.
//
// Replaces solver.py:82-113 (spatial_residual), numerics.py:90-196,
// solver.py:116-125, solver.py:158-173 and, fused into the last stage,
// solver.py:128-149 + 231-242.
//
// Work decomposition (B200):
//  * The slowest axis (y in 2D, z in 3D) is MARCHED: a block owns a strip of
//    columns (x [, y]) and walks H rows (planes) of one march chunk, so the
//    march-axis faces and fluxes are computed exactly once per cell and each
//    cell of u^s is read from HBM once per stage.
//  * Kernels, by default use:
//      pair_kernel   2D Euler, fast mode: one-warp blocks, two x-columns per
//                    lane, rows in a cp.async shared-memory ring (16-byte
//                    copies), x neighbours by shuffle.
//      ring_kernel   2D otherwise: one column per thread, the same ring.
//      ring3i_kernel 3D: 32 x 8 threads own a 30 x 8 cell tile, planes in a
//                    cp.async ring, x sweep by shuffle, y sweep via shared
//                    memory, every warp an interior row.
//      stage_kernel  1D (and the FVB_KERNEL=tile alternative in 2D / 3D):
//                    per-thread register window.
//    Alternatives for A/B runs: strip_kernel (FVB_KERNEL=strip), ring3_kernel
//    (FVB_KERNEL=ring3, the round-1 3D kernel).
//  * Thread <-> "face cell" mapping: a block's threads cover its updated
//    cells plus one halo face cell each side in x, so every WENO face pair is
//    computed once per row and each interface flux once (+2 per strip).
//  * Ghost cells are never materialised for periodic/outflow axes: indices
//    outside the interior are wrapped/clamped on load, which reproduces
//    fill_boundary (grid.py:147-175) exactly; FVB_BC_HALO axes read ghosts
//    from memory (filled by the halo exchange).
//  * The transverse-interior crop of solver.py:99-104 means no corner ghost
//    is ever read, so a face-only halo exchange is result-identical.
//
// This header is compiled twice (FVB_FAST=0 with -fmad=false -> namespace
// exact; FVB_FAST=1 -> namespace fast).
#pragma once
#include <cuda_runtime.h>
#include "fvb_physics.cuh"
#include "fvb_state.cuh"

namespace fvb {
namespace FVB_NS {

__device__ __forceinline__ int64_t map_index(int64_t i, int64_t n, int bc, int g) {
  i = i < -g ? -g : (i > n + g - 1 ? n + g - 1 : i);   // memory safety
  if (bc == FVB_BC_PERIODIC) return i < 0 ? i + n : (i >= n ? i - n : i);
  if (bc == FVB_BC_OUTFLOW) return i < 0 ? 0 : (i >= n ? n - 1 : i);
  return i;
}

template <int DIM>
__device__ __forceinline__ int64_t cell_off(const StageParams& p, int64_t x, int64_t y, int64_t z) {
  int64_t o = map_index(x, p.n[0], p.bc[0], p.g);
  if (DIM >= 2) o += map_index(y, p.n[1], p.bc[1], p.g) * p.sy;
  if (DIM >= 3) o += map_index(z, p.n[2], p.bc[2], p.g) * p.sz;
  return o;
}

template <int NC>
__device__ __forceinline__ void load_nc(const double* __restrict__ b, int64_t off, int64_t sc, double* v) {
#pragma unroll
  for (int c = 0; c < NC; ++c) v[c] = __ldg(b + off + c * sc);
}

__device__ __forceinline__ double ddiv(double a, const StageParams& p, int axis) {
#if FVB_FAST
  return a * p.id[axis];
#else
  return p.divd[axis] ? a / p.dd[axis] : a * p.id[axis];
#endif
}

// Fused halo exchange of a decomposed run whose march axis is split: a cell
// of the first / last g march rows is also stored into the ghost rows of the
// low / high neighbour's copy of the same buffer (peer memory over NVLink),
// so the next stage reads its halo without a separate exchange
// (parallel.py:201-254; the transverse crop of solver.py:99-104 means the
// face layers suffice).  A no-op outside such runs (null peers).
__device__ __forceinline__ void peer_store(const StageParams& p, int64_t o, int64_t row, int64_t cstride, int c,
                                           double v) {
  if (p.peer_lo && row < p.g) p.peer_lo[o + p.peer_shift + c * cstride] = v;
  if (p.peer_hi && row >= p.n_march - p.g) p.peer_hi[o - p.peer_shift + c * cstride] = v;
}

// RK stage combination (solver.py:166-173)
__device__ __forceinline__ double rk_combine(int kind, double un, double us, double dt, double L) {
#if FVB_FAST
  switch (kind) {
    case 0: return L;
    case 1: return fma(dt, L, us);
    case 2: return fma(0.5, un, 0.5 * fma(dt, L, us));
    case 3: return fma(0.75, un, 0.25 * fma(dt, L, us));
    default: return fma(1.0 / 3.0, un, (2.0 / 3.0) * fma(dt, L, us));
  }
#else
  switch (kind) {
    case 0: return L;
    case 1: return us + dt * L;
    case 2: return 0.5 * un + 0.5 * (us + dt * L);
    case 3: return 0.75 * un + 0.25 * (us + dt * L);
    default: return (1.0 / 3.0) * un + (2.0 / 3.0) * (us + dt * L);
  }
#endif
}

template <int DIM>
__device__ __forceinline__ long long flat_cell(const StageParams& p, int64_t x, int64_t y, int64_t z) {
  return ((long long)z * p.n[1] + y) * p.n[0] + x;
}

// Post-step work on the new value of one interior cell (last stage only).
template <int EQ, int DIM, int NC>
__device__ __forceinline__ void post_cell(const StageParams& p, FvbState* st, const double* v,
                                          int64_t x, int64_t y, int64_t z, double* smax) {
  const long long cell = flat_cell<DIM>(p, x, y, z);
  // non-finite <=> exponent field all ones: one integer test per component,
  // one (rare) branch for the first bad component
  unsigned bad = 0u;
#pragma unroll
  for (int c = 0; c < NC; ++c) bad |= ((((unsigned)__double2hiint(v[c]) >> 20) & 0x7ffu) == 0x7ffu) ? (1u << c) : 0u;
  if (bad) {
    const long long ncell = (long long)p.n[0] * p.n[1] * p.n[2];
    atomicMin(&st->bad_nonfinite, (long long)(__ffs(bad) - 1) * ncell + cell);
  }
  double s[DIM];
#if FVB_FAST
  if constexpr (EQ == EQ_EULER) {  // one pressure for the physical check and the sound speed
    const double r = frcp(v[0]);
    double msq = v[1] * v[1];
#pragma unroll
    for (int k = 1; k < DIM; ++k) msq = fma(v[1 + k], v[1 + k], msq);
    const double pr = p.P.gm1 * fma(-0.5 * msq, r, v[1 + DIM]);
    if (!((v[0] > kFloor) & (pr > kFloor))) atomicMin(&st->bad_unphys, cell);
    const double c = fsqrt(p.P.gamma * pr * r);
#pragma unroll
    for (int k = 0; k < DIM; ++k) s[k] = fabs(v[1 + k] * r) + c;
  } else {
    wave_speeds<EQ, DIM>(v, p.P, s);
  }
#else
  if constexpr (EQ == EQ_EULER) {
    if (!euler_physical<DIM>(v, p.P)) atomicMin(&st->bad_unphys, cell);
  }
  wave_speeds<EQ, DIM>(v, p.P, s);
#endif
#pragma unroll
  for (int k = 0; k < DIM; ++k) smax[k] = fmax(smax[k], s[k]);
}

// Block reduction of the per-thread maxima + last-block finalisation.
template <int DIM>
__device__ __forceinline__ void block_epilogue(const StageParams& p, FvbState* st, int inst,
                                               const double* smax, bool post) {
  const int lane = (threadIdx.y * blockDim.x + threadIdx.x) & 31;
#pragma unroll
  for (int k = 0; k < DIM; ++k) {
    unsigned long long b = (unsigned long long)__double_as_longlong(smax[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long q = __shfl_xor_sync(0xffffffffu, b, o);
      b = q > b ? q : b;
    }
    if (lane == 0 && b != 0ull) atomicMax(&st->smax[k], b);
  }
  if (p.defer_finalize) return;  // maxima stay in the state for the cross-rank reduce
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&st->blocks_done, 1u);
    if (prev == p.nblocks - 1) {
      __threadfence();
      finalize_step(st, p.ctl, p.shared_state ? 0 : inst, post, true);
    }
  }
}

// ---------------------------------------------------------------------------
// Shared-memory tile kernel (default for 1D/2D, the 3D path).
//
// A block of NT (x) [x NTY (y, 3D)] threads owns NT-2 [x NTY-2] cells of the
// plane and marches H rows along the slowest axis.  Thread <-> "face cell"
// mapping: every WENO face pair of the plane is computed once per row and
// every interface flux once (+2/NT halo).  The march axis uses a per-thread
// 3-row register window; the row loop is unrolled by 3 with the window
// arrays rotated by NAME (no register moves) and the row after next loaded
// into the slot that just died.
// ---------------------------------------------------------------------------
template <int DIM, int EQ, int FLUX, int RECON, int NT, int NTY, bool FIN>
struct TileCtx {
  static constexpr int NC = NComp<EQ, DIM>::value;
  static constexpr bool WENO = RECON != RECON_NONE;
  static constexpr bool MARCH = DIM >= 2;
  static constexpr bool PY = DIM == 3;          // y handled in-plane (3D)
  static constexpr int SUY = PY ? NTY + 2 : 1;  // rows of the plane tile in smem
  static constexpr int OY = PY ? 1 : 0;
  static constexpr int MA = DIM - 1;            // march axis
  static constexpr int nU = NC * SUY * (NT + 2);
  static constexpr int nFX = WENO ? NC * NTY * NT : 0;
  static constexpr int nGX = NC * NTY * NT;
  static constexpr int nFY = (WENO && PY) ? NC * NTY * NT : 0;

  const StageParams& p;
  FvbState* st;
  const double* __restrict__ us;
  const double* un;
  double* out;
  double* smem;
  double dt;
  int tx, ty;
  int64_t x0, y0, xf, yf;
  bool cell;
  int64_t ra, rb;
  int64_t co;  // mapped in-plane offset of this thread's column
  unsigned errb;
  double smax[DIM];

  __device__ __forceinline__ double& U(int c, int y, int x) const { return smem[(c * SUY + y) * (NT + 2) + x]; }
  __device__ __forceinline__ double& HX(int c, int y, int x) const { return smem[nU + (c * NTY + y) * NT + x]; }
  __device__ __forceinline__ double& LX(int c, int y, int x) const { return smem[nU + nFX + (c * NTY + y) * NT + x]; }
  __device__ __forceinline__ double& GX(int c, int y, int x) const {
    return smem[nU + 2 * nFX + (c * NTY + y) * NT + x];
  }
  __device__ __forceinline__ double& HY(int c, int y, int x) const {
    return smem[nU + 2 * nFX + nGX + (c * NTY + y) * NT + x];
  }
  __device__ __forceinline__ double& LY(int c, int y, int x) const {
    return smem[nU + 2 * nFX + nGX + nFY + (c * NTY + y) * NT + x];
  }
  __device__ __forceinline__ double& GY(int c, int y, int x) const {
    return smem[nU + 2 * nFX + nGX + 2 * nFY + (c * NTY + y) * NT + x];
  }
  // 3D: the z recurrence (high face H, flux G of the previous plane) lives
  // in shared memory -- it is idle during the in-plane sweeps
  static constexpr int nGY = PY ? NC * NTY * NT : 0;
  __device__ __forceinline__ double& HS(int c) const {
    return smem[nU + 2 * nFX + nGX + 2 * nFY + nGY + (c * NTY + ty) * NT + tx];
  }
  __device__ __forceinline__ double& GS(int c) const {
    return smem[nU + 2 * nFX + nGX + 2 * nFY + nGY + NC * NTY * NT + (c * NTY + ty) * NT + tx];
  }

  __device__ __forceinline__ int64_t roff(int64_t r) const {
    if constexpr (DIM == 2) return map_index(r, p.n[1], p.bc[1], p.g) * p.sy;
    else if constexpr (DIM == 3) return map_index(r, p.n[2], p.bc[2], p.g) * p.sz;
    else return 0;
  }
  __device__ __forceinline__ int64_t pin(int64_t x, int64_t y) const {
    int64_t o = map_index(x, p.n[0], p.bc[0], p.g);
    if constexpr (PY) o += map_index(y, p.n[1], p.bc[1], p.g) * p.sy;
    return o;
  }
  __device__ __forceinline__ void load_col(int64_t r, double* v) const { load_nc<NC>(us, co + roff(r), p.sc, v); }

  __device__ __forceinline__ void finish(int64_t r, const double* usc, const double* unc, const double* Lc) {
    double v[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) v[c] = rk_combine(p.kind, unc[c], usc[c], dt, Lc[c]);
    const int64_t o = co + roff(r);
#pragma unroll
    for (int c = 0; c < NC; ++c) out[o + c * p.sc] = v[c];
    if constexpr (FIN) post_cell<EQ, DIM, NC>(p, st, v, xf, PY ? yf : (MARCH ? r : 0), PY ? r : 0, smax);
  }

  // in-plane axes (x; x and y in 3D) of row r: R <- residual of this cell
  __device__ __forceinline__ void inplane(int64_t r, const double* B, double* R) {
    if constexpr (EQ == EQ_EULER) {  // stage-start interior check (solver.py:90-93)
      if (p.check_input && cell && !euler_physical<DIM>(B, p.P)) {
        const long long key = ((long long)p.stage_idx << 42) |
                              flat_cell<DIM>(p, xf, PY ? yf : (MARCH ? r : 0), PY ? r : 0);
        atomicMin(&st->stage_err, key);
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) U(c, ty + OY, tx + 1) = B[c];
    if constexpr (WENO) {
      if ((!PY || (ty >= 1 && ty <= NTY - 2)) && (tx == 0 || tx == NT - 1)) {
        const int64_t hxo = pin(tx == 0 ? x0 - 2 : x0 + NT - 1, yf) + roff(r);
        const int col = tx == 0 ? 0 : NT + 1;
#pragma unroll
        for (int c = 0; c < NC; ++c) U(c, ty + OY, col) = __ldg(us + hxo + c * p.sc);
      }
      if constexpr (PY) {
        if ((ty == 0 || ty == NTY - 1) && tx >= 1 && tx <= NT - 2) {
          const int64_t hyo = pin(xf, ty == 0 ? y0 - 2 : y0 + NTY - 1) + roff(r);
          const int row = ty == 0 ? 0 : NTY + 1;
#pragma unroll
          for (int c = 0; c < NC; ++c) U(c, row, tx + 1) = __ldg(us + hyo + c * p.sc);
        }
      }
    }
    __syncthreads();
    if constexpr (WENO) {
      if (!PY || (ty >= 1 && ty <= NTY - 2)) {
        double um[NC], uc[NC], up[NC], hi[NC], lo[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          um[c] = U(c, ty + OY, tx);
          uc[c] = U(c, ty + OY, tx + 1);
          up[c] = U(c, ty + OY, tx + 2);
        }
        weno_faces_nc<NC, RECON>(um, uc, up, p.P.eps, hi, lo);
#pragma unroll
        for (int c = 0; c < NC; ++c) { HX(c, ty, tx) = hi[c]; LX(c, ty, tx) = lo[c]; }
      }
      if constexpr (PY) {
        if (tx >= 1 && tx <= NT - 2) {
          double um[NC], uc[NC], up[NC], hi[NC], lo[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            um[c] = U(c, ty, tx + 1);
            uc[c] = U(c, ty + 1, tx + 1);
            up[c] = U(c, ty + 2, tx + 1);
          }
          weno_faces_nc<NC, RECON>(um, uc, up, p.P.eps, hi, lo);
#pragma unroll
          for (int c = 0; c < NC; ++c) { HY(c, ty, tx) = hi[c]; LY(c, ty, tx) = lo[c]; }
        }
      }
      __syncthreads();
    }
    // interface fluxes: x interface tx sits between face cells tx-1 and tx
    // (lane 0 computes an unused one: no divergence inside cell warps)
    if (!PY || (ty >= 1 && ty <= NTY - 2)) {
      const int tl = tx >= 1 ? tx - 1 : 0;
      double uL[NC], uR[NC], G[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        uL[c] = WENO ? HX(c, ty, tl) : U(c, ty + OY, tx);
        uR[c] = WENO ? LX(c, ty, tx) : U(c, ty + OY, tx + 1);
      }
      auto cells = [&](double* a, double* b) {  // fallback only: loaded on demand
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          a[c] = U(c, ty + OY, tx);
          b[c] = U(c, ty + OY, tx + 1);
        }
      };
      unsigned eb = 0;
      interface_flux_lazy<EQ, FLUX, DIM, RECON>(uL, uR, cells, 0, p.P, G, eb);
      if (eb && tx >= 1 && xf <= p.n[0] && (!PY || yf < p.n[1])) errb |= 1u;
#pragma unroll
      for (int c = 0; c < NC; ++c) GX(c, ty, tx) = G[c];
    }
    if constexpr (PY) {
      if (ty >= 1) {  // lanes 0 and NT-1 compute unused fluxes (no divergence)
        double uL[NC], uR[NC], G[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          uL[c] = WENO ? HY(c, ty - 1, tx) : U(c, ty, tx + 1);
          uR[c] = WENO ? LY(c, ty, tx) : U(c, ty + 1, tx + 1);
        }
        auto cells = [&](double* a, double* b) {  // fallback only: loaded on demand
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            a[c] = U(c, ty, tx + 1);
            b[c] = U(c, ty + 1, tx + 1);
          }
        };
        unsigned eb = 0;
        interface_flux_lazy<EQ, FLUX, DIM, RECON>(uL, uR, cells, 1, p.P, G, eb);
        if (eb && tx >= 1 && tx <= NT - 2 && yf <= p.n[1] && xf < p.n[0]) errb |= 2u;
#pragma unroll
        for (int c = 0; c < NC; ++c) GY(c, ty, tx) = G[c];
      }
    }
    __syncthreads();
    if (cell) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
#if FVB_FAST
        double res = (GX(c, ty, tx) - GX(c, ty, tx + 1)) * p.id[0];
        if constexpr (PY) res = fma(GY(c, ty, tx) - GY(c, ty + 1, tx), p.id[1], res);
#else
        double res = 0.0 - ddiv(GX(c, ty, tx + 1) - GX(c, ty, tx), p, 0);
        if constexpr (PY) res = res - ddiv(GY(c, ty + 1, tx) - GY(c, ty, tx), p, 1);
#endif
        R[c] = res;
      }
    }
  }

  // One march row r.  On entry A,B,C = u[r-1], u[r], u[r+1]; on exit A
  // holds u[r+2].  H: high march-face of row r-1 -> r; G: march flux
  // (r-2|r-1) -> (r-1|r); R: in-plane residual of row r-1 -> r.
  __device__ __forceinline__ void row(int64_t r, double* A, const double* B, const double* C, double* H, double* G,
                                      double* R) {
    const bool fin = cell && r - 1 >= ra;
    // every lane of a warp that holds cells computes (halo lanes on real
    // neighbour columns); only side effects are predicated on `cell`.  Whole
    // halo warps (3D: ty = 0, NTY-1) skip the march work.
    const bool active = !PY || (ty >= 1 && ty <= NTY - 2);
    double unc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) unc[c] = 0.0;
    if (active && r - 1 >= ra && p.kind >= 2) {
      const int64_t o = co + roff(r - 1);
#pragma unroll
      for (int c = 0; c < NC; ++c) unc[c] = un[o + c * p.sc];
    }
    if (active) {
      double hi[NC], lo[NC];
      weno_faces_nc<NC, RECON>(A, B, C, p.P.eps, hi, lo);
      if (r >= ra) {
        double GC[NC], Hc[NC], Gc[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          Hc[c] = PY ? HS(c) : H[c];
          Gc[c] = PY ? GS(c) : G[c];
        }
        unsigned eb = 0;
        interface_flux<EQ, FLUX, DIM, RECON>(Hc, lo, A, B, MA, p.P, GC, eb);
        if (eb && cell) errb |= 1u << MA;
        if (fin) {
          double Lc[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) {
#if FVB_FAST
            Lc[c] = fma(Gc[c] - GC[c], p.id[MA], R[c]);
#else
            Lc[c] = R[c] - ddiv(GC[c] - Gc[c], p, MA);
#endif
          }
          finish(r - 1, A, unc, Lc);
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          if constexpr (PY) GS(c) = GC[c];
          else G[c] = GC[c];
        }
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        if constexpr (PY) HS(c) = hi[c];
        else H[c] = hi[c];
      }
    }
    if (r + 2 <= rb + 1) load_col(r + 2, A);  // A is dead: the row after next
    if (r >= ra && r < rb) inplane(r, B, R);
  }
};

#ifndef FVB_TILE_MINB
#define FVB_TILE_MINB 8  // 2D: cap at 128 registers -> 16 warps/SM (measured best)
#endif
#ifndef FVB_TILE3_MINB
#define FVB_TILE3_MINB 2  // 3D: 256-thread tile, cap at 128 registers -> 2 blocks/SM
#endif
#ifndef FVB_TILE_UNROLL
#define FVB_TILE_UNROLL 1
#endif
template <int DIM, int EQ, int FLUX, int RECON, int NT, int NTY, bool FIN>
__global__ void __launch_bounds__(NT * NTY, (DIM == 2 ? FVB_TILE_MINB : (DIM == 3 ? FVB_TILE3_MINB : 1)))
stage_kernel(const StageParams p) {
  using T = TileCtx<DIM, EQ, FLUX, RECON, NT, NTY, FIN>;
  constexpr int NC = T::NC;
  extern __shared__ double smem[];
  int inst, chunk;
  int64_t y0 = 0;
  if constexpr (DIM == 3) {
    inst = blockIdx.z / p.chunks;
    chunk = blockIdx.z % p.chunks;
    y0 = (int64_t)blockIdx.y * (NTY - 2);
  } else if constexpr (DIM == 2) {
    inst = blockIdx.z;
    chunk = blockIdx.y;
  } else {
    inst = blockIdx.z;
    chunk = 0;
  }
  FvbState* st = p.st + (p.shared_state ? 0 : inst);
  if (*(volatile int*)&st->done) return;  // uniform over the block
  const int tx = threadIdx.x;
  const int ty = T::PY ? threadIdx.y : 0;
  const int64_t x0 = (int64_t)blockIdx.x * (NT - 2);
  const int64_t xf = x0 - 1 + tx;
  const int64_t yf = T::PY ? y0 - 1 + ty : 0;
  bool cell = tx >= 1 && tx <= NT - 2 && xf < p.n[0];
  if (T::PY) cell = cell && ty >= 1 && ty <= NTY - 2 && yf < p.n[1];
  const int64_t ra = T::MARCH ? p.row_lo + (int64_t)chunk * p.H : 0;
  const int64_t rb = T::MARCH ? min(ra + (int64_t)p.H, p.row_hi) : 1;
  T t{p, st, p.us + p.origin + inst * p.si, p.un + p.origin + inst * p.si, p.out + p.origin + inst * p.si, smem,
      p.kind == 0 ? 0.0 : *(volatile double*)&st->dt, tx, ty, x0, y0, xf, yf, cell, ra, rb, 0, 0u, {}};
  t.co = t.pin(xf, yf);
#pragma unroll
  for (int k = 0; k < DIM; ++k) t.smax[k] = 0.0;

  double H[NC], G[NC], R[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) H[c] = G[c] = R[c] = 0.0;
  if constexpr (T::MARCH) {
    double W0[NC], W1[NC], W2[NC];
    t.load_col(ra - 2, W0);
    t.load_col(ra - 1, W1);
    t.load_col(ra, W2);
#if FVB_TILE_UNROLL == 3
    for (int64_t r = ra - 1; r <= rb; r += 3) {
      t.row(r, W0, W1, W2, H, G, R);
      if (r + 1 > rb) break;
      t.row(r + 1, W1, W2, W0, H, G, R);
      if (r + 2 > rb) break;
      t.row(r + 2, W2, W0, W1, H, G, R);
    }
#else
    // one copy of the row body (instruction-cache friendly); the window is
    // rotated with register moves
    for (int64_t r = ra - 1; r <= rb; ++r) {
      t.row(r, W0, W1, W2, H, G, R);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double w = W0[c];
        W0[c] = W1[c];
        W1[c] = W2[c];
        W2[c] = w;
      }
    }
#endif
  } else {
    double B[NC], unc[NC];
    t.load_col(0, B);
    t.inplane(0, B, R);
    if (cell) {
      if (p.kind >= 2) {
#pragma unroll
        for (int c = 0; c < NC; ++c) unc[c] = t.un[t.co + c * p.sc];
      }
      t.finish(0, B, unc, R);
    }
  }
  if (t.errb) {
#pragma unroll
    for (int a = 0; a < DIM; ++a)
      if (t.errb & (1u << a))
        atomicMin(&st->stage_err, ((long long)p.stage_idx << 42) | ((long long)(1 + a) << 40));
  }
  if constexpr (FIN) block_epilogue<DIM>(p, st, inst, t.smax, true);
}

template <int DIM, int EQ, int RECON, int NT, int NTY>
constexpr int stage_smem_bytes() {
  constexpr int NC = NComp<EQ, DIM>::value;
  constexpr bool WENO = RECON != RECON_NONE;
  constexpr bool PY = DIM == 3;
  constexpr int SUY = PY ? NTY + 2 : 1;
  return 8 * (NC * SUY * (NT + 2) + (WENO ? 2 : 0) * NC * NTY * NT + NC * NTY * NT +
              ((WENO && PY) ? 2 : 0) * NC * NTY * NT + (PY ? 3 * NC * NTY * NT : 0));
}

// ---------------------------------------------------------------------------
// Warp-strip kernel (1D and 2D; FVB_KERNEL=strip, an A/B alternative).
//
// Each WARP owns a strip of 30 cells in x (lanes 1..30; lanes 0 and 31 are
// the halo face cells) and marches along y over one chunk of rows.  x
// neighbours are exchanged with warp shuffles, so there is no shared memory
// and no block barrier at all; y uses the per-thread register window.  The
// row loop is unrolled by 4 with the window arrays rotated by name, so no
// register moves are spent on the march.
// ---------------------------------------------------------------------------
constexpr int kStripCells = 30;
#ifndef FVB_STRIP_MINB
#define FVB_STRIP_MINB 4
#endif

template <int NC>
__device__ __forceinline__ void shfl_up_nc(const double* v, double* out) {
#pragma unroll
  for (int c = 0; c < NC; ++c) out[c] = __shfl_up_sync(0xffffffffu, v[c], 1);
}
template <int NC>
__device__ __forceinline__ void shfl_down_nc(const double* v, double* out) {
#pragma unroll
  for (int c = 0; c < NC; ++c) out[c] = __shfl_down_sync(0xffffffffu, v[c], 1);
}

template <int DIM, int EQ, int FLUX, int RECON, bool FIN>
struct StripCtx {
  static constexpr int NC = NComp<EQ, DIM>::value;
  const StageParams& p;
  FvbState* st;
  const double* __restrict__ us;
  const double* un;
  double* out;
  double dt;
  int lane;
  int64_t x0, xf;
  bool cell;
  int64_t ra, rb;
  unsigned errb;
  double smax[DIM];
  int64_t xo;   // mapped x offset of this lane's column
  int64_t hxo;  // mapped x offset of the halo column (lanes 0 and 31)

  __device__ __forceinline__ int64_t roff(int64_t r) const {
    if constexpr (DIM == 1) return 0;
    else return map_index(r, p.n[1], p.bc[1], p.g) * p.sy;
  }
  __device__ __forceinline__ int64_t off(int64_t x, int64_t r) const {
    return map_index(x, p.n[0], p.bc[0], p.g) + roff(r);
  }
  __device__ __forceinline__ void load_row(int64_t r, double* v) const { load_nc<NC>(us, xo + roff(r), p.sc, v); }
  // halo value: lane 0 -> x0-2, lane 31 -> x0+31 (WENO only)
  __device__ __forceinline__ void load_halo(int64_t r, double* v) const {
    if constexpr (RECON != RECON_NONE) {
      if (lane == 0 || lane == 31) load_nc<NC>(us, hxo + roff(r), p.sc, v);
    }
  }

  // x direction of one row: returns the in-plane residual of this lane's cell
  __device__ __forceinline__ void xrow(const double* uc, const double* halo, double* res) {
    double um[NC], up[NC], hi[NC], lo[NC], hiL[NC], G[NC], Gn[NC];
    shfl_up_nc<NC>(uc, um);
    shfl_down_nc<NC>(uc, up);
    if constexpr (RECON != RECON_NONE) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        if (lane == 0) um[c] = halo[c];
        if (lane == 31) up[c] = halo[c];
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) weno_faces<RECON>(um[c], uc[c], up[c], p.P.eps, hi[c], lo[c]);
      shfl_up_nc<NC>(hi, hiL);
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c) { hiL[c] = um[c]; lo[c] = uc[c]; }
    }
    // interface (lane-1 | lane): uL = high face of lane-1, uR = low face of lane
    double uL[NC], uR[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) { uL[c] = hiL[c]; uR[c] = lo[c]; }
    unsigned eb = 0;
    interface_flux<EQ, FLUX, DIM, RECON>(uL, uR, um, uc, 0, p.P, G, eb);
    if (eb && lane >= 1 && xf <= p.n[0]) errb |= 1u;
    shfl_down_nc<NC>(G, Gn);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
#if FVB_FAST
      res[c] = (G[c] - Gn[c]) * p.id[0];
#else
      res[c] = 0.0 - ddiv(Gn[c] - G[c], p, 0);
#endif
    }
  }

  __device__ __forceinline__ void finish(int64_t r, const double* usc, const double* unc, const double* Lc) {
    double v[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) v[c] = rk_combine(p.kind, unc[c], usc[c], dt, Lc[c]);
    const int64_t o = xo + roff(r);
#pragma unroll
    for (int c = 0; c < NC; ++c) out[o + c * p.sc] = v[c];
    if constexpr (FIN) post_cell<EQ, DIM, NC>(p, st, v, xf, DIM == 2 ? r : 0, 0, smax);
  }

  __device__ __forceinline__ void stage_check(int64_t r, const double* uc) {
    if constexpr (EQ == EQ_EULER) {
      if (cell && !euler_physical<DIM>(uc, p.P)) {
        const long long key = ((long long)p.stage_idx << 42) | flat_cell<DIM>(p, xf, DIM == 2 ? r : 0, 0);
        atomicMin(&st->stage_err, key);
      }
    }
  }

  // One march row r.  On entry A,B,C = u[r-1], u[r], u[r+1]; on exit A
  // holds u[r+2] (loaded once A is dead), so the caller rotates (B, C, A).
  // H: high y-face of row r-1 -> r;  G: y flux (r-2|r-1) -> (r-1|r);
  // R: x residual of row r-1 -> r.
  __device__ __forceinline__ void row(int64_t r, double* A, const double* B, const double* C,
                                      double* H, double* G, double* R) {
    const bool in_row = r >= ra && r < rb;
    double halo[NC], unc[NC];
    if (in_row) load_halo(r, halo);
    const bool fin = cell && r - 1 >= ra;
    if (fin && p.kind >= 2) {
      const int64_t o = xo + roff(r - 1);
#pragma unroll
      for (int c = 0; c < NC; ++c) unc[c] = un[o + c * p.sc];
    }
    if (cell) {
      double hi[NC], lo[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) weno_faces<RECON>(A[c], B[c], C[c], p.P.eps, hi[c], lo[c]);
      if (r >= ra) {
        double uL[NC], uR[NC], GC[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) { uL[c] = H[c]; uR[c] = lo[c]; }
        unsigned eb = 0;
        interface_flux<EQ, FLUX, DIM, RECON>(uL, uR, A, B, 1, p.P, GC, eb);
        if (eb) errb |= 2u;
        if (fin) {
          double Lc[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) {
#if FVB_FAST
            Lc[c] = fma(G[c] - GC[c], p.id[1], R[c]);
#else
            Lc[c] = R[c] - ddiv(GC[c] - G[c], p, 1);
#endif
          }
          finish(r - 1, A, unc, Lc);
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) G[c] = GC[c];
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) H[c] = hi[c];
    }
    if (r + 2 <= rb + 1) load_row(r + 2, A);  // A is dead: prefetch the row after next
    if (in_row) {
      stage_check(r, B);
      xrow(B, halo, R);
    }
  }
};

template <int DIM, int EQ, int FLUX, int RECON, int WPB, bool FIN>
__global__ void __launch_bounds__(32 * WPB, FVB_STRIP_MINB)
strip_kernel(const StageParams p) {
  using S = StripCtx<DIM, EQ, FLUX, RECON, FIN>;
  constexpr int NC = S::NC;
  const int lane = threadIdx.x & 31;
  const int64_t strip = (int64_t)blockIdx.x * WPB + (threadIdx.x >> 5);
  const int inst = blockIdx.z;
  FvbState* st = p.st + (p.shared_state ? 0 : inst);
  if (*(volatile int*)&st->done) return;  // uniform over the grid
  const int64_t x0 = strip * kStripCells;
  S s{p, st, p.us + p.origin + inst * p.si, p.un + p.origin + inst * p.si, p.out + p.origin + inst * p.si,
      p.kind == 0 ? 0.0 : *(volatile double*)&st->dt, lane, x0, x0 - 1 + lane, false, 0, 1, 0u, {},
      map_index(x0 - 1 + lane, p.n[0], p.bc[0], p.g),
      map_index(lane == 0 ? x0 - 2 : x0 + 31, p.n[0], p.bc[0], p.g)};
#pragma unroll
  for (int k = 0; k < DIM; ++k) s.smax[k] = 0.0;
  const bool active = x0 < p.n[0];  // warp-uniform
  if (active) {
    s.cell = lane >= 1 && lane <= kStripCells && s.xf < p.n[0];
    if constexpr (DIM == 1) {
      double B[NC], halo[NC], res[NC], unc[NC];
      s.load_row(0, B);
      s.load_halo(0, halo);
      s.stage_check(0, B);
      s.xrow(B, halo, res);
      if (s.cell) {
        if (p.kind >= 2) {
#pragma unroll
          for (int c = 0; c < NC; ++c) unc[c] = s.un[s.xo + c * p.sc];
        }
        s.finish(0, B, unc, res);
      }
    } else {
      s.ra = p.row_lo + (int64_t)blockIdx.y * p.H;
      s.rb = min(s.ra + (int64_t)p.H, p.row_hi);
      double W0[NC], W1[NC], W2[NC], H[NC], G[NC], R[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) H[c] = G[c] = R[c] = 0.0;
      const int64_t ra = s.ra, rb = s.rb;
      s.load_row(ra - 2, W0);
      s.load_row(ra - 1, W1);
      s.load_row(ra, W2);
      // rows r = ra-1 .. rb, window rotated by name (period 3)
      for (int64_t r = ra - 1; r <= rb; r += 3) {
        s.row(r, W0, W1, W2, H, G, R);
        if (r + 1 > rb) break;
        s.row(r + 1, W1, W2, W0, H, G, R);
        if (r + 2 > rb) break;
        s.row(r + 2, W2, W0, W1, H, G, R);
      }
    }
    if (s.errb) {
#pragma unroll
      for (int a = 0; a < DIM; ++a)
        if (s.errb & (1u << a))
          atomicMin(&st->stage_err, ((long long)p.stage_idx << 42) | ((long long)(1 + a) << 40));
    }
  }
  if constexpr (FIN) block_epilogue<DIM>(p, st, inst, s.smax, true);
}

// ---------------------------------------------------------------------------
// 2D ring kernel (variant 2): the tile kernel with the march window moved
// out of registers into a shared-memory ring of rows filled by cp.async
// (LDGSTS) PD rows ahead.  Loads never stall the math (no long-scoreboard
// waits, no register moves of freshly loaded data), the x phase reads its
// row straight from the ring (no staging store), and the 24 window
// registers are freed for occupancy.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

#ifndef FVB_PDL
#define FVB_PDL 1
#endif
#ifndef FVB_RING_MINB
#define FVB_RING_MINB (512 / NT)  // 16 warps/SM at 128 registers
#endif
#ifndef FVB_RING_PD
#define FVB_RING_PD 1  // measured (profiles/r01_ring_pd_sweep.json): 1 row ahead +1 % over 2; 3-4 exceed the shared memory of 8 blocks/SM
#endif
constexpr int kRingPD = FVB_RING_PD;     // rows in flight ahead of the consumer
constexpr int kRingRows = kRingPD + 3;   // ring slots
#ifndef FVB_RING_XSHFL
#define FVB_RING_XSHFL 1
#endif
template <int NT>
constexpr bool kXShfl = FVB_RING_XSHFL && NT > 32 && NT % 32 == 0;  // hybrid shuffle x faces

// NI > 1 (scalar laws, batched ensembles): one block marches the same
// strip of NI instances at once -- the instances are "virtual components"
// (component stride = instance stride), so the row bookkeeping, barriers
// and copies are shared and the per-instance math interleaves.
// KS (stage combination, compile time): 0 = the residual L itself
// (spatial_residual); 1 = u^s + dt L (forward Euler, RK stage 1);
// 2 = a u^n + b (u^s + dt L) (later SSP-RK stages, a/b per p.kind).
template <int EQ, int FLUX, int RECON, int NT, int KS, bool FIN, int NI = 1>
__global__ void __launch_bounds__(NT, FVB_RING_MINB)
ring_kernel(const StageParams p) {
  constexpr int DIM = 2;
  constexpr int NCP = NComp<EQ, DIM>::value;  // physical components
  static_assert(NI == 1 || NCP == 1, "instance batching is for scalar laws");
  constexpr int NC = NCP * NI;                // components held per cell here
  // one-warp blocks: the x neighbours are lanes of the warp -> the x sweep
  // runs on shuffles, and gx holds each column's own x residual
  constexpr bool kShflX = NT == 32;
  constexpr bool WENO = RECON != RECON_NONE;
  constexpr bool UN = KS == 2;                // the stage reads u^n
  static_assert(!UN || kRingPD == 1, "the 2-slot u^n ring assumes one ring row in flight");
  constexpr int W = NT + 2;
  extern __shared__ double smem[];
  double* ring = smem;                               // [kRingRows][NC][W]
  // x faces: one-warp blocks exchange them by shuffle; wider blocks shuffle
  // inside each warp and pass only the high face of every warp's last lane
  // through shared memory (kXShfl), or stage all faces (hx / lx)
  constexpr bool kFaceBuf = WENO && NT != 32 && !kXShfl<NT>;
  double* hx = ring + kRingRows * NC * W;            // [NC][NT]
  double* lx = hx + (kFaceBuf ? NC * NT : 0);        // [NC][NT]
  double* bnd = lx + (kFaceBuf ? NC * NT : 0);       // [NT/32][NC] (kXShfl)
  double* gx = bnd + (WENO && kXShfl<NT> ? NC * (NT / 32) : 0);  // [NC][NT]
  double* nring = gx + NC * NT;                      // [2][NC][NT]: u^n rows for the RK combination
  // march recurrence (high face H and flux G of the previous row) lives in
  // shared memory, not registers: it is idle during the whole x sweep
  double* hs = nring + 2 * NC * NT;                  // [NC][NT]
  double* gs = hs + NC * NT;                         // [NC][NT]
  auto RG = [&](int slot, int c, int x) -> double& { return ring[(slot * NC + c) * W + x]; };
  auto NR = [&](int slot, int c) -> double& { return nring[(slot * NC + c) * NT + threadIdx.x]; };

#if FVB_PDL
  // programmatic dependent launch: this grid may be scheduled while the
  // previous stage drains; nothing it reads is touched before the wait
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
#endif
  const int inst = blockIdx.z * NI;
  FvbState* st = p.st + (p.shared_state ? 0 : inst);
  FvbState* sts[NI];
  double dts[NI];
  bool act[NI];
  bool any = false;
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    sts[i] = p.st + (p.shared_state ? 0 : inst + i);
    act[i] = !*(volatile int*)&sts[i]->done;
    any = any || act[i];
    dts[i] = KS == 0 ? 0.0 : *(volatile double*)&sts[i]->dt;
  }
  if (!any) return;
  const double dt = dts[0];
  // 32-bit element offsets inside one instance (fvb_capi.cu checks the
  // instance fits); one 64-bit base per block
  const int cs = (int)(NI > 1 ? p.si : p.sc);  // stride between the components held here
  const double* __restrict__ us = p.us + p.origin + inst * p.si;
  const double* un = p.un + p.origin + inst * p.si;
  double* out = p.out + p.origin + inst * p.si;
  const int tx = threadIdx.x;
  const int x0 = (int)p.x_lo + blockIdx.x * (NT - 2);
  const int xf = x0 - 1 + tx;
  const int nx = (int)p.n[0];
  const bool cell = tx >= 1 && tx <= NT - 2 && xf < (int)p.x_hi;
  const int ra = (int)p.row_lo + blockIdx.y * p.H;
  const int rb = min(ra + p.H, (int)p.row_hi);
  const int co = (int)map_index(xf, nx, p.bc[0], p.g);
  // halo columns: thread 0 also copies x0-2, thread NT-1 also x0+NT-1
  const bool halo_t = WENO && (tx == 0 || tx == NT - 1);
  const int hco = (int)map_index(tx == 0 ? x0 - 2 : x0 + NT - 1, nx, p.bc[0], p.g);
  const int hcol = tx == 0 ? 0 : NT + 1;
  // row offsets of rows ra-2 .. rb+PD+1, computed once per block
  int* rtab = reinterpret_cast<int*>(gs + NC * NT);
  for (int i = tx; i < p.H + kRingPD + 4; i += NT) rtab[i] = (int)(map_index(ra - 2 + i, p.n[1], p.bc[1], p.g) * p.sy);
  __syncthreads();
  auto roff = [&](int r) -> int { return rtab[r - (ra - 2)]; };
  auto fetch = [&](int r, int slot) {  // async copy of row r into a ring slot
    const int ro = roff(r);
#pragma unroll
    for (int c = 0; c < NC; ++c) cp_async8(&RG(slot, c, tx + 1), us + (co + ro + c * cs));
    if (halo_t) {
#pragma unroll
      for (int c = 0; c < NC; ++c) cp_async8(&RG(slot, c, hcol), us + (hco + ro + c * cs));
    }
  };

  unsigned errb = 0, errbs[NI];
  double smax[DIM] = {0.0, 0.0}, smaxs[NI][DIM];
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    errbs[i] = 0;
    smaxs[i][0] = smaxs[i][1] = 0.0;
  }
  // RK stage as a*u^n + b*(u^s + dt L) (solver.py:166-173); fast mode folds
  // b, dt and 1/delta into the flux differences
  const double rk_a = p.kind == 2 ? 0.5 : (p.kind == 3 ? 0.75 : (p.kind == 4 ? 1.0 / 3.0 : 0.0));
  const double rk_b = p.kind == 2 ? 0.5 : (p.kind == 3 ? 0.25 : (p.kind == 4 ? 2.0 / 3.0 : 1.0));
#if FVB_FAST
  const double cx = KS == 0 ? p.id[0] : (KS == 1 ? dt * p.id[0] : rk_b * dt * p.id[0]);
  const double cy = KS == 0 ? p.id[1] : (KS == 1 ? dt * p.id[1] : rk_b * dt * p.id[1]);
#endif

  // prologue: rows ra-2 .. ra-1+PD (slot of row r = (r - ra + 2) % kRingRows)
  for (int k = 0; k < kRingPD + 2; ++k) {
    fetch(ra - 2 + k, k);
    cp_async_commit();
  }
  int sA = 0;   // slot of row r-1 at the top of the loop (r = ra-1 -> row ra-2)
  int nsw = 1;  // u^n slot written this iteration (row r): (r - ra) & 1
                // -- each thread's own column: no cross-thread hazard
  for (int r = ra - 1; r <= rb; ++r) {
    const int sB = sA + 1 == kRingRows ? 0 : sA + 1;
    const int sC = sB + 1 == kRingRows ? 0 : sB + 1;
    // iteration ra-1 has no in-plane barrier: make sure its reads of the
    // slot about to be refilled (row ra-2) are done
    if (r == ra) __syncthreads();
    // issue row r+1+PD into the slot that held row r-2 (free since last row),
    // and u^n of row r (consumed by the next iteration's finish) into its
    // 2-slot ring
    {
      int sN = sC + kRingPD;  // slot(row) = (row - ra + 2) % kRingRows -> the slot of row r-2
      sN = sN >= kRingRows ? sN - kRingRows : sN;
      if (r + 1 + kRingPD <= rb + 1) fetch(r + 1 + kRingPD, sN);
      if constexpr (UN) {
        nsw ^= 1;
        if (cell && r >= ra && r < rb) {
          const int o = co + roff(r);
#pragma unroll
          for (int c = 0; c < NC; ++c) cp_async8(&NR(nsw, c), un + (o + c * cs));
        }
      }
      cp_async_commit();
    }
    cp_async_wait<kRingPD>();  // rows up to r+1 have landed (this thread's copies)
    __syncthreads();           // ... and everybody's
    // Every lane computes (the two halo lanes on real neighbour columns), only
    // side effects are predicated on `cell`: no divergent regions, so no
    // reconvergence bookkeeping in the hot loop.
    const bool fin = cell && r - 1 >= ra;
    double B[NC];  // row r of this column: the march stencil's centre and the x sweep's
#pragma unroll
    for (int c = 0; c < NC; ++c) B[c] = RG(sB, c, tx + 1);
    {  // march (y) direction: faces of row r, flux (r-1|r), finish row r-1
      double A[NC], C[NC], hi[NC], lo[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        A[c] = RG(sA, c, tx + 1);
        C[c] = RG(sC, c, tx + 1);
      }
      weno_faces_nc<NC, RECON>(A, B, C, p.P.eps, hi, lo);
      if (r >= ra) {
        double GC[NC], H[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) H[c] = hs[c * NT + tx];
        if constexpr (NI == 1) {
          unsigned eb = 0;
          interface_flux<EQ, FLUX, DIM, RECON>(H, lo, A, B, 1, p.P, GC, eb);
          if (eb && cell) errb |= 2u;
        } else {
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            unsigned eb = 0;
            interface_flux<EQ, FLUX, DIM, RECON>(H + i, lo + i, A + i, B + i, 1, p.P, GC + i, eb);
            if (eb && cell) errbs[i] |= 2u;
          }
        }
        double unc[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) unc[c] = 0.0;
        if constexpr (UN) {
          if (r - 1 >= ra) {  // u^n of row r-1 landed with the group of iteration r-1
#pragma unroll
            for (int c = 0; c < NC; ++c) unc[c] = NR(nsw ^ 1, c);
          }
        }
        double v[NC];
        const int tr = tx + 1 < NT ? tx + 1 : NT - 1;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const double Gp = gs[c * NT + tx];
#if FVB_FAST
          // x: gx holds the raw fluxes (two-warp blocks) or this column's own
          // difference (shuffle x sweep, already scaled by 1/dx)
          if constexpr (NI == 1) {
            double base = KS == 0 ? 0.0 : (KS == 1 ? A[c] : fma(rk_b, A[c], rk_a * unc[c]));
            if constexpr (kShflX) {
              base = fma(KS == 0 ? 1.0 : (KS == 1 ? dt : rk_b * dt), gx[c * NT + tx], base);
            } else {
              base = fma(cx, gx[c * NT + tx] - gx[c * NT + tr], base);
            }
            v[c] = fma(cy, Gp - GC[c], base);
          } else {  // per-instance dt (the instances of a batch differ)
            const double dtc = dts[c];
            const double xs = kShflX ? gx[c * NT + tx] : (gx[c * NT + tx] - gx[c * NT + tr]) * p.id[0];
            const double Lc = fma(Gp - GC[c], p.id[1], xs);
            v[c] = KS == 0 ? Lc : (KS == 1 ? fma(dtc, Lc, A[c]) : fma(rk_a, unc[c], rk_b * fma(dtc, Lc, A[c])));
          }
#else
          double xres;
          if constexpr (kShflX) {
            xres = gx[c * NT + tx];  // this column's own, computed by the x sweep
          } else {
            const double g0 = gx[c * NT + tx], g1 = gx[c * NT + tr];
            xres = 0.0 - ddiv(g1 - g0, p, 0);
          }
          const double Lc = xres - ddiv(GC[c] - Gp, p, 1);
          v[c] = KS == 0 ? Lc : rk_combine(p.kind, unc[c], A[c], NI > 1 ? dts[c] : dt, Lc);
#endif
        }
        if (fin) {
          const int o = co + roff(r - 1);
          if constexpr (NI == 1) {
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              out[o + c * cs] = v[c];
              peer_store(p, o, r - 1, cs, c, v[c]);
            }
            if constexpr (FIN) post_cell<EQ, DIM, NC>(p, st, v, xf, r - 1, 0, smax);
          } else {
#pragma unroll
            for (int i = 0; i < NI; ++i) {
              if (act[i]) {
                out[o + i * cs] = v[i];
                if constexpr (FIN) post_cell<EQ, DIM, NCP>(p, sts[i], v + i, xf, r - 1, 0, smaxs[i]);
              }
            }
          }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) gs[c * NT + tx] = GC[c];
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) hs[c * NT + tx] = hi[c];
    }
    if (r >= ra && r < rb) {  // in-plane (x) direction of row r, straight from the ring
      if constexpr (EQ == EQ_EULER) {
        if (p.check_input && cell) {
          if (!euler_physical<DIM>(B, p.P))
            atomicMin(&st->stage_err, ((long long)p.stage_idx << 42) | flat_cell<DIM>(p, xf, r, 0));
        }
      }
      if constexpr (kShflX) {  // x sweep on shuffles: no shared-memory faces, no barrier
        double uL[NC], uR[NC], Gx[NC];
        if constexpr (WENO) {
          double um[NC], uc[NC], up[NC], hi[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            um[c] = RG(sB, c, tx);
            uc[c] = B[c];
            up[c] = RG(sB, c, tx + 2);
          }
          weno_faces_nc<NC, RECON>(um, uc, up, p.P.eps, hi, uR);
#pragma unroll
          for (int c = 0; c < NC; ++c) uL[c] = __shfl_up_sync(0xffffffffu, hi[c], 1);
        } else {
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            uL[c] = RG(sB, c, tx);
            uR[c] = RG(sB, c, tx + 1);
          }
        }
        if constexpr (NI == 1) {
          auto cells = [&](double* a, double* b) {  // fallback only: loaded on demand
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              a[c] = RG(sB, c, tx);
              b[c] = RG(sB, c, tx + 1);
            }
          };
          unsigned eb = 0;
          interface_flux_lazy<EQ, FLUX, DIM, RECON>(uL, uR, cells, 0, p.P, Gx, eb);
          if (eb && tx >= 1 && xf <= nx) errb |= 1u;
        } else {
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            unsigned eb = 0;
            interface_flux<EQ, FLUX, DIM, RECON>(uL + i, uR + i, uL + i, uR + i, 0, p.P, Gx + i, eb);
            if (eb && tx >= 1 && xf <= nx) errbs[i] |= 1u;
          }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const double Gr = __shfl_down_sync(0xffffffffu, Gx[c], 1);  // lane 31's is unused
#if FVB_FAST
          gx[c * NT + tx] = (Gx[c] - Gr) * p.id[0];
#else
          gx[c * NT + tx] = 0.0 - ddiv(Gr - Gx[c], p, 0);
#endif
        }
      } else {
      double uL[NC], uR[NC];
      if constexpr (WENO) {
        double um[NC], uc[NC], up[NC], hi[NC], lo[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          um[c] = RG(sB, c, tx);
          uc[c] = B[c];
          up[c] = RG(sB, c, tx + 2);
        }
        weno_faces_nc<NC, RECON>(um, uc, up, p.P.eps, hi, lo);
        if constexpr (kXShfl<NT>) {
          const int lane = tx & 31;
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            uR[c] = lo[c];
            uL[c] = __shfl_up_sync(0xffffffffu, hi[c], 1);
            if (lane == 31) bnd[(tx >> 5) * NC + c] = hi[c];
          }
          __syncthreads();
          if (lane == 0 && tx > 0) {
#pragma unroll
            for (int c = 0; c < NC; ++c) uL[c] = bnd[((tx >> 5) - 1) * NC + c];
          }
        } else {
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            hx[c * NT + tx] = hi[c];
            lx[c * NT + tx] = lo[c];
          }
          __syncthreads();
        }
      }
      if constexpr (!WENO) __syncthreads();  // every lane has read row r-1's gx
      {  // x interface tx sits between face cells tx-1 and tx (lane 0's is unused)
        const int tl = tx >= 1 ? tx - 1 : 0;
        double Gx[NC];
        if constexpr (!(WENO && kXShfl<NT>)) {
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            uL[c] = WENO ? hx[c * NT + tl] : RG(sB, c, tx);
            uR[c] = WENO ? lx[c * NT + tx] : RG(sB, c, tx + 1);
          }
        }
        if constexpr (NI == 1) {
          auto cells = [&](double* a, double* b) {  // fallback only: loaded on demand
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              a[c] = RG(sB, c, tx);
              b[c] = RG(sB, c, tx + 1);
            }
          };
          unsigned eb = 0;
          interface_flux_lazy<EQ, FLUX, DIM, RECON>(uL, uR, cells, 0, p.P, Gx, eb);
          if (eb && tx >= 1 && xf <= nx) errb |= 1u;
        } else {  // scalar laws: no positivity fallback, the cells are never read
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            unsigned eb = 0;
            interface_flux<EQ, FLUX, DIM, RECON>(uL + i, uR + i, uL + i, uR + i, 0, p.P, Gx + i, eb);
            if (eb && tx >= 1 && xf <= nx) errbs[i] |= 1u;
          }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) gx[c * NT + tx] = Gx[c];
      }
      }
      // the x residual of this row is read from gx by the next iteration's
      // finish, after that iteration's top barrier
    }
    sA = sB;
  }
  cp_async_wait<0>();
#if FVB_PDL
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");  // this block's stage work is done
#endif
  if constexpr (NI == 1) {
    if (errb) {
#pragma unroll
      for (int a = 0; a < DIM; ++a)
        if (errb & (1u << a))
          atomicMin(&st->stage_err, ((long long)p.stage_idx << 42) | ((long long)(1 + a) << 40));
    }
    if constexpr (FIN) block_epilogue<DIM>(p, st, inst, smax, true);
  } else {
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      if (!act[i]) continue;  // block-uniform
      if (errbs[i]) {
#pragma unroll
        for (int a = 0; a < DIM; ++a)
          if (errbs[i] & (1u << a))
            atomicMin(&sts[i]->stage_err, ((long long)p.stage_idx << 42) | ((long long)(1 + a) << 40));
      }
      if constexpr (FIN) block_epilogue<DIM>(p, sts[i], inst + i, smaxs[i], true);
    }
  }
}

template <int EQ, int RECON, int NT, int NI = 1>
constexpr int ring_smem_bytes() {
  constexpr int NC = NComp<EQ, 2>::value * NI;
  constexpr bool weno = RECON != RECON_NONE;
  return 8 * (kRingRows * NC * (NT + 2) + (weno && NT != 32 && !kXShfl<NT> ? 2 : 0) * NC * NT +
              (weno && kXShfl<NT> ? NC * (NT / 32) : 0) + NC * NT + 2 * NC * NT + 2 * NC * NT);
}

// ---------------------------------------------------------------------------
// 2D pair kernel: the ring kernel with TWO x-columns per thread.
//
// A one-warp block owns 62 x-cells (64 face cells: lane t holds face cells
// f0 = x0-1+2t and f1 = f0+1, lane 0's f0 and lane 31's f1 are the halo
// face cells) and marches H rows in y.  Per thread and row: two WENO
// stencils per axis, the x interface between its own two cells computed
// in-thread and one more with the neighbour lane's face (shuffle), two y
// interfaces -- two independent chains of the same physics interleave
// (ILP 2), and the per-row bookkeeping (ring copies, slot rotation, march
// recurrence, stores) is shared by two cells: ring rows arrive by 16-byte
// cp.async (pairs of cells; 8-byte copies where a pair is not contiguous:
// outflow edges, odd periodic extents), the x stencil and the march
// recurrence move as 16-byte shared-memory accesses, and a one-warp block
// synchronises with __syncwarp only.  Same operation order as the ring
// kernel, so the exact mode stays bitwise.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}

#ifndef FVB_BLOCK_TIMES
#define FVB_BLOCK_TIMES 0  // 1: record per-block start/end (globaltimer) and SM of the last pair-kernel launch per stage
#endif
#if FVB_BLOCK_TIMES
__device__ unsigned long long g_bt[3][8192][2];
__device__ unsigned g_bt_sm[3][8192];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif
constexpr int kPairNT = 32;                // one warp
constexpr int kPairW = 2 * kPairNT + 2;    // ring row width: cells x0-2 .. x0+63

#ifndef FVB_PAIR_MINB
#define FVB_PAIR_MINB 12  // <= 168 registers: 12 one-warp blocks/SM (measured: 23.5 vs 22.9 at 8, 17.8 at 14 -- spills)
#endif

template <int EQ, int FLUX, int RECON, int KS, bool FIN>
__global__ void __launch_bounds__(kPairNT, FVB_PAIR_MINB)
pair_kernel(const StageParams p) {
  constexpr int DIM = 2;
  constexpr int NC = NComp<EQ, DIM>::value;
  constexpr int W = kPairW;
  constexpr bool UN = KS == 2;
  static_assert(!UN || kRingPD == 1, "the 2-slot u^n ring assumes one ring row in flight");
  extern __shared__ __align__(16) double smem[];
  double* ring = smem;                          // [kRingRows][NC][W]
  double* gx = ring + kRingRows * NC * W;       // [NC][64]: x residual of each face cell (own column pair)
  double* nrow = gx + NC * 64;                  // [NC][64]: u^n of the row finished next
  double* hs = nrow + NC * 64;                  // [NC][64]: high y face of the previous row
  double* gs = hs + NC * 64;                    // [NC][64]: y flux below the previous row
  auto RG = [&](int slot, int c, int x) -> double& { return ring[(slot * NC + c) * W + x]; };

#if FVB_PDL
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
#endif
#if FVB_BLOCK_TIMES
  const unsigned long long bt0 = gtimer();
#endif
  const int inst = blockIdx.z;
  FvbState* st = p.st + (p.shared_state ? 0 : inst);
  if (*(volatile int*)&st->done) return;
  const double dt = KS == 0 ? 0.0 : *(volatile double*)&st->dt;
  const int cs = (int)p.sc;
  const double* __restrict__ us = p.us + p.origin + inst * p.si;
  const double* un = p.un + p.origin + inst * p.si;
  double* out = p.out + p.origin + inst * p.si;
  const int t = threadIdx.x;
  const int nx = (int)p.n[0];
  const int x0 = (int)p.x_lo + blockIdx.x * (2 * kPairNT - 2);
  const int f0 = x0 - 1 + 2 * t;                     // face cells f0, f0+1 of this lane
  const int xh = (int)p.x_hi;
  const bool cell0 = t >= 1 && f0 < xh;              // updated cells (lane 0's f0 is the halo face cell)
  const bool cell1 = t <= kPairNT - 2 && f0 + 1 < xh;
  const int ra = (int)p.row_lo + blockIdx.y * p.H;
  const int rb = min(ra + p.H, (int)p.row_hi);
  const int co0 = (int)map_index(f0, nx, p.bc[0], p.g), co1 = (int)map_index(f0 + 1, nx, p.bc[0], p.g);
  // ring pair j = cells (x0-2+2j, x0-1+2j): lane t copies pair t, lane 0 also pair 32
  const int pa = (int)map_index(x0 - 2 + 2 * t, nx, p.bc[0], p.g);
  const int pb = (int)map_index(x0 - 1 + 2 * t, nx, p.bc[0], p.g);
  const int qa = (int)map_index(x0 + 62, nx, p.bc[0], p.g), qb = (int)map_index(x0 + 63, nx, p.bc[0], p.g);
  // 16-byte copies need the pair contiguous and 16-byte aligned in memory
  const bool vec = ((((int64_t)p.origin + pa) & 1) == 0) && pb == pa + 1 && qb == qa + 1 &&
                   ((reinterpret_cast<uintptr_t>(p.us) & 15) == 0) && ((p.sy & 1) == 0) && ((cs & 1) == 0);
  const bool vec_all = __all_sync(0xffffffffu, vec);
  int* rtab = reinterpret_cast<int*>(gs + NC * 64);
  for (int i = t; i < p.H + kRingPD + 4; i += kPairNT)
    rtab[i] = (int)(map_index(ra - 2 + i, p.n[1], p.bc[1], p.g) * p.sy);
  __syncwarp();
  auto roff = [&](int r) -> int { return rtab[r - (ra - 2)]; };
  auto fetch = [&](int r, int slot) {
    const int ro = roff(r);
    if (vec_all) {
#pragma unroll
      for (int c = 0; c < NC; ++c) cp_async16(&RG(slot, c, 2 * t), us + (pa + ro + c * cs));
      // pair 32 (cells x0+62, x0+63): one component per lane, in parallel
      if (t < NC) cp_async16(&RG(slot, t, 64), us + (qa + ro + t * cs));
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        cp_async8(&RG(slot, c, 2 * t), us + (pa + ro + c * cs));
        cp_async8(&RG(slot, c, 2 * t + 1), us + (pb + ro + c * cs));
      }
      if (t < NC) {
        cp_async8(&RG(slot, t, 64), us + (qa + ro + t * cs));
        cp_async8(&RG(slot, t, 65), us + (qb + ro + t * cs));
      }
    }
  };

  unsigned errb = 0;
  double smax[DIM] = {0.0, 0.0};
  const double rk_a = p.kind == 2 ? 0.5 : (p.kind == 3 ? 0.75 : (p.kind == 4 ? 1.0 / 3.0 : 0.0));
  const double rk_b = p.kind == 2 ? 0.5 : (p.kind == 3 ? 0.25 : (p.kind == 4 ? 2.0 / 3.0 : 1.0));
#if FVB_FAST
  const double cxs = KS == 0 ? 1.0 : (KS == 1 ? dt : rk_b * dt);  // gx is already scaled by 1/dx
  const double cy = KS == 0 ? p.id[1] : (KS == 1 ? dt * p.id[1] : rk_b * dt * p.id[1]);
#endif

  for (int k = 0; k < kRingPD + 2; ++k) {
    fetch(ra - 2 + k, k);
    cp_async_commit();
  }
  // u^n of row r (finished at iteration r+1) is copied into the single
  // per-lane slot right after iteration r's finish read it, in its own
  // commit group -- the next iteration's wait covers it
  auto fetch_un = [&](int r) {
    if constexpr (UN) {
      if (r >= ra && r < rb) {
        const int o = roff(r);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          if (cell0) cp_async8(&nrow[c * 64 + 2 * t], un + (co0 + o + c * cs));
          if (cell1) cp_async8(&nrow[c * 64 + 2 * t + 1], un + (co1 + o + c * cs));
        }
      }
      cp_async_commit();
    }
  };
  int sA = 0;
  for (int r = ra - 1; r <= rb; ++r) {
    const int sB = sA + 1 == kRingRows ? 0 : sA + 1;
    const int sC = sB + 1 == kRingRows ? 0 : sB + 1;
    if (r == ra) __syncwarp();
    {
      int sN = sC + kRingPD;
      sN = sN >= kRingRows ? sN - kRingRows : sN;
      if (r + 1 + kRingPD <= rb + 1) fetch(r + 1 + kRingPD, sN);
      cp_async_commit();
    }
    // groups pending: [u^n of row r-1 (UN), ring row r+1+PD]; everything
    // older -- ring rows up to r+1 and u^n of row r-1 -- must have landed
    cp_async_wait<kRingPD>();
    __syncwarp();
    // row r of this lane's stencil: p0..p3 = cells f0-1, f0, f1, f1+1
    double P0[NC], P1[NC], P2[NC], P3[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double2 lo2 = *reinterpret_cast<const double2*>(&RG(sB, c, 2 * t));
      const double2 hi2 = *reinterpret_cast<const double2*>(&RG(sB, c, 2 * t + 2));
      P0[c] = lo2.x;
      P1[c] = lo2.y;
      P2[c] = hi2.x;
      P3[c] = hi2.y;
    }
    {  // march (y): faces of row r, fluxes (r-1|r), finish row r-1 -- both columns
      double A0[NC], A1[NC], C0[NC], C1[NC], hi0[NC], lo0[NC], hi1[NC], lo1[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        A0[c] = RG(sA, c, 2 * t + 1);
        A1[c] = RG(sA, c, 2 * t + 2);
        C0[c] = RG(sC, c, 2 * t + 1);
        C1[c] = RG(sC, c, 2 * t + 2);
      }
      weno_faces_nc<NC, RECON>(A0, P1, C0, p.P.eps, hi0, lo0);
      weno_faces_nc<NC, RECON>(A1, P2, C1, p.P.eps, hi1, lo1);
      if (r >= ra) {
        double H0[NC], H1[NC], G0[NC], G1[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const double2 h = *reinterpret_cast<const double2*>(&hs[c * 64 + 2 * t]);
          H0[c] = h.x;
          H1[c] = h.y;
        }
        unsigned eb0 = 0, eb1 = 0;
        // fallback cells reloaded from the ring only when needed: no stencil
        // registers held live across the flux
        interface_flux_lazy<EQ, FLUX, DIM, RECON>(H0, lo0, [&](double* a, double* b) {
#pragma unroll
          for (int c = 0; c < NC; ++c) { a[c] = RG(sA, c, 2 * t + 1); b[c] = RG(sB, c, 2 * t + 1); }
        }, 1, p.P, G0, eb0);
        interface_flux_lazy<EQ, FLUX, DIM, RECON>(H1, lo1, [&](double* a, double* b) {
#pragma unroll
          for (int c = 0; c < NC; ++c) { a[c] = RG(sA, c, 2 * t + 2); b[c] = RG(sB, c, 2 * t + 2); }
        }, 1, p.P, G1, eb1);
        if ((eb0 && cell0) || (eb1 && cell1)) errb |= 2u;
        if (r - 1 >= ra) {
          double v0[NC], v1[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const double2 gp = *reinterpret_cast<const double2*>(&gs[c * 64 + 2 * t]);
            const double2 xr = *reinterpret_cast<const double2*>(&gx[c * 64 + 2 * t]);
            double un0 = 0.0, un1 = 0.0;
            if constexpr (UN) {
              const double2 u2 = *reinterpret_cast<const double2*>(&nrow[c * 64 + 2 * t]);
              un0 = u2.x;
              un1 = u2.y;
            }
#if FVB_FAST
            const double a0c = RG(sA, c, 2 * t + 1), a1c = RG(sA, c, 2 * t + 2);  // u^s of row r-1, re-read
            double b0 = KS == 0 ? 0.0 : (KS == 1 ? a0c : fma(rk_b, a0c, rk_a * un0));
            double b1 = KS == 0 ? 0.0 : (KS == 1 ? a1c : fma(rk_b, a1c, rk_a * un1));
            v0[c] = fma(cy, gp.x - G0[c], fma(cxs, xr.x, b0));
            v1[c] = fma(cy, gp.y - G1[c], fma(cxs, xr.y, b1));
#else
            const double L0 = xr.x - ddiv(G0[c] - gp.x, p, 1);
            const double L1 = xr.y - ddiv(G1[c] - gp.y, p, 1);
            v0[c] = KS == 0 ? L0 : rk_combine(p.kind, un0, A0[c], dt, L0);
            v1[c] = KS == 0 ? L1 : rk_combine(p.kind, un1, A1[c], dt, L1);
#endif
          }
          const int o = roff(r - 1);
          if (cell0) {
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              out[co0 + o + c * cs] = v0[c];
              peer_store(p, co0 + o, r - 1, cs, c, v0[c]);
            }
            if constexpr (FIN) post_cell<EQ, DIM, NC>(p, st, v0, f0, r - 1, 0, smax);
          }
          if (cell1) {
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              out[co1 + o + c * cs] = v1[c];
              peer_store(p, co1 + o, r - 1, cs, c, v1[c]);
            }
            if constexpr (FIN) post_cell<EQ, DIM, NC>(p, st, v1, f0 + 1, r - 1, 0, smax);
          }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) *reinterpret_cast<double2*>(&gs[c * 64 + 2 * t]) = make_double2(G0[c], G1[c]);
      }
      fetch_un(r);  // the slot was read above (row r-1): refill with row r
#pragma unroll
      for (int c = 0; c < NC; ++c) *reinterpret_cast<double2*>(&hs[c * 64 + 2 * t]) = make_double2(hi0[c], hi1[c]);
    }
    if (r >= ra && r < rb) {  // x direction of row r
      if constexpr (EQ == EQ_EULER) {
        if (p.check_input) {
          const bool bad0 = cell0 && !euler_physical<DIM>(P1, p.P);
          const bool bad1 = cell1 && !euler_physical<DIM>(P2, p.P);
          if (bad0 || bad1)
            atomicMin(&st->stage_err, ((long long)p.stage_idx << 42) | flat_cell<DIM>(p, bad0 ? f0 : f0 + 1, r, 0));
        }
      }
      double hi0[NC], lo0[NC], hi1[NC], lo1[NC];
      weno_faces_nc<NC, RECON>(P0, P1, P2, p.P.eps, hi0, lo0);
      weno_faces_nc<NC, RECON>(P1, P2, P3, p.P.eps, hi1, lo1);
      double uLa[NC], Ga[NC], Gb[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) uLa[c] = __shfl_up_sync(0xffffffffu, hi1[c], 1);  // f0-1's high face
      unsigned eba = 0, ebb = 0;
      // interface (f0-1 | f0): cells P0, P1; interface (f0 | f1): cells P1, P2 (fallback operands)
      interface_flux_lazy<EQ, FLUX, DIM, RECON>(uLa, lo0, [&](double* a, double* b) {
#pragma unroll
        for (int c = 0; c < NC; ++c) { a[c] = RG(sB, c, 2 * t); b[c] = RG(sB, c, 2 * t + 1); }
      }, 0, p.P, Ga, eba);
      interface_flux_lazy<EQ, FLUX, DIM, RECON>(hi0, lo1, [&](double* a, double* b) {
#pragma unroll
        for (int c = 0; c < NC; ++c) { a[c] = RG(sB, c, 2 * t + 1); b[c] = RG(sB, c, 2 * t + 2); }
      }, 0, p.P, Gb, ebb);
      if ((eba && t >= 1 && f0 <= nx) || (ebb && f0 + 1 <= nx)) errb |= 1u;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double Gc = __shfl_down_sync(0xffffffffu, Ga[c], 1);  // (f1 | f1+1) of the next lane
#if FVB_FAST
        *reinterpret_cast<double2*>(&gx[c * 64 + 2 * t]) = make_double2((Ga[c] - Gb[c]) * p.id[0],
                                                                         (Gb[c] - Gc) * p.id[0]);
#else
        *reinterpret_cast<double2*>(&gx[c * 64 + 2 * t]) = make_double2(0.0 - ddiv(Gb[c] - Ga[c], p, 0),
                                                                         0.0 - ddiv(Gc - Gb[c], p, 0));
#endif
      }
    }
    sA = sB;
  }
  cp_async_wait<0>();
#if FVB_PDL
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#endif
  if (errb) {
#pragma unroll
    for (int a = 0; a < DIM; ++a)
      if (errb & (1u << a))
        atomicMin(&st->stage_err, ((long long)p.stage_idx << 42) | ((long long)(1 + a) << 40));
  }
  if constexpr (FIN) block_epilogue<DIM>(p, st, inst, smax, true);
#if FVB_BLOCK_TIMES
  if (threadIdx.x == 0 && p.stage_idx < 3) {
    const unsigned b = blockIdx.y * gridDim.x + blockIdx.x;
    if (b < 8192) {
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      g_bt[p.stage_idx][b][0] = bt0;
      g_bt[p.stage_idx][b][1] = gtimer();
      g_bt_sm[p.stage_idx][b] = sm;
    }
  }
#endif
}

template <int EQ>
constexpr int pair_smem_bytes() {
  constexpr int NC = NComp<EQ, 2>::value;
  return 8 * (kRingRows * NC * kPairW + NC * 64 + NC * 64 + 2 * NC * 64);
}

// ---------------------------------------------------------------------------
// 3D ring kernel (variant 2 in 3D): the 2D ring design on an in-plane tile.
//
// A block of 32 x 8 threads owns the 30 x 6 interior cells of its (x, y)
// tile (thread <-> face cell, the outer ring of threads are the halo face
// cells) and marches H planes along z.  Planes of the tile, WENO halos
// included, stream into a 4-slot shared-memory ring by cp.async one plane
// ahead, so no load ever stalls the math and the halo reads no longer sit
// in front of a barrier.  Per plane: the z face / flux / finish of the
// previous plane from the ring (own column, no barrier), then the in-plane
// sweeps x and y one after the other through one face and one flux buffer
// (fits two blocks per SM), the in-plane residual accumulating in
// registers.  Row offsets come from a per-block table; the in-plane offsets
// of every copy a thread issues are fixed for the whole march.
// ---------------------------------------------------------------------------
#ifndef FVB_RING3_MINB
#define FVB_RING3_MINB 2
#endif
#ifndef FVB_RING3_NTY
#define FVB_RING3_NTY 8
#endif
constexpr int kRing3NT = 32, kRing3NTY = FVB_RING3_NTY, kRing3Slots = 4;

template <int EQ, int FLUX, int RECON, bool FIN>
__global__ void __launch_bounds__(kRing3NT * kRing3NTY, FVB_RING3_MINB)
ring3_kernel(const StageParams p) {
  constexpr int DIM = 3, NT = kRing3NT, NTY = kRing3NTY;
  constexpr int NC = NComp<EQ, DIM>::value;
  constexpr bool WENO = RECON != RECON_NONE;
  constexpr int W = NT + 2, WY = NTY + 2, PL = WY * W, FB = NC * NTY * NT;
  extern __shared__ double smem[];
  double* ring = smem;                      // [slot][NC][WY][W]: planes, tile col j <-> x0-2+j, row i <-> y0-2+i
  double* hf = ring + kRing3Slots * NC * PL;  // [NC][NTY][NT] faces (x sweep, then y sweep)
  double* lf = hf + FB;
  double* gf = lf + FB;                     // [NC][NTY][NT] fluxes (x sweep, then y sweep)
  double* hs = gf + FB;                     // [NC][NTY][NT] z recurrence: high face of the previous plane
  double* gs = hs + FB;                     //                             z flux below the previous plane
  int64_t* rtab = reinterpret_cast<int64_t*>(gs + FB);
  auto RG = [&](int slot, int c, int y, int x) -> double& { return ring[((slot * NC + c) * WY + y) * W + x]; };
  const int tx = threadIdx.x, ty = threadIdx.y;
  auto FI = [&](int c, int y, int x) { return (c * NTY + y) * NT + x; };

  const int inst = blockIdx.z / p.chunks;
  const int chunk = blockIdx.z % p.chunks;
  FvbState* st = p.st + (p.shared_state ? 0 : inst);
  if (*(volatile int*)&st->done) return;
  const double dt = p.kind == 0 ? 0.0 : *(volatile double*)&st->dt;
  const double* __restrict__ us = p.us + p.origin + inst * p.si;
  const double* un = p.un + p.origin + inst * p.si;
  double* out = p.out + p.origin + inst * p.si;
  const int64_t x0 = (int64_t)blockIdx.x * (NT - 2);
  const int64_t y0 = (int64_t)blockIdx.y * (NTY - 2);
  const int64_t xf = x0 - 1 + tx, yf = y0 - 1 + ty;
  const bool inrow = ty >= 1 && ty <= NTY - 2;  // warp-uniform: interior face rows
  const bool cell = inrow && tx >= 1 && tx <= NT - 2 && xf < p.n[0] && yf < p.n[1];
  const int64_t ra = p.row_lo + (int64_t)chunk * p.H;
  const int64_t rb = min(ra + (int64_t)p.H, p.row_hi);
  const int64_t mxf = map_index(xf, p.n[0], p.bc[0], p.g), myf = map_index(yf, p.n[1], p.bc[1], p.g) * p.sy;
  const int64_t co = mxf + myf;
  // halo copies: lanes 0 / NT-1 also copy tile columns 0 / W-1 of their row,
  // warps 0 / NTY-1 also copy tile rows 0 / WY-1 of their column
  const bool hx_t = WENO && (tx == 0 || tx == NT - 1);
  const int64_t hxo = map_index(tx == 0 ? x0 - 2 : x0 + NT - 1, p.n[0], p.bc[0], p.g) + myf;
  const int hxc = tx == 0 ? 0 : W - 1;
  const bool hy_t = WENO && (ty == 0 || ty == NTY - 1);
  const int64_t hyo = mxf + map_index(ty == 0 ? y0 - 2 : y0 + NTY - 1, p.n[1], p.bc[1], p.g) * p.sy;
  const int hyr = ty == 0 ? 0 : WY - 1;
  const int tid = ty * NT + tx;
  for (int i = tid; i < p.H + 4; i += NT * NTY) rtab[i] = map_index(ra - 2 + i, p.n[2], p.bc[2], p.g) * p.sz;
  __syncthreads();
  auto roff = [&](int64_t r) -> int64_t { return rtab[r - (ra - 2)]; };
  auto fetch = [&](int64_t r, int slot) {
    const int64_t ro = roff(r);
#pragma unroll
    for (int c = 0; c < NC; ++c) cp_async8(&RG(slot, c, ty + 1, tx + 1), us + co + ro + c * p.sc);
    if (hx_t) {
#pragma unroll
      for (int c = 0; c < NC; ++c) cp_async8(&RG(slot, c, ty + 1, hxc), us + hxo + ro + c * p.sc);
    }
    if (hy_t) {
#pragma unroll
      for (int c = 0; c < NC; ++c) cp_async8(&RG(slot, c, hyr, tx + 1), us + hyo + ro + c * p.sc);
    }
  };

  unsigned errb = 0;
  double smax[DIM] = {0.0, 0.0, 0.0};
  double R[NC], unc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) R[c] = unc[c] = 0.0;

  // prologue: planes ra-2, ra-1, ra (slot of plane r = (r - ra + 2) % 4)
  for (int k = 0; k < 3; ++k) {
    fetch(ra - 2 + k, k);
    cp_async_commit();
  }
  int sA = 0;  // slot of plane r-1 at the top of the loop
  for (int64_t r = ra - 1; r <= rb; ++r) {
    const int sB = (sA + 1) & 3, sC = (sA + 2) & 3;
    if (r == ra) __syncthreads();  // iteration ra-1 had no in-plane barrier
    if (r + 2 <= rb + 1) fetch(r + 2, (sA + 3) & 3);  // into the slot of plane r-2
    cp_async_commit();
    cp_async_wait<1>();  // planes up to r+1 have landed (own copies)
    __syncthreads();     // ... everybody's; also: plane r-1's y fluxes (gf) are visible
    if (inrow && r - 1 >= ra && r - 1 < rb) {  // plane r-1's y residual, deferred past this barrier
#pragma unroll
      for (int c = 0; c < NC; ++c) {
#if FVB_FAST
        R[c] = fma(gf[FI(c, ty, tx)] - gf[FI(c, ty + 1, tx)], p.id[1], R[c]);
#else
        R[c] = R[c] - ddiv(gf[FI(c, ty + 1, tx)] - gf[FI(c, ty, tx)], p, 1);
#endif
      }
    }
    if (inrow) {  // z: faces of plane r, flux (r-1|r), finish plane r-1 (own column)
      double A[NC], B[NC], C[NC], hi[NC], lo[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        A[c] = RG(sA, c, ty + 1, tx + 1);
        B[c] = RG(sB, c, ty + 1, tx + 1);
        C[c] = RG(sC, c, ty + 1, tx + 1);
      }
      weno_faces_nc<NC, RECON>(A, B, C, p.P.eps, hi, lo);
      if (r >= ra) {
        double H[NC], GC[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) H[c] = hs[FI(c, ty, tx)];
        unsigned eb = 0;
        interface_flux<EQ, FLUX, DIM, RECON>(H, lo, A, B, 2, p.P, GC, eb);
        if (eb && cell) errb |= 4u;
        if (r - 1 >= ra) {
          double v[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const double Gp = gs[FI(c, ty, tx)];
#if FVB_FAST
            const double Lc = fma(Gp - GC[c], p.id[2], R[c]);
#else
            const double Lc = R[c] - ddiv(GC[c] - Gp, p, 2);
#endif
            v[c] = rk_combine(p.kind, unc[c], A[c], dt, Lc);
          }
          if (cell) {
            const int64_t o = co + roff(r - 1);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              out[o + c * p.sc] = v[c];
              peer_store(p, o, r - 1, p.sc, c, v[c]);
            }
            if constexpr (FIN) post_cell<EQ, DIM, NC>(p, st, v, xf, yf, r - 1, smax);
          }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) gs[FI(c, ty, tx)] = GC[c];
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) hs[FI(c, ty, tx)] = hi[c];
    }
    if (r >= ra && r < rb) {
      // u^n of plane r for the next iteration's finish (latency covered by
      // the in-plane sweeps)
      if (p.kind >= 2 && cell) {
        const int64_t o = co + roff(r);
#pragma unroll
        for (int c = 0; c < NC; ++c) unc[c] = un[o + c * p.sc];
      }
      if constexpr (EQ == EQ_EULER) {  // stage-start interior check (solver.py:90-93)
        if (p.check_input && cell) {
          double B[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) B[c] = RG(sB, c, ty + 1, tx + 1);
          if (!euler_physical<DIM>(B, p.P))
            atomicMin(&st->stage_err, ((long long)p.stage_idx << 42) | flat_cell<DIM>(p, xf, yf, r));
        }
      }
      // ---- x sweep (interior face rows) ----
      // A warp is one face row of the tile (32 consecutive x cells), so the
      // x neighbours are lanes of the same warp: faces and fluxes move by
      // shuffle, with no shared-memory round trip and no barrier.
      if (inrow) {  // warp-uniform; x interface tx sits between face cells tx-1 and tx (lane 0's is unused)
        double uL[NC], uR[NC], G[NC];
        if constexpr (WENO) {
          double um[NC], uc[NC], up[NC], hi[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            um[c] = RG(sB, c, ty + 1, tx);
            uc[c] = RG(sB, c, ty + 1, tx + 1);
            up[c] = RG(sB, c, ty + 1, tx + 2);
          }
          weno_faces_nc<NC, RECON>(um, uc, up, p.P.eps, hi, uR);
#pragma unroll
          for (int c = 0; c < NC; ++c) uL[c] = __shfl_up_sync(0xffffffffu, hi[c], 1);
        } else {
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            uL[c] = RG(sB, c, ty + 1, tx);
            uR[c] = RG(sB, c, ty + 1, tx + 1);
          }
        }
        auto cells = [&](double* a, double* b) {  // fallback only: loaded on demand
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            a[c] = RG(sB, c, ty + 1, tx);
            b[c] = RG(sB, c, ty + 1, tx + 1);
          }
        };
        unsigned eb = 0;
        interface_flux_lazy<EQ, FLUX, DIM, RECON>(uL, uR, cells, 0, p.P, G, eb);
        if (eb && tx >= 1 && xf <= p.n[0] && yf < p.n[1]) errb |= 1u;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const double Gr = __shfl_down_sync(0xffffffffu, G[c], 1);  // lane 31's is unused
#if FVB_FAST
          R[c] = (G[c] - Gr) * p.id[0];
#else
          R[c] = 0.0 - ddiv(Gr - G[c], p, 0);
#endif
        }
      }
      // ---- y sweep (all face rows) ----
      if constexpr (WENO) {
        double um[NC], uc[NC], up[NC], hi[NC], lo[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          um[c] = RG(sB, c, ty, tx + 1);
          uc[c] = RG(sB, c, ty + 1, tx + 1);
          up[c] = RG(sB, c, ty + 2, tx + 1);
        }
        weno_faces_nc<NC, RECON>(um, uc, up, p.P.eps, hi, lo);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          hf[FI(c, ty, tx)] = hi[c];
          lf[FI(c, ty, tx)] = lo[c];
        }
      }
      __syncthreads();  // y faces visible
      if (ty >= 1) {  // y interface ty sits between face rows ty-1 and ty
        double uL[NC], uR[NC], G[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          uL[c] = WENO ? hf[FI(c, ty - 1, tx)] : RG(sB, c, ty, tx + 1);
          uR[c] = WENO ? lf[FI(c, ty, tx)] : RG(sB, c, ty + 1, tx + 1);
        }
        auto cells = [&](double* a, double* b) {  // fallback only: loaded on demand
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            a[c] = RG(sB, c, ty, tx + 1);
            b[c] = RG(sB, c, ty + 1, tx + 1);
          }
        };
        unsigned eb = 0;
        interface_flux_lazy<EQ, FLUX, DIM, RECON>(uL, uR, cells, 1, p.P, G, eb);
        if (eb && tx >= 1 && tx <= NT - 2 && yf <= p.n[1] && xf < p.n[0]) errb |= 2u;
#pragma unroll
        for (int c = 0; c < NC; ++c) gf[FI(c, ty, tx)] = G[c];
      }
      // the y residual of this plane is added after the next iteration's top
      // barrier (one barrier per plane fewer); gf / hf / lf are rewritten only
      // after the next iteration's mid barrier
    }
    sA = sB;
  }
  cp_async_wait<0>();
  if (errb) {
#pragma unroll
    for (int a = 0; a < DIM; ++a)
      if (errb & (1u << a))
        atomicMin(&st->stage_err, ((long long)p.stage_idx << 42) | ((long long)(1 + a) << 40));
  }
  if constexpr (FIN) block_epilogue<DIM>(p, st, inst, smax, true);
}

template <int EQ>
constexpr int ring3_smem_bytes() {
  constexpr int NC = NComp<EQ, 3>::value;
  return 8 * (kRing3Slots * NC * (kRing3NTY + 2) * (kRing3NT + 2) + 5 * NC * kRing3NTY * kRing3NT);
}

// ---------------------------------------------------------------------------
// 3D ring kernel, all-interior rows (variant 4, default 3D).
//
// A block of 32 x 8 threads owns a 30 x 8 cell tile: warp ty is cell row
// y0+ty (every warp updates cells; lanes 0 / 31 are the x-halo face cells)
// and marches H planes along z.  The tile's y-halo work -- the high face of
// row -1 and the low face of row 8 -- is two extra WENO passes (warps 0 and
// 7), and the extra interface (7|8) is computed by warp 7; a plane ring of 12
// rows (y0-2 .. y0+9) x 34 columns streams in by cp.async one plane ahead.
// z and x sweeps read only the thread's own warp's copies; the y sweep goes
// through one face and one flux buffer with two block barriers per plane
// (the y residual of a plane is added after the next plane's top barrier).
// Compared with ring3_kernel (30 x 6 cells, rows 0 and 7 halo warps idle
// through the z and x sweeps) every warp has z/x work and a block carries
// 33 % more cells for the same two barriers.
// ---------------------------------------------------------------------------
constexpr int kR3iNT = 32, kR3iNTY = 8, kR3iRows = kR3iNTY + 4, kR3iW = kR3iNT + 2;


template <int EQ, int FLUX, int RECON, int KS, bool FIN>
__global__ void __launch_bounds__(kR3iNT * kR3iNTY, FVB_RING3_MINB)
ring3i_kernel(const StageParams p) {
  constexpr int DIM = 3, NT = kR3iNT, NTY = kR3iNTY, WY = kR3iRows, W = kR3iW;
  constexpr int NC = NComp<EQ, DIM>::value;
  constexpr int PL = WY * W;
  constexpr int FR = NC * (NTY + 1) * NT;    // face / flux buffers: rows 0..NTY
  constexpr bool UN = KS == 2;                 // the stage reads u^n (compile time: no u^n registers otherwise)
  extern __shared__ double smem[];
  double* ring = smem;                          // [slot][NC][WY][W]: ring row i <-> y0-2+i, col j <-> x0-2+j
  double* hf = ring + kRing3Slots * NC * PL;    // [NC][NTY+1][NT]: high y face of cell row i-1 (i = 0..NTY)
  double* gf = hf + FR;                         // [NC][NTY+1][NT]: y flux below cell row i (interface (i-1|i))
  double* hs = gf + FR;                         // [NC][NTY][NT] z recurrence: high face of the previous plane
  double* gs = hs + NC * NTY * NT;              //                             z flux below the previous plane
  int* rtab = reinterpret_cast<int*>(gs + NC * NTY * NT);
  auto RG = [&](int slot, int c, int y, int x) -> double& { return ring[((slot * NC + c) * WY + y) * W + x]; };
  const int tx = threadIdx.x, ty = threadIdx.y;
  auto FI = [&](int c, int y, int x) { return (c * (NTY + 1) + y) * NT + x; };
  auto ZI = [&](int c, int y, int x) { return (c * NTY + y) * NT + x; };

  const int inst = blockIdx.z / p.chunks;
  const int chunk = blockIdx.z % p.chunks;
  FvbState* st = p.st + (p.shared_state ? 0 : inst);
  if (*(volatile int*)&st->done) return;
  const double dt = KS == 0 ? 0.0 : *(volatile double*)&st->dt;
  const double* __restrict__ us = p.us + p.origin + inst * p.si;
  const double* un = p.un + p.origin + inst * p.si;
  double* out = p.out + p.origin + inst * p.si;
  const int64_t x0 = p.x_lo + (int64_t)blockIdx.x * (NT - 2);
  const int64_t y0 = p.y_lo + (int64_t)blockIdx.y * NTY;
  const int64_t xf = x0 - 1 + tx, yf = y0 + ty;
  const bool cell = tx >= 1 && tx <= NT - 2 && xf < p.x_hi && yf < p.y_hi;
  const int64_t ra = p.row_lo + (int64_t)chunk * p.H;
  const int64_t rb = min(ra + (int64_t)p.H, p.row_hi);
  const int64_t mxf = map_index(xf, p.n[0], p.bc[0], p.g);
  const int co = (int)(mxf + map_index(yf, p.n[1], p.bc[1], p.g) * p.sy);  // < 2^31 (validated)
  // extra copies: lanes 0 / NT-1 the x-halo columns of their row; warps 0, 1 /
  // NTY-2, NTY-1 one y-halo row each (ring rows 0, 1 / WY-2, WY-1), interior columns
  // (as 32-bit deltas from co: an instance component spans < 2^31 elements,
  // and two int32 registers instead of two int64 pairs keep the loop spill-free)
  const bool hx_t = tx == 0 || tx == NT - 1;
  const int dxh = (int)(map_index(tx == 0 ? x0 - 2 : x0 + NT - 1, p.n[0], p.bc[0], p.g) - mxf);
  const int hxc = tx == 0 ? 0 : W - 1;
  const bool hy_t = ty <= 1 || ty >= NTY - 2;
  const int hyr = ty <= 1 ? ty : WY - NTY + ty;  // ring row 0, 1 | WY-2, WY-1
  const int dyh = (int)((map_index(y0 - 2 + hyr, p.n[1], p.bc[1], p.g) - map_index(yf, p.n[1], p.bc[1], p.g)) * p.sy);
  const int tid = ty * NT + tx;
  for (int i = tid; i < p.H + 4; i += NT * NTY) rtab[i] = (int)(map_index(ra - 2 + i, p.n[2], p.bc[2], p.g) * p.sz);
  __syncthreads();
  auto roff = [&](int64_t r) -> int { return rtab[r - (ra - 2)]; };
  auto fetch = [&](int64_t r, int slot) {
    const int ro = roff(r);
#pragma unroll
    for (int c = 0; c < NC; ++c) cp_async8(&RG(slot, c, ty + 2, tx + 1), us + (co + ro) + c * p.sc);
    if (hx_t) {
#pragma unroll
      for (int c = 0; c < NC; ++c) cp_async8(&RG(slot, c, ty + 2, hxc), us + (co + dxh + ro) + c * p.sc);
    }
    if (hy_t) {
#pragma unroll
      for (int c = 0; c < NC; ++c) cp_async8(&RG(slot, c, hyr, tx + 1), us + (co + dyh + ro) + c * p.sc);
    }
  };

  unsigned errb = 0;
  double smax[DIM] = {0.0, 0.0, 0.0};
  double R[NC], unc[UN ? NC : 1];
#pragma unroll
  for (int c = 0; c < NC; ++c) R[c] = 0.0;
#pragma unroll
  for (int c = 0; c < (UN ? NC : 1); ++c) unc[c] = 0.0;

  for (int k = 0; k < 3; ++k) {
    fetch(ra - 2 + k, k);
    cp_async_commit();
  }
  int sA = 0;
  for (int64_t r = ra - 1; r <= rb; ++r) {
    const int sB = (sA + 1) & 3, sC = (sA + 2) & 3;
    if (r == ra) __syncthreads();  // iteration ra-1 had no in-plane barrier
    if (r + 2 <= rb + 1) fetch(r + 2, (sA + 3) & 3);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();  // everybody's copies of planes <= r+1; plane r-1's y fluxes (gf) visible
    if (r - 1 >= ra && r - 1 < rb) {  // plane r-1's y residual, deferred past this barrier
#pragma unroll
      for (int c = 0; c < NC; ++c) {
#if FVB_FAST
        R[c] = fma(gf[FI(c, ty, tx)] - gf[FI(c, ty + 1, tx)], p.id[1], R[c]);
#else
        R[c] = R[c] - ddiv(gf[FI(c, ty + 1, tx)] - gf[FI(c, ty, tx)], p, 1);
#endif
      }
    }
    {  // z: faces of plane r, flux (r-1|r), finish plane r-1 (own column)
      double A[NC], B[NC], C[NC], hi[NC], lo[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        A[c] = RG(sA, c, ty + 2, tx + 1);
        B[c] = RG(sB, c, ty + 2, tx + 1);
        C[c] = RG(sC, c, ty + 2, tx + 1);
      }
      weno_faces_nc<NC, RECON>(A, B, C, p.P.eps, hi, lo);
      if (r >= ra) {
        double H[NC], GC[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) H[c] = hs[ZI(c, ty, tx)];
        unsigned eb = 0;
        interface_flux<EQ, FLUX, DIM, RECON>(H, lo, A, B, 2, p.P, GC, eb);
        if (eb && cell) errb |= 4u;
        if (r - 1 >= ra) {
          double v[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const double Gp = gs[ZI(c, ty, tx)];
#if FVB_FAST
            const double Lc = fma(Gp - GC[c], p.id[2], R[c]);
#else
            const double Lc = R[c] - ddiv(GC[c] - Gp, p, 2);
#endif
            v[c] = KS == 0 ? Lc : rk_combine(p.kind, UN ? unc[UN ? c : 0] : 0.0, A[c], dt, Lc);
          }
          if (cell) {
            const int o = co + roff(r - 1);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              out[o + c * p.sc] = v[c];
              peer_store(p, o, r - 1, p.sc, c, v[c]);
            }
            if constexpr (FIN) post_cell<EQ, DIM, NC>(p, st, v, xf, yf, r - 1, smax);
          }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) gs[ZI(c, ty, tx)] = GC[c];
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) hs[ZI(c, ty, tx)] = hi[c];
    }
    if (r >= ra && r < rb) {
      if constexpr (UN) {
        if (cell) {  // u^n of plane r for the next iteration's finish
          const int o = co + roff(r);
#pragma unroll
          for (int c = 0; c < NC; ++c) unc[c] = un[o + c * p.sc];
        }
      }
      double B[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) B[c] = RG(sB, c, ty + 2, tx + 1);
      if constexpr (EQ == EQ_EULER) {  // stage-start interior check (solver.py:90-93)
        if (p.check_input && cell && !euler_physical<DIM>(B, p.P))
          atomicMin(&st->stage_err, ((long long)p.stage_idx << 42) | flat_cell<DIM>(p, xf, yf, r));
      }
      // ---- x sweep: a warp is one face row; faces and fluxes by shuffle ----
      {
        double uL[NC], uR[NC], G[NC];
        if constexpr (RECON != RECON_NONE) {
          double um[NC], up[NC], hi[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            um[c] = RG(sB, c, ty + 2, tx);
            up[c] = RG(sB, c, ty + 2, tx + 2);
          }
          weno_faces_nc<NC, RECON>(um, B, up, p.P.eps, hi, uR);
#pragma unroll
          for (int c = 0; c < NC; ++c) uL[c] = __shfl_up_sync(0xffffffffu, hi[c], 1);
        } else {
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            uL[c] = RG(sB, c, ty + 2, tx);
            uR[c] = B[c];
          }
        }
        auto cells = [&](double* a, double* b) {
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            a[c] = RG(sB, c, ty + 2, tx);
            b[c] = RG(sB, c, ty + 2, tx + 1);
          }
        };
        unsigned eb = 0;
        interface_flux_lazy<EQ, FLUX, DIM, RECON>(uL, uR, cells, 0, p.P, G, eb);
        if (eb && tx >= 1 && xf <= p.n[0] && yf < p.n[1]) errb |= 1u;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const double Gr = __shfl_down_sync(0xffffffffu, G[c], 1);
#if FVB_FAST
          R[c] = (G[c] - Gr) * p.id[0];
#else
          R[c] = 0.0 - ddiv(Gr - G[c], p, 0);
#endif
        }
      }
      // ---- y sweep ----
      double lo_own[NC], hi_own[NC], lo_top[NC];
      if constexpr (RECON != RECON_NONE) {
        double um[NC], up[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          um[c] = RG(sB, c, ty + 1, tx + 1);
          up[c] = RG(sB, c, ty + 3, tx + 1);
        }
        weno_faces_nc<NC, RECON>(um, B, up, p.P.eps, hi_own, lo_own);
#pragma unroll
        for (int c = 0; c < NC; ++c) hf[FI(c, ty + 1, tx)] = hi_own[c];
        if (ty == 0) {  // high face of row -1 (ring rows 0, 1, 2)
          double a[NC], b[NC], d[NC], h[NC], l[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            a[c] = RG(sB, c, 0, tx + 1);
            b[c] = RG(sB, c, 1, tx + 1);
            d[c] = RG(sB, c, 2, tx + 1);
          }
          weno_faces_nc<NC, RECON>(a, b, d, p.P.eps, h, l);
#pragma unroll
          for (int c = 0; c < NC; ++c) hf[FI(c, 0, tx)] = h[c];
        }
        if (ty == NTY - 1) {  // low face of row NTY (ring rows WY-3, WY-2, WY-1)
          double a[NC], b[NC], d[NC], h[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            a[c] = RG(sB, c, WY - 3, tx + 1);
            b[c] = RG(sB, c, WY - 2, tx + 1);
            d[c] = RG(sB, c, WY - 1, tx + 1);
          }
          weno_faces_nc<NC, RECON>(a, b, d, p.P.eps, h, lo_top);
        }
      } else {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          hi_own[c] = lo_own[c] = B[c];
          lo_top[c] = RG(sB, c, WY - 2, tx + 1);
          hf[FI(c, ty + 1, tx)] = B[c];
          if (ty == 0) hf[FI(c, 0, tx)] = RG(sB, c, 1, tx + 1);
        }
      }
      __syncthreads();  // y faces visible
      {  // interface (ty-1 | ty): uL = high face of row ty-1, uR = own low face
        double uL[NC], G[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) uL[c] = hf[FI(c, ty, tx)];
        auto cells = [&](double* a, double* b) {
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            a[c] = RG(sB, c, ty + 1, tx + 1);
            b[c] = B[c];
          }
        };
        double uR[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) uR[c] = lo_own[c];
        unsigned eb = 0;
        interface_flux_lazy<EQ, FLUX, DIM, RECON>(uL, uR, cells, 1, p.P, G, eb);
        if (eb && tx >= 1 && tx <= NT - 2 && yf <= p.n[1] && xf < p.n[0]) errb |= 2u;
#pragma unroll
        for (int c = 0; c < NC; ++c) gf[FI(c, ty, tx)] = G[c];
      }
      if (ty == NTY - 1) {  // interface (NTY-1 | NTY)
        double G[NC];
        auto cells = [&](double* a, double* b) {
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            a[c] = B[c];
            b[c] = RG(sB, c, WY - 2, tx + 1);
          }
        };
        unsigned eb = 0;
        interface_flux_lazy<EQ, FLUX, DIM, RECON>(hi_own, lo_top, cells, 1, p.P, G, eb);
        if (eb && tx >= 1 && tx <= NT - 2 && yf + 1 <= p.n[1] && xf < p.n[0]) errb |= 2u;
#pragma unroll
        for (int c = 0; c < NC; ++c) gf[FI(c, NTY, tx)] = G[c];
      }
      // the y residual of this plane is added after the next top barrier
    }
    sA = sB;
  }
  cp_async_wait<0>();
  if (errb) {
#pragma unroll
    for (int a = 0; a < DIM; ++a)
      if (errb & (1u << a))
        atomicMin(&st->stage_err, ((long long)p.stage_idx << 42) | ((long long)(1 + a) << 40));
  }
  if constexpr (FIN) block_epilogue<DIM>(p, st, inst, smax, true);
}

template <int EQ>
constexpr int ring3i_smem_bytes() {
  constexpr int NC = NComp<EQ, 3>::value;
  return 8 * (kRing3Slots * NC * kR3iRows * kR3iW + 2 * NC * (kR3iNTY + 1) * kR3iNT + 2 * NC * kR3iNTY * kR3iNT);
}

// Standalone wave-speed pass: solver.py:128-136 (+ the initial is_physical
// check of solver.py:211-212).  finalize = 1 also computes the first dt.
template <int DIM, int EQ>
__global__ void __launch_bounds__(256) speed_kernel(const StageParams p, int finalize) {
  constexpr int NC = NComp<EQ, DIM>::value;
  const int inst = blockIdx.y;
  FvbState* st = p.st + (p.shared_state ? 0 : inst);
  const double* u = p.us + p.origin + inst * p.si;
  double smax[DIM];
#pragma unroll
  for (int k = 0; k < DIM; ++k) smax[k] = 0.0;
  const int64_t ncell = p.n[0] * p.n[1] * p.n[2];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ncell;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = i % p.n[0];
    const int64_t yz = i / p.n[0];
    const int64_t y = yz % p.n[1];
    const int64_t z = yz / p.n[1];
    const int64_t o = x + y * p.sy + z * p.sz;
    double v[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) v[c] = u[o + c * p.sc];
    if constexpr (EQ == EQ_EULER) {
      if (!euler_physical<DIM>(v, p.P)) atomicMin(&st->bad_unphys, (long long)i);
    }
    double s[DIM];
    wave_speeds<EQ, DIM>(v, p.P, s);
#pragma unroll
    for (int k = 0; k < DIM; ++k) smax[k] = fmax(smax[k], s[k]);
  }
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < DIM; ++k) {
    unsigned long long b = (unsigned long long)__double_as_longlong(smax[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long q = __shfl_xor_sync(0xffffffffu, b, o);
      b = q > b ? q : b;
    }
    if (lane == 0 && b != 0ull) atomicMax(&st->smax[k], b);
  }
  if (!finalize) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&st->blocks_done, 1u);
    if (prev == gridDim.x * (p.shared_state ? gridDim.y : 1u) - 1) {
      __threadfence();
      finalize_step(st, p.ctl, p.shared_state ? 0 : inst, false, true);
    }
  }
}

// host-side launchers (defined in fvb_kernels.cu, once per namespace)
int launch_stage(int dim, int eq, int flux, int recon, const StageParams& p, dim3 grid, cudaStream_t s);
int launch_speed(int dim, int eq, const StageParams& p, int finalize, dim3 grid, cudaStream_t s);
void stage_block(int dim, int variant, int& nt, int& nty);

}  // namespace FVB_NS
}  // namespace fvb
