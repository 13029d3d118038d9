// Device-side physics for the finite-volume stage: equation of state,
// physical fluxes, wave speeds, WENO2/3 face reconstruction, Rusanov and
// HLLC numerical fluxes.
//
// Two arithmetic modes share this header:
//   FVB_FAST == 0  "exact": compiled with -fmad=false and written in the
//                  reference's operation order, so every value is bitwise
//                  identical to numpy (one IEEE binary64 op per numpy pass).
//   FVB_FAST == 1  "fast": same algorithm, algebraically restructured to
//                  remove divides (one reciprocal per WENO pair, 1/rho per
//                  state, MUFU reciprocal/rsqrt seeds + Newton steps) and
//                  FMA-contracted; parity is relative L1 <= 1e-12 over the
//                  test windows (tests/test_gpu_parity.py).
//
// Reference citations: /root/reference/pkg/src/conslaw/<file>:<line>.
#pragma once
#include <cstdint>
#include <cmath>
#include "fvb_common.cuh"

#ifndef FVB_FAST
#error "FVB_FAST must be defined to 0 or 1"
#endif
// Warp-uniform shortcuts (flat WENO stencils, uniform interface states, no
// star state in the warp): 1 = take them when the whole warp agrees.  Off by
// default: in a developed flow (the KH roll-up bench.py times) whole warps
// rarely agree and the votes cost more than they save (KH2D 1024^2 at
// t ~ 1: 22.7 Gcell-stage/s without vs 21.2 with, profiles/r02_variants.json).
#ifndef FVB_WARP_SKIP
#define FVB_WARP_SKIP 0
#endif
#ifndef FVB_FAST_NO_EQ
#define FVB_FAST_NO_EQ 1
#endif

namespace fvb {

// numpy.maximum / numpy.minimum: NaN-propagating (numerics.py:138,164-165).
// The fast mode uses a plain compare + select (one DSETP, two FSEL; fmax
// costs DSETP.MAX plus a NaN fix-up and register moves): it differs only on
// NaN inputs, i.e. on states whose run is already failing a check.
#if FVB_FAST
__device__ __forceinline__ double np_max(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double np_min(double a, double b) { return a < b ? a : b; }
#else
__device__ __forceinline__ double np_max(double a, double b) { return (a > b || a != a) ? a : b; }
__device__ __forceinline__ double np_min(double a, double b) { return (a < b || a != a) ? a : b; }
#endif

// Bitwise equality on the integer pipes (keeps warp-shortcut tests off the
// FP64 pipe).  It is conservative: +0/-0 count as different, so such lanes
// simply take the general path, whose own numeric tests decide.
__device__ __forceinline__ bool bit_eq(double a, double b) {
  return __double_as_longlong(a) == __double_as_longlong(b);
}

#if FVB_FAST
// 1/x: MUFU seed (relative error e0 ~ 1e-6) + one third-order step
// r (1 + e + e^2), e = 1 - x r: error e0^3 ~ 1e-18, below half an ulp, in
// three DFMA instead of the four of two Newton steps
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}
// a/b: a times the (<= 1 ulp) reciprocal, <= 2 ulp
__device__ __forceinline__ double fdiv(double a, double b) { return a * frcp(b); }
// sqrt(x), x > 0: rsqrt seed y (relative error e0 ~ 1e-6), then one
// third-order step of the series 1/sqrt(1-e) = 1 + e/2 + 3e^2/8 + ...
// with e = 1 - x y^2, applied to s = x y directly:
//   sqrt(x) = s (1 + e/2 + 3e^2/8) + O(e^3 s),  e^3 ~ 1e-17
// -- five FP64 instructions instead of eight for Newton + residual
// correction, within 2 ulp (tools/mufu_precision.cu).  The sound speed it
// feeds enters the HLLC/Rusanov flux only through the wave-speed estimates,
// whose errors are multiplied by the state jump (the flux is consistent for
// any speeds).
__device__ __forceinline__ double fsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double s = x * y;
  const double e = fma(-s, y, 1.0);
  return fma(s * e, fma(e, 0.375, 0.5), s);
}
#endif

// All components of two states bitwise equal, on the integer pipes: one
// three-input LOP3 per 32-bit half folds (a ^ b) | acc.  Conservative
// (+0 / -0 differ), see bit_eq.
template <int NC>
__device__ __forceinline__ bool bits_equal_all(const double* a, const double* b) {
  unsigned acc = 0u;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    acc |= (unsigned)__double2loint(a[c]) ^ (unsigned)__double2loint(b[c]);
    acc |= (unsigned)__double2hiint(a[c]) ^ (unsigned)__double2hiint(b[c]);
  }
  return acc == 0u;
}
// um == uc == up bitwise in every component (a flat WENO stencil)
template <int NC>
__device__ __forceinline__ bool bits_flat_all(const double* um, const double* uc, const double* up) {
  unsigned acc = 0u;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const unsigned cl = (unsigned)__double2loint(uc[c]), ch = (unsigned)__double2hiint(uc[c]);
    acc |= cl ^ (unsigned)__double2loint(um[c]);
    acc |= cl ^ (unsigned)__double2loint(up[c]);
    acc |= ch ^ (unsigned)__double2hiint(um[c]);
    acc |= ch ^ (unsigned)__double2hiint(up[c]);
  }
  return acc == 0u;
}

// ---------------------------------------------------------------------------
// Euler equation of state (equations.py:62-73, 128-129)
// ---------------------------------------------------------------------------
template <int DIM>
__device__ __forceinline__ double euler_pressure(const double* u, const Phys& P) {
  // sum(m_k**2) starts from int 0 in the reference: 0 + m0^2 == m0^2 exactly
  double msq = u[1] * u[1];
#pragma unroll
  for (int k = 1; k < DIM; ++k) msq = msq + u[1 + k] * u[1 + k];
#if FVB_FAST
  return P.gm1 * (u[1 + DIM] - msq * (0.5 * frcp(u[0])));
#else
  return P.gm1 * (u[1 + DIM] - msq / (2.0 * u[0]));
#endif
}

template <int DIM>
__device__ __forceinline__ bool euler_physical(const double* u, const Phys& P) {
#if FVB_FAST
  // reciprocal free: for rho > 0, p > floor  <=>  gm1 (E rho - |m|^2 / 2) > floor rho
  double msq = u[1] * u[1];
#pragma unroll
  for (int k = 1; k < DIM; ++k) msq = fma(u[1 + k], u[1 + k], msq);
  const double t = fma(u[1 + DIM], u[0], -0.5 * msq);
  return (u[0] > kFloor) & (P.gm1 * t > kFloor * u[0]);
#else
  return (u[0] > kFloor) & (euler_pressure<DIM>(u, P) > kFloor);
#endif
}

// Physical flux F_axis(u) (equations.py:91-110), given p and v = m_axis/rho.
template <int DIM>
__device__ __forceinline__ void euler_flux(const double* u, double p, double v, int axis, double* f) {
  f[0] = u[1 + axis];
#pragma unroll
  for (int j = 0; j < DIM; ++j) f[1 + j] = u[1 + j] * v;
  f[1 + axis] = f[1 + axis] + p;
  f[1 + DIM] = (u[1 + DIM] + p) * v;
}

// Per-state quantities shared by flux, wave speed and HLLC.
struct EState { double rho, v, p, c, rinv; };

template <int DIM>
__device__ __forceinline__ EState euler_state(const double* u, int axis, const Phys& P) {
  EState s;
  s.rho = u[0];
#if FVB_FAST
  const double r = frcp(u[0]);
  s.rinv = r;
  s.v = u[1 + axis] * r;
  double msq = u[1] * u[1];
#pragma unroll
  for (int k = 1; k < DIM; ++k) msq = fma(u[1 + k], u[1 + k], msq);
  s.p = P.gm1 * fma(-0.5 * msq, r, u[1 + DIM]);
  s.c = fsqrt(P.gamma * s.p * r);
#else
  s.rinv = 0.0;
  s.v = u[1 + axis] / s.rho;                      // numerics.py:159
  s.p = euler_pressure<DIM>(u, P);                // numerics.py:160
  s.c = sqrt(P.gamma * s.p / s.rho);              // equations.py:128-129
#endif
  return s;
}

// ---------------------------------------------------------------------------
// WENO face reconstruction of one component (numerics.py:64-87, 109-117)
//
// For a cell with neighbours (um, uc, up) along the axis, returns the value
// at its high face (uL of the interface to its right) and at its low face
// (uR of the interface to its left).  The reference computes the low face
// with the mirrored stencil (up, uc, um); with D0 = uc-um, D1 = up-uc the
// mirrored smoothness indicators are (D1^2, D0^2) bitwise, so both faces
// share beta, (eps+beta)^2 and -- for WENO2's symmetric ideal weights -- the
// normalised weights themselves.  All shares are exact (negation, swap of a
// commutative add), so the exact mode stays bitwise.
// ---------------------------------------------------------------------------
template <int RECON>
__device__ __forceinline__ void weno_faces(double um, double uc, double up, double eps,
                                           double& hi, double& lo) {
  if constexpr (RECON == RECON_NONE) {
    hi = uc;
    lo = uc;
  } else {
    const double D0 = uc - um;
    const double D1 = up - uc;
#if FVB_FAST
    const double e0 = fma(D0, D0, eps);
    const double e1 = fma(D1, D1, eps);
    const double q0 = e0 * e0;
    const double q1 = e1 * e1;
    if constexpr (RECON == RECON_WENO2) {
      // w0 = q1/(q0+q1), w1 = q0/(q0+q1)
      const double h = (0.5 * frcp(q0 + q1)) * fma(q1, D0, q0 * D1);
      hi = uc + h;
      lo = uc - h;
    } else {
      // high face: a0 = (1/3)/q0, a1 = (2/3)/q1 -> w0 = q1/(q1 + 2 q0)
      // low face : a0 = (1/3)/q1, a1 = (2/3)/q0 -> w0' = q0/(q0 + 2 q1)
      const double th = fma(q1, D0, 2.0 * q0 * D1) * frcp(fma(2.0, q0, q1));
      const double tl = fma(q0, D1, 2.0 * q1 * D0) * frcp(fma(2.0, q1, q0));
      hi = fma(0.5, th, uc);
      lo = fma(-0.5, tl, uc);
    }
#else
    const double e0 = eps + D0 * D0;
    const double e1 = eps + D1 * D1;
    const double q0 = e0 * e0;
    const double q1 = e1 * e1;
    if constexpr (RECON == RECON_WENO2) {
      const double a0 = 0.5 / q0;
      const double a1 = 0.5 / q1;
      const double s = a0 + a1;
      const double w0 = a0 / s;
      const double w1 = a1 / s;
      const double S = w0 * D0 + w1 * D1;
      const double h = 0.5 * S;
      hi = uc + h;
      lo = uc - h;
    } else {
      constexpr double d0 = 1.0 / 3.0, d1 = 2.0 / 3.0;  // numerics.py:53
      const double a0 = d0 / q0, a1 = d1 / q1;
      const double s = a0 + a1;
      const double w0 = a0 / s, w1 = a1 / s;
      hi = uc + 0.5 * (w0 * D0 + w1 * D1);
      const double b0 = d0 / q1, b1 = d1 / q0;   // mirrored stencil
      const double t = b0 + b1;
      const double v0 = b0 / t, v1 = b1 / t;
      lo = uc - 0.5 * (v0 * D1 + v1 * D0);
    }
#endif
  }
}

#if FVB_FAST
// Fast-mode WENO2 faces of all components of one cell.  With D0 = uc - um,
// D1 = up - uc, q_i = (eps + D_i^2)^2: both faces share the weights and
// hi/lo = uc +- (1/2) (q1 D0 + q0 D1) / (q0 + q1), written as two FMAs with
// r = 1/(2 (q0 + q1)).  One reciprocal serves all components
// (1/den_c = prod_{k!=c} den_k / prod_k den_k; den_c >= 2 eps^2 keeps the
// product in range).  A warp whose every stencil is flat skips the weights
// (r = T = 0 gives hi = lo = uc).
template <int NC>
__device__ __forceinline__ void weno2_faces_fast(const double* um, const double* uc, const double* up, double eps,
                                                 double* hi, double* lo) {
  double rd[NC], T[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    rd[c] = 0.0;
    T[c] = 0.0;
  }
  if (!FVB_WARP_SKIP || __any_sync(__activemask(), !bits_flat_all<NC>(um, uc, up))) {
    double den[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double D0 = uc[c] - um[c];
      const double D1 = up[c] - uc[c];
      const double e0 = fma(D0, D0, eps);
      const double e1 = fma(D1, D1, eps);
      const double q1 = e1 * e1;
      den[c] = fma(e0, e0, q1);
      T[c] = fma(q1, D0, e0 * (e0 * D1));
    }
    if constexpr (NC == 1) {
      rd[0] = 0.5 * frcp(den[0]);
    } else if constexpr (NC == 4) {  // product tree: 9 multiplies for the 4 cofactors
      const double p01 = den[0] * den[1], p23 = den[2] * den[3];
      const double inv = 0.5 * frcp(p01 * p23);
      const double a = inv * p23, b = inv * p01;
      rd[0] = a * den[1];
      rd[1] = a * den[0];
      rd[2] = b * den[3];
      rd[3] = b * den[2];
    } else if constexpr (NC == 5) {
      const double p01 = den[0] * den[1], p23 = den[2] * den[3], p234 = p23 * den[4];
      const double inv = 0.5 * frcp(p01 * p234);
      const double a = inv * p234, b = inv * p01, b4 = b * den[4];
      rd[0] = a * den[1];
      rd[1] = a * den[0];
      rd[2] = b4 * den[3];
      rd[3] = b4 * den[2];
      rd[4] = b * p23;
    } else {
      double pre[NC + 1], suf[NC + 1];
      pre[0] = 1.0;
      suf[NC] = 1.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) pre[c + 1] = pre[c] * den[c];
#pragma unroll
      for (int c = NC - 1; c >= 0; --c) suf[c] = suf[c + 1] * den[c];
      const double inv = 0.5 * frcp(pre[NC]);
#pragma unroll
      for (int c = 0; c < NC; ++c) rd[c] = (inv * pre[c]) * suf[c + 1];
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    hi[c] = fma(rd[c], T[c], uc[c]);
    lo[c] = fma(-rd[c], T[c], uc[c]);
  }
}
#endif

// All components of one cell: a warp whose every cell has a flat stencil
// (um == uc == up, the uniform KH bands) skips the weights.  The shortcut
// returns exactly what the formula gives for D0 = D1 = +0 (h = +0, so
// hi = uc + 0.0 and lo = uc - 0.0, signed zeros included) in both modes.
template <int NC, int RECON>
__device__ __forceinline__ void weno_faces_nc(const double* um, const double* uc, const double* up, double eps,
                                              double* hi, double* lo) {
  if constexpr (RECON == RECON_NONE) {
#pragma unroll
    for (int c = 0; c < NC; ++c) { hi[c] = uc[c]; lo[c] = uc[c]; }
  } else {
#if FVB_FAST
    if constexpr (RECON == RECON_WENO2) {
      weno2_faces_fast<NC>(um, uc, up, eps, hi, lo);
      return;
    }
#endif
    // hi = uc + dh, lo = uc - dl.  A warp whose every stencil is flat
    // (D0 = D1 = +0 in all components) skips the weights: the formula then
    // gives dh = dl = +0 exactly in both modes (signed zeros included).
    double dh[NC], dl[NC];
#if FVB_FAST
    const bool flat = bits_flat_all<NC>(um, uc, up);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      dh[c] = 0.0;
      dl[c] = 0.0;
    }
#else
    bool flat = true;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      flat &= bit_eq(uc[c], um[c]) & bit_eq(up[c], uc[c]);
      dh[c] = 0.0;
      dl[c] = 0.0;
    }
#endif
    if (__any_sync(__activemask(), !flat)) {
      double D0[NC], D1[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        D0[c] = uc[c] - um[c];
        D1[c] = up[c] - uc[c];
      }
#if FVB_FAST
      if constexpr (RECON == RECON_WENO2 && NC > 1) {
        // one reciprocal for all components: 1/den_c = (prod_{k!=c} den_k) / prod_k den_k
        // (den_c = q0 + q1 >= 2 eps^2, so the product stays in range)
        double den[NC], T[NC], pre[NC + 1], suf[NC + 1];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const double e0 = fma(D0[c], D0[c], eps);
          const double e1 = fma(D1[c], D1[c], eps);
          const double q0 = e0 * e0;
          const double q1 = e1 * e1;
          den[c] = q0 + q1;
          T[c] = fma(q1, D0[c], q0 * D1[c]);
        }
        double rden[NC];  // 0.5 / den_c
        if constexpr (NC == 4) {  // product tree: 9 multiplies for the 4 cofactors
          const double p01 = den[0] * den[1], p23 = den[2] * den[3];
          const double inv = 0.5 * frcp(p01 * p23);
          const double a = inv * p23, b = inv * p01;
          rden[0] = a * den[1];
          rden[1] = a * den[0];
          rden[2] = b * den[3];
          rden[3] = b * den[2];
        } else if constexpr (NC == 5) {
          const double p01 = den[0] * den[1], p23 = den[2] * den[3], p234 = p23 * den[4];
          const double inv = 0.5 * frcp(p01 * p234);
          const double a = inv * p234, b = inv * p01, b4 = b * den[4];
          rden[0] = a * den[1];
          rden[1] = a * den[0];
          rden[2] = b4 * den[3];
          rden[3] = b4 * den[2];
          rden[4] = b * p23;
        } else {
          pre[0] = 1.0;
          suf[NC] = 1.0;
#pragma unroll
          for (int c = 0; c < NC; ++c) pre[c + 1] = pre[c] * den[c];
#pragma unroll
          for (int c = NC - 1; c >= 0; --c) suf[c] = suf[c + 1] * den[c];
          const double inv = 0.5 * frcp(pre[NC]);
#pragma unroll
          for (int c = 0; c < NC; ++c) rden[c] = (inv * pre[c]) * suf[c + 1];
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          dh[c] = rden[c] * T[c];
          dl[c] = dh[c];
        }
      } else
#endif
#pragma unroll
      for (int c = 0; c < NC; ++c) {
#if FVB_FAST
        const double e0 = fma(D0[c], D0[c], eps);
        const double e1 = fma(D1[c], D1[c], eps);
        const double q0 = e0 * e0;
        const double q1 = e1 * e1;
        if constexpr (RECON == RECON_WENO2) {
          dh[c] = (0.5 * frcp(q0 + q1)) * fma(q1, D0[c], q0 * D1[c]);
          dl[c] = dh[c];
        } else {
          dh[c] = 0.5 * (fma(q1, D0[c], 2.0 * q0 * D1[c]) * frcp(fma(2.0, q0, q1)));
          dl[c] = 0.5 * (fma(q0, D1[c], 2.0 * q1 * D0[c]) * frcp(fma(2.0, q1, q0)));
        }
#else
        const double e0 = eps + D0[c] * D0[c];
        const double e1 = eps + D1[c] * D1[c];
        const double q0 = e0 * e0;
        const double q1 = e1 * e1;
        if constexpr (RECON == RECON_WENO2) {
          const double a0 = 0.5 / q0;
          const double a1 = 0.5 / q1;
          const double sm = a0 + a1;
          dh[c] = 0.5 * ((a0 / sm) * D0[c] + (a1 / sm) * D1[c]);
          dl[c] = dh[c];
        } else {
          constexpr double d0 = 1.0 / 3.0, d1 = 2.0 / 3.0;  // numerics.py:53
          const double a0 = d0 / q0, a1 = d1 / q1;
          const double sa = a0 + a1;
          dh[c] = 0.5 * ((a0 / sa) * D0[c] + (a1 / sa) * D1[c]);
          const double b0 = d0 / q1, b1 = d1 / q0;  // mirrored stencil
          const double sb = b0 + b1;
          dl[c] = 0.5 * ((b0 / sb) * D1[c] + (b1 / sb) * D0[c]);
        }
#endif
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      hi[c] = uc[c] + dh[c];
      lo[c] = uc[c] - dl[c];
    }
  }
}

// ---------------------------------------------------------------------------
// Numerical fluxes.  errbits |= 1: degenerate HLLC fan (numerics.py:166-167).
// ---------------------------------------------------------------------------

// Rusanov (numerics.py:133-142)
template <int EQ, int DIM>
__device__ __forceinline__ void rusanov(const double* uL, const double* uR, const EState& L, const EState& R,
                                        int axis, const Phys& P, double* F) {
  constexpr int NC = NComp<EQ, DIM>::value;
  if constexpr (EQ == EQ_EULER) {
    double fL[NC], fR[NC];
    euler_flux<DIM>(uL, L.p, L.v, axis, fL);
    euler_flux<DIM>(uR, R.p, R.v, axis, fR);
    const double s = np_max(fabs(L.v) + L.c, fabs(R.v) + R.c);
    const double hs = 0.5 * s;
#pragma unroll
    for (int c = 0; c < NC; ++c) F[c] = 0.5 * (fL[c] + fR[c]) - hs * (uR[c] - uL[c]);
  } else if constexpr (EQ == EQ_BURGERS) {
    const double fL = 0.5 * uL[0] * uL[0];
    const double fR = 0.5 * uR[0] * uR[0];
    const double s = np_max(fabs(uL[0]), fabs(uR[0]));
    F[0] = 0.5 * (fL + fR) - 0.5 * s * (uR[0] - uL[0]);
  } else {
    const double a = P.adv[axis];
    const double fL = a * uL[0];
    const double fR = a * uR[0];
    const double s = fabs(a);
    F[0] = 0.5 * (fL + fR) - 0.5 * s * (uR[0] - uL[0]);
  }
}

// HLLC with Davis speeds (numerics.py:145-196), branch free: the side K of
// the reference's nested np.where (sL>=0 -> fL; sM>=0 -> F*L; sR>0 -> F*R;
// else fR; uL==uR -> fL) is selected first, then ONE physical flux and ONE
// star state are evaluated for that side.  The selected value is the same
// expression as the reference's, so the exact mode stays bitwise.  Work a
// whole warp does not need is skipped on a warp vote (uniform regions, where
// every lane has uL == uR, cost one physical flux).
template <int DIM>
__device__ __forceinline__ void hllc(const double* uL, const double* uR, const EState& L, const EState& R,
                                     int axis, const Phys& P, double* F, unsigned& errbits, bool eq_bits) {
  constexpr int NC = DIM + 2;
  const unsigned am = __activemask();
#if FVB_FAST
  // the caller's bitwise test (conservative on +0/-0: such lanes take the
  // general formula, which is consistent up to rounding)
  const bool equal = eq_bits;
#else
  bool equal = true;
#pragma unroll
  for (int c = 0; c < NC; ++c) equal &= (uL[c] == uR[c]);
#endif
  const double sL = np_min(L.v - L.c, R.v - R.c);
  const double sR = np_max(L.v + L.c, R.v + R.c);
  if (sR - sL <= 0.0) errbits |= 1u;
  if (FVB_WARP_SKIP && !__any_sync(am, !equal)) {  // whole warp: F(u, u) = f(u)
    euler_flux<DIM>(uL, L.p, L.v, axis, F);
    return;
  }
#if FVB_FAST
  // rho v is the momentum itself: sM = (pR - pL + mL (sL - vL) - mR (sR - vR)) / den
  const double aL = sL - L.v, aR = sR - R.v;
  const double den = fma(L.rho, aL, -R.rho * aR);
  const double sM = fdiv(fma(-uR[1 + axis], aR, fma(uL[1 + axis], aL, R.p - L.p)), den);
#else
  const double den = L.rho * (sL - L.v) - R.rho * (sR - R.v);
  const double sM = (R.p - L.p + L.rho * L.v * (sL - L.v) - R.rho * R.v * (sR - R.v)) / den;
#endif
  const bool left = equal || (sL >= 0.0) || (sM >= 0.0);
  const bool star = !equal && !(sL >= 0.0) && ((sM >= 0.0) || (sR > 0.0));
  double u[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) u[c] = left ? uL[c] : uR[c];
  const double rho = left ? L.rho : R.rho;
  const double v = left ? L.v : R.v;
  const double p = left ? L.p : R.p;
  const double sK = left ? sL : sR;
  euler_flux<DIM>(u, p, v, axis, F);
  if (FVB_WARP_SKIP && !__any_sync(am, star)) return;
  // star state (numerics.py:173-181), evaluated for the selected side only
  double st[NC];
#if FVB_FAST
  // one reciprocal serves 1/(sK - sM) and 1/(sK - v); lanes without a star
  // state get a = 1 (everything stays finite) and a zero weight sKs, so the
  // update needs no per-component select
  const double rinv = left ? L.rinv : R.rinv;
  const double sKv = sK - v;
  const double a = star ? sK - sM : 1.0;
  const double sKs = star ? sK : 0.0;
  const double r2 = frcp(a * sKv);
  const double fac = rho * (sKv * (r2 * sKv));  // rho (sK - v) / (sK - sM)
  st[0] = fac;
#pragma unroll
  for (int j = 0; j < DIM; ++j) st[1 + j] = fac * (u[1 + j] * rinv);
  st[1 + axis] = fac * sM;
  st[1 + DIM] = fac * fma(sM - v, fma(p * rinv, r2 * a, sM), u[1 + DIM] * rinv);
#pragma unroll
  for (int c = 0; c < NC; ++c) F[c] = fma(sKs, st[c] - u[c], F[c]);
#else
  const double fac = rho * (sK - v) / (sK - sM);
  st[0] = fac;
#pragma unroll
  for (int j = 0; j < DIM; ++j) {
    if (j != axis) st[1 + j] = fac * (u[1 + j] / rho);
  }
  st[1 + axis] = fac * sM;
  st[1 + DIM] = fac * (u[1 + DIM] / rho + (sM - v) * (sM + p / (rho * (sK - v))));
#pragma unroll
  for (int c = 0; c < NC; ++c) F[c] = star ? F[c] + sK * (st[c] - u[c]) : F[c];
#endif
}

// Interface flux with the positivity fallback (solver.py:116-125; Euler +
// WENO only): if either reconstructed state is unphysical, both become the
// adjacent cell values cL, cR.  The physical check reuses the per-state
// pressure the flux needs anyway (same expression -> exact mode bitwise).
// `cells(cL, cR)` loads the two adjacent cell states; it is called only on
// the (rare) fallback path, so callers that keep the cells in shared memory
// pay no loads for them.
template <int EQ, int FLUX, int DIM, int RECON, typename CellsFn>
__device__ __forceinline__ void interface_flux_lazy(const double* uL0, const double* uR0, CellsFn cells, int axis,
                                                    const Phys& P, double* F, unsigned& errbits) {
  constexpr int NC = NComp<EQ, DIM>::value;
  if constexpr (EQ == EQ_EULER) {
    double uL[NC], uR[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      uL[c] = uL0[c];
      uR[c] = uR0[c];
    }
    // uL == uR -> fL (numerics.py:195-196).  The fast mode without the warp
    // shortcuts skips the test: for bitwise-equal states the general HLLC
    // formula returns f(u) up to rounding, and equal inputs give equal
    // fluxes, so uniform regions still have an exactly zero residual.
    bool equal = (FVB_FAST && !FVB_WARP_SKIP && FVB_FAST_NO_EQ) ? false : bits_equal_all<NC>(uL, uR);
    const unsigned am = __activemask();
    if (FVB_WARP_SKIP && !__any_sync(am, !equal)) {
      // Whole warp on uniform states (the KH bands): F(u, u) = f(u) for
      // HLLC (numerics.py:195-196) and Rusanov (0.5(f+f) - hs*(+0) == f), so
      // only v and p of one state are needed -- no second state, no sqrt.
#if FVB_FAST
      const double r = frcp(uL[0]);
      double msq = uL[1] * uL[1];
#pragma unroll
      for (int k = 1; k < DIM; ++k) msq = fma(uL[1 + k], uL[1 + k], msq);
      const double p = P.gm1 * fma(-0.5 * msq, r, uL[1 + DIM]);
      const double v = uL[1 + axis] * r;
#else
      const double p = euler_pressure<DIM>(uL, P);
      const double v = uL[1 + axis] / uL[0];
#endif
      const bool ok = RECON == RECON_NONE || ((uL[0] > kFloor) & (p > kFloor));
      if (__all_sync(am, ok)) {
#if !FVB_FAST
        if constexpr (FLUX == FLUX_HLLC) {  // the reference's degenerate-fan check still applies
          const double c = sqrt(P.gamma * p / uL[0]);
          if ((v + c) - (v - c) <= 0.0) errbits |= 1u;
        }
#endif
        euler_flux<DIM>(uL, p, v, axis, F);
        return;
      }
    }
    EState L = euler_state<DIM>(uL, axis, P);
    EState R = euler_state<DIM>(uR, axis, P);
    if constexpr (RECON != RECON_NONE) {
      const bool ok = (uL[0] > kFloor) & (L.p > kFloor) & (uR[0] > kFloor) & (R.p > kFloor);
      if (!ok) {
        cells(uL, uR);
        L = euler_state<DIM>(uL, axis, P);
        R = euler_state<DIM>(uR, axis, P);
        equal = (FVB_FAST && !FVB_WARP_SKIP && FVB_FAST_NO_EQ) ? false : bits_equal_all<NC>(uL, uR);
      }
    }
    if constexpr (FLUX == FLUX_HLLC) hllc<DIM>(uL, uR, L, R, axis, P, F, errbits, equal);
    else rusanov<EQ, DIM>(uL, uR, L, R, axis, P, F);
  } else {
    EState dummy{};
    rusanov<EQ, DIM>(uL0, uR0, dummy, dummy, axis, P, F);
  }
}

template <int EQ, int FLUX, int DIM, int RECON>
__device__ __forceinline__ void interface_flux(const double* uL0, const double* uR0, const double* cL,
                                               const double* cR, int axis, const Phys& P, double* F,
                                               unsigned& errbits) {
  constexpr int NC = NComp<EQ, DIM>::value;
  interface_flux_lazy<EQ, FLUX, DIM, RECON>(
      uL0, uR0,
      [&](double* a, double* b) {
#pragma unroll
        for (int c = 0; c < NC; ++c) { a[c] = cL[c]; b[c] = cR[c]; }
      },
      axis, P, F, errbits);
}

// Max wave speed of one state along every axis (equations.py:113-125)
template <int EQ, int DIM>
__device__ __forceinline__ void wave_speeds(const double* u, const Phys& P, double* s) {
  if constexpr (EQ == EQ_EULER) {
#if FVB_FAST
    const double r = frcp(u[0]);
    double msq = u[1] * u[1];
#pragma unroll
    for (int k = 1; k < DIM; ++k) msq = fma(u[1 + k], u[1 + k], msq);
    const double p = P.gm1 * fma(-0.5 * msq, r, u[1 + DIM]);
    const double c = fsqrt(P.gamma * p * r);
#pragma unroll
    for (int k = 0; k < DIM; ++k) s[k] = fabs(u[1 + k] * r) + c;
#else
    const double p = euler_pressure<DIM>(u, P);
    const double c = sqrt(P.gamma * p / u[0]);
#pragma unroll
    for (int k = 0; k < DIM; ++k) s[k] = fabs(u[1 + k] / u[0]) + c;
#endif
  } else if constexpr (EQ == EQ_BURGERS) {
#pragma unroll
    for (int k = 0; k < DIM; ++k) s[k] = fabs(u[0]);
  } else {
#pragma unroll
    for (int k = 0; k < DIM; ++k) s[k] = fabs(P.adv[k]);
  }
}

}  // namespace fvb
