// Mode-independent definitions shared by the kernels and the C-ABI layer.
#pragma once
#include <cstdint>

namespace fvb {

enum Eq : int { EQ_EULER = 0, EQ_BURGERS = 1, EQ_ADVECTION = 2 };
enum Flux : int { FLUX_RUSANOV = 0, FLUX_HLLC = 1 };
enum Recon : int { RECON_NONE = 0, RECON_WENO2 = 1, RECON_WENO3 = 2 };

constexpr double kFloor = 1e-12;  // equations.py:20

template <int EQ, int DIM>
struct NComp { static constexpr int value = (EQ == EQ_EULER) ? DIM + 2 : 1; };

struct Phys {
  double gamma;   // equations.py:31
  double gm1;     // gamma - 1.0 (equations.py:66), computed on the host
  double eps;     // WENO epsilon (numerics.py:43)
  double adv[3];  // advection speeds
};

}  // namespace fvb
