"""B200-native finite-volume hot path of Alsvinn (arXiv 1912.07645).

Drop-in for the reference package ``conslaw``'s solver path: the fused
WENO/HLLC/SSP-RK stage, CFL reduction, ghost fill, halo exchange and on-GPU
MC/QMC statistics run as hand-written sm_100a CUDA (csrc/, C ABI in
include/fvb200.h), driven from this Python layer with the reference's API.
"""

__version__ = "0.1.0"

from .errors import (  # noqa: F401
    ConfigError, ConslawError, ExprError, ProtocolError, SimulationError, StaticFieldError, UnphysicalStateError,
)
from .grid import BoundaryKind, Field, GridSpec, field_from_interior, fill_boundary, make_field, total_integral  # noqa: F401
from .equations import EquationModel  # noqa: F401
from .numerics import FluxKind, Reconstruction, ReconstructionKind  # noqa: F401
from .solver import (  # noqa: F401
    DeviceField, SchemeConfig, TimeStepRecord, dt_from_maxima, run_simulation, spatial_residual,
    ssp_rk_advance, ssp_rk_step, stable_dt, wave_speed_maxima,
)
from .initdev import DeviceInit, parse_expr  # noqa: F401,E402
