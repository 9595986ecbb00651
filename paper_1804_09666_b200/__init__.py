"""bandix_b200: B200-native batched band-SLAE solvers.

Drop-in for the hot path of the reference package ``bandix`` 0.1.0: the
direct (NTDM/NPDM/MNPDM), symbolic (SPDM/STDM) and iterative (ILU(0)/SIP,
SIP with Hotelling-Bodewig inverses) solvers, with the reference's entry
points and argument conventions, batched over a system index and executed
by hand-written sm_100a CUDA kernels behind a C ABI
(``include/bandix_b200.h``, ``libbandix_b200.so``).  There is no CPU
fallback: without the built library or a GPU every solver raises.
"""

from .core import (BandFactors, CounterBox, OpCounter, OuterSparsePenta, PentaMatrix,  # noqa: F401
                   SolveReport, TriMatrix, inf_norm, matvec, outer_nonzero_count, penta_matvec,
                   residual, tri_matvec)
from .direct import (lu_penta, pd_to_td, solve_mnpdm, solve_npdm, solve_ntdm,  # noqa: F401
                     solve_pd2td_ntdm)
from .exact import (BandDeterminant, ExactSolveResult, exact_det_band, exact_solve_spdm,  # noqa: F401
                    exact_solve_stdm, rcond_band)
from .inverse import (BandedApproxInverse, InversionReport, dense_lower_factor,  # noqa: F401
                      dense_upper_factor, hb_invert_banded, hb_invert_dense, hb_invert_factors,
                      sip_hb_solve)
from .iterative import (DefectMatrix, SipConfig, StencilMatrix, backward_sub,  # noqa: F401
                        backward_sub_batched, defect_matrix, forward_sub, ilu0_penta, sip_solve)
from .errors import (BandixError, DenseCapExceeded, DimensionMismatch, Diverged,  # noqa: F401
                     InvalidInput, InvalidSpec, MaxIterationsExceeded, NonAffine,
                     ReductionPivotZero, SingularMatrix, SolverError, Stagnated, ZeroDiagonal,
                     ZeroPivot)

__version__ = "0.1.0"
