"""B200-native hot path of the scan-resolved PBF thermal simulator
(arXiv 2302.05164): the matrix-free heat operator, the fused explicit
step, the backward-Euler cool-down and layer activation tables, behind
the reference package's ThermalOperator interface.  See DESIGN.md."""

__version__ = "0.1.0"

from .params import (BoundaryParams, ConfigError, HeatSourceParams, MaterialParams,
                     MeshParams, ProcessParams, SolverSettings, STEFAN_BOLTZMANN)
from .material import HistoryField
from .physics import (BeamState, LayerPath, ScanPath, Segment, flatten_schedule,
                      layer_beam_state, pack_beams)
from .mesh import (DofMap, Forest, StructuredBox, build_dofmap, initial_history,
                   interface_faces)
from .operators import ThermalOperator, close_constraints
from .timestepping import (InstabilityError, JacobianApply, PhaseStats, SimulationState,
                           StepCriteria, compute_step_criteria, estimate_spectral_radius,
                           krylov_solve, run_cooldown_phase, run_scan_phase)
