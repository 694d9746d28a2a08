"""B200-native harmonic-balance residual-and-smoothing loop.

A drop-in for the hot path of the reference `hbproxy` package (arXiv
1304.7654): the same case files, topology/partition/cut-plan semantics and
run API (run_case / RunSpec / CaseRunResult), with the per-stage residual,
RK update, halo exchange and force integration executed by hand-written
sm_100a CUDA kernels in libhbgpu.so (C ABI: include/hbgpu.h).  There is no
CPU compute path.
"""

from .builders import (BUILDERS, Workload, baseline_workload, builtin_case_names, cut2500,
                       lattice_case, load_builtin, pair_case, ring_case, seeded_initial,
                       stacked_pair_case, tc1_full, tc1_mini, tc2_full, tc2_mini, tc_tiny)
from .casefile import case_text, load_case, parse_case
from .cutplan import (CutPlan, DirectionPlan, ExchangeForecast, ExchangeMode, ExchangeStrategy,
                      PlannedCut, ThreadMode, build_cut_plan, predicted_message_count)
from .exceptions import (CapacityError, CollectiveError, ConfigError, DivergenceError, DomainError,
                         HBProxyError, NativeUnavailable, PlanError, ProtocolError, RankFailure,
                         RunAborted, TopologyError)
from .hbop import (ADVECTION, NPDE, NU, RK_ALPHAS, RKScheme, SpectralDeriv, forcing_values,
                   initial_values, spectral_matrix)
from .solver import (CaseRunResult, DeviceRank, ForceCoefficients, ForceReduceStrategy, RunRecord,
                     RunSpec, run_case)
from .topology import (BlockSpec, CaseConfig, CutRole, CutSide, CutSpec, Partition, Topology,
                       build_topology, cut_role, partition_blocks)

__version__ = "0.1.0"
