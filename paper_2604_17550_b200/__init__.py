"""B200-native engine for Flint's data-parallel hot path.

Batched evaluation of per-rank workload graphs across design points -- the
reference's ``simulate`` + ``critical_path`` + sweep row
(pkg/src/trainsim/simulator.py:203-460, cli.py:319-377) -- as hand-written
sm_100a CUDA behind a C-ABI (include/flint_b200.h).  The graph data model,
graph families and topology parsing mirror the reference's API so its graphs
and specs can be handed over unchanged.
"""

from .costs import (DEFAULT_DEVICE, CollectiveAlgo, DeviceSpec, ProfileTable, analytical_duration,
                    analytical_time, load_profile, op_flops, round_half_up_ns)
from .engine import (ROW_FIELDS, DesignPoints, Engine, RankStats, SimOptions, SimReport, TraceEvent,
                     cost_only, critical_path, critical_path_trace, simulate, simulate_batch)
from .errors import (DeadlockError, EngineError, FormatError, InconsistentGroupsError, TrainsimError,
                     UnsupportedAlgoTopologyError, UnsupportedComboError)
from .expansion import (P2pPlan, PlanOp, check_plan, collective_instances, dataflow_check, expand,
                     expand_collectives, wire_bytes)
from .graph import (CollectiveKind, CollSpec, Dtype, Node, NodeKind, P2pSpec, TensorMeta, Violation, WorkloadGraph,
                    tensor_bytes, topo_order, validate_graph)
from .ingest import RawExport, RawIrNode, convert, parse_raw_export, read_raw_export
from .passes import apply_pass, bucket_allreduce, reorder_allgather, verify_pass_safety
from .synth import (PRESETS, FsdpMode, ModelConfig, ParallelConfig, Strategy, parse_parallel,
                    synth_transformer)
from .topology import Topology, TopologyKind, parse_bandwidth, parse_latency, parse_topology

__version__ = "0.1.0"
