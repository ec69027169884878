"""B200-native HongTu partition-based full-graph GCN training path.

A drop-in for the training path of the reference package ``chunktrain``
(graph load, two-level partition + reorganize, dedup plan, HostStore /
DeviceFleet, ModelConfig, train_epoch): same names, signatures and
exceptions, executed by hand-written sm_100a kernels behind the C ABI in
``include/hongtu_b200.h``.  See DESIGN.md.
"""

from .errors import (CheckpointMissingError, ChunktrainError, ConfigError, DeviceError,
                     GraphFormatError, GraphParseError, PartitionError, PlanError,
                     SimulationError)
from .graph import Graph, from_edges, gcn_edge_weights, load_edge_list, load_graph_cache, save_graph_cache
from .partition import (ChunkSubgraph, PartitionAssignment, TwoLevelPartition, balance_capacity,
                        chunk_from_vertices, edge_cut, load_partition, partition_vertices,
                        replication_factor, save_partition, split_chunks, split_ranges,
                        two_level_from_ranges)
from .planner import (MODES, BufferLayout, CostParams, DedupPlan, ReorgResult, Volumes,
                      build_buffer_layout, build_plan, build_plan_gpu, chunk_edge_sources, comm_cost, comm_volumes, intra_split,
                      plan_for_partition, plan_summary, predicted_transfers, remote_fetch_sets,
                      reorganize, save_plan, transition_sets)
from .devices import DeviceArray, DeviceFleet, DeviceState, HostStore
from .engine import (ActivationTracker, EpochResult, ModelConfig, comm_passes_per_epoch, init_model,
                     load_labels, load_matrix, save_labels, save_matrix, sync_and_update, train_epoch)
from .synth import (SynthDataset, SynthSpec, synth_dataset, synth_graph, synth_graph_streaming,
                    synth_node_data)

__version__ = "0.1.0"
