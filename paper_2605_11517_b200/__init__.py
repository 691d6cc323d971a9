"""B200-native partition-wise full-graph GNN training (GriNNder's hot path).

Drop-in for the reference package ``grinder``'s training path: the same
public names for graph/partition loading, model construction and the
train-epoch entry point, executed by hand-written sm_100a CUDA kernels in
``libgrinder_b200.so`` (C ABI: include/grinder_b200.h).  Host-side
preprocessing (generator, switching-aware partitioner, plan) is native C++
and bit-exact with the reference.
"""

from .dataset import LabeledDataset, load_dataset, make_random_dataset
from .graph import CsrGraph, build_csr, generate_kronecker
from .hierarchy import (CACHE_GRANULARITIES, POLICY_KINDS, HierarchyConfig, IoLedger, PolicySpec,
                        TierSession, ledger_summary, modeled_time, schedule_partitions,
                        simulate_epoch)
from .model import ModelState, create_model, softmax_cross_entropy_loss, train_accuracy
from .partition import (PartitionerParams, PartitionQuality, PartitionResult, expansion_ratio,
                        partition_objective, random_partition, switching_aware_partition)
from .plan import PartitionPlan, PartitionTopology, build_partition_plan
from .training import (TrainSession, compute_gradients, layer_forward, partitioned_train,
                       reference_train, regather_backward, scatter_accumulate, trace_to_csv,
                       write_trace_csv)

__all__ = [
    "CACHE_GRANULARITIES",
    "CsrGraph",
    "HierarchyConfig",
    "IoLedger",
    "POLICY_KINDS",
    "PolicySpec",
    "TierSession",
    "ledger_summary",
    "modeled_time",
    "schedule_partitions",
    "simulate_epoch",
    "LabeledDataset",
    "ModelState",
    "PartitionPlan",
    "PartitionQuality",
    "PartitionResult",
    "PartitionTopology",
    "PartitionerParams",
    "TrainSession",
    "build_csr",
    "build_partition_plan",
    "compute_gradients",
    "create_model",
    "expansion_ratio",
    "generate_kronecker",
    "layer_forward",
    "load_dataset",
    "make_random_dataset",
    "partition_objective",
    "partitioned_train",
    "random_partition",
    "reference_train",
    "regather_backward",
    "scatter_accumulate",
    "softmax_cross_entropy_loss",
    "switching_aware_partition",
    "trace_to_csv",
    "train_accuracy",
    "write_trace_csv",
]
