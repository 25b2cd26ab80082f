"""B200-native hot path of arXiv 1904.04956: the BLSTM acoustic-model
training step plus the SSGD / ADPSGD / H-ADPSGD model-sync step, behind the
reference `distsgd` strategy API (/root/reference/pkg/src/distsgd/__init__.py).

Compute runs in hand-written sm_100a kernels (libds.so, C ABI in
include/ds_blstm.h): tcgen05/TMEM GEMMs fed by TMA, persistent recurrent
kernels with W_hh resident in shared memory, fused soft-max/CE epilogues,
SGD fused with the operand snapshot, pairwise mixing and a canonical-order
allreduce fused with the update.  Host code here is the schedule layer.
"""

from .engines import (
    ChecksumError,
    EngineAborted,
    EngineFailure,
    RunResult,
    WeightMessage,
    run_adpsgd,
    run_hadpsgd,
    run_hybrid,
    run_single,
    run_ssgd,
)
from .metrics import MetricsRecord, StalenessRecord
from .runtime import DeadlockError, DelayModel, RealClock, RunAborted, VirtualClock, make_clock
from .schedule import (
    ChunkPlan,
    LrSchedule,
    MinibatchPool,
    Topology,
    baseline_schedule,
    epoch_minibatches,
    large_batch_schedule,
    learning_rate,
    make_chunk_plan,
    static_partition,
    transfer_phase_count,
)

__version__ = "0.1.0"


def __getattr__(name):
    # GPU objective pieces load libds lazily (importing the package never needs a GPU)
    if name in ("BlstmObjective", "Learner", "DeviceDataset", "initial_weights", "training_flops_per_frame"):
        from . import blstm

        return getattr(blstm, name)
    if name in ("GpuBackend",):
        from .backend import GpuBackend

        return GpuBackend
    if name in ("Dataset", "make_blstm_dataset", "gradient", "evaluate", "heldout_loss"):
        from . import objective

        return getattr(objective, name)
    raise AttributeError(name)
