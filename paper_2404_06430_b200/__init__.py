"""B200-native central-iteration engine for private federated learning
simulation (pfl-research, arXiv 2404.06430, as restated by fedsim).

``GpuSimulationEngine`` is the drop-in for fedsim's SimulationEngine: fedsim's
own ``run_simulation`` drives it with fedsim's own algorithm, postprocessor
and aggregator objects (recognised by duck typing, see ``interop``), and the
cohort work runs in hand-written sm_100a kernels (libfedsim_b200.so).  The
package also keeps the reference's names (FedAvg, ClippingPostprocessor,
GaussianCentralMechanism, SumAggregator, ...) in device-resident form, whose
parameters and aggregates stay in HBM between iterations.
"""

from .aggregator import Aggregator, SumAggregator
from .algorithms import (
    AdaFedProx,
    AlgorithmState,
    CohortPlan,
    FederatedAlgorithm,
    FedAvg,
    FedProx,
    Scaffold,
    UserResult,
    adafedprox_update_mu,
)
from .checkpoint import CsvMetricsWriter, load_params, save_params
from .core import (
    CentralContext,
    Constant,
    EvalParams,
    HyperParam,
    LinearWarmup,
    LocalTrainParams,
    MetricKind,
    MetricValue,
    PiecewiseConstant,
    Population,
    Statistics,
    accumulate,
    average,
    cohort_seed,
    derive_seed,
    global_norm,
    make_rng,
    merge_metrics,
    metric_aggregate,
    noise_seed,
    resolve,
    scale_entries,
    user_seed,
    weighted,
)
from .device import ControlStore, DeviceParams, DevicePopulation, DeviceStatistics
from .engine import GpuSimulationEngine, IterationResult, client_permutations
from .interop import cohort_plan, native_model
from .errors import (
    CohortTooLarge,
    DataError,
    EmptyCohort,
    EngineError,
    FedsimError,
    IncompatibleShapes,
    NativeError,
    NativeUnavailable,
    NotClippedUpstream,
    TooFewPoints,
    ZeroLocalSteps,
    ZeroWeight,
)
from .feddata import (
    FederatedDataset,
    UserDataset,
    load_partition,
    make_synthetic_classification,
    make_synthetic_images,
    make_synthetic_sentences,
    partition_iid,
    sample_cohort,
    save_partition,
)
from .models import (CNN, MLP, AdamOptimizer, LogisticRegression, Model, ResNet18, SGDOptimizer, TransformerLM,
                     central_step, count_local_steps)
from .privacy import (
    AdaptiveClipConfig,
    ClippingPostprocessor,
    GaussianCentralMechanism,
    adaptive_clip_update,
    payload_names,
    snr,
    validate_pipeline,
)
from .scheduling import WorkerAssignment, compute_base_weight, round_robin_schedule, schedule_users

# SimulationEngine is the name the reference's loop and runner use
SimulationEngine = GpuSimulationEngine

__version__ = "0.1.0"
