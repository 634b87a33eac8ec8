"""paper_2107_09789_b200 — B200-native drop-in for traceobf's candidate-evaluation path.

Same public surface as the reference package (reference
pkg/src/traceobf/__init__.py:8-49): graph IR, knobs + apply_plan, fusion and
schedules, the analytical cost model and the reference executor — the last
two now backed by sm_100a kernels in libtobf.so — plus the spec-level
attacker / GA entry points the reference lacks (levenshtein, ler, fitness,
run_ga, search_space) and the batched population evaluator.

    import paper_2107_09789_b200 as traceobf      # drop-in

Every public function also accepts the reference's OWN objects (a
``traceobf.Graph``, ``ObfuscationPlan``, ``DeviceProfile``, ``LeakageCase``
...) and then answers in the reference's classes and exception types
(refcompat.py); ``refcompat.install(traceobf)`` routes the reference
package's hot entry points here.
"""

from .ir import (
    COMPLEX_KINDS,
    INJECTIVE_KINDS,
    CycleDetected,
    Graph,
    GraphError,
    Node,
    OperatorKind,
    ShapeMismatch,
    TensorShape,
    Violation,
    infer_shapes,
    label_sequence,
    topo_order,
    validate,
)
from .knobs import (
    BRANCH_MODES,
    WIDEN_FACTORS,
    BackendDirectives,
    NoActivation,
    NotDivisible,
    NotWidenable,
    ObfuscationPlan,
    PlanApplicationError,
    PlanEntry,
    TransformError,
    add_dummy,
    apply_plan,
    branch_layer,
    channel_identity_kernel,
    deepen_layer,
    identity_plan,
    skip_layer,
    widen_kernel,
    widen_layer,
    widenable,
)
from .kernels import (
    DEFAULT_UNROLL,
    FUSION_SATURATION,
    TILE_FACTORS,
    TRIVIAL_SCHEDULE,
    InvalidStrategy,
    Kernel,
    Schedule,
    balanced_pair,
    candidate_triples,
    default_schedule,
    fuse,
    modify_schedule,
)
from .trace import (
    BUILTIN_PROFILES,
    CASE_FEATURES,
    FEATURE_NAMES,
    CompiledGraph,
    DeviceProfile,
    LeakageCase,
    Trace,
    TraceStep,
    compile_graph,
    profile_graph,
    profile_kernel,
    profile_pipeline,
)
from .formats import GraphParseError, dump_graph, dump_plan, dump_trace, load_graph, load_plan, load_trace
from .executor import equivalence_check, evaluate_equivalence, execute
from .attacker import FitnessReport, Predictor, bagged_predictors, init_predictor, ler, levenshtein
from .evaluate import Evaluator, PopulationEvaluator, fitness
from .dimattack import DimRegressor, ZeroTruth, der, load_dim_regressors, train_dim_regressors
from .ga import GaParams, GaResult, run_ga, search_space

from . import refcompat

# the drop-in boundary: reference objects in, reference classes (and exception
# types) out; engine objects pass straight through
for _name in ("infer_shapes", "label_sequence", "topo_order", "validate",
              "add_dummy", "apply_plan", "branch_layer", "deepen_layer", "identity_plan", "skip_layer",
              "widen_kernel", "widen_layer", "widenable",
              "default_schedule", "fuse", "modify_schedule",
              "compile_graph", "profile_graph", "profile_kernel", "profile_pipeline",
              "dump_graph", "dump_plan", "dump_trace",
              "equivalence_check", "evaluate_equivalence", "execute",
              "fitness", "run_ga", "search_space"):
    globals()[_name] = refcompat.dropin(globals()[_name])
del _name

__version__ = "0.1.0"
