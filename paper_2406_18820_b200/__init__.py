"""B200-native reshard hot path of Universal Checkpointing (arXiv 2406.18820).

Drop-in for the reference package's convert / load / resume / union /
extract_fragment API (``/root/reference/pkg/src/ucp``): swap ``import ucp``
for ``import paper_2406_18820_b200 as ucp``. The per-element work runs in
``libucp_b200.so`` (sm_100a kernels behind the C ABI in
``include/ucp_b200.h``); there is no CPU fallback.
"""

from ._errors import (
    CheckpointLayoutError,
    CorruptHeaderError,
    IncompatibleConfigError,
    ManifestError,
    MissingFragmentError,
    ModelConfigError,
    NativeUnavailableError,
    OverlappingRangeError,
    PaddingError,
    PatternCoverageError,
    ReplicateMismatchError,
    ShapeError,
    TensorFileError,
    TensorIOError,
    TruncatedPayloadError,
    UcpError,
    UnsupportedCastError,
)
# the submodule import binds the package attribute `reshard` to the module;
# it must precede `from .api import reshard`, which rebinds it to the function
from .reshard import ReshardPlan  # noqa: E402  (isort: skip)
from .api import (
    AtomicCheckpoint,
    DeviceTensor,
    FragmentMsg,
    LoadedWorld,
    LoadStats,
    ModelState,
    ParamState,
    UcpInfo,
    WorldShard,
    cast,
    consolidate_world,
    conversions_invoked,
    convert,
    extract_fragment,
    init_state,
    load,
    load_atomic,
    partition,
    reshard,
    resident_bound_elements,
    resume,
    source_fingerprint,
    ucp_info,
    union,
)
from .codec import DistributedCheckpoint, load_checkpoint, read_manifest, read_tensor, write_tensor
from .layout import (
    enumerate_rank_records,
    pp_layer_map,
    tp_fragment_shape,
    tp_mode,
    validate_model_config,
    zero_flatten_meta,
)
from .spec import (
    DType,
    ModelSpec,
    ParallelConfig,
    ParamKind,
    ParamSpec,
    PPSchedule,
    RecordMeta,
    Tensor,
    ZeroStage,
    format_config_string,
    make_tensor,
    parse_config_string,
    spec_from_dict,
    spec_to_dict,
)
from .trainer import TrainerConfig, first_diff, states_equal, train_steps
from .zoo import FAMILIES, bench_config, llama_spec, make_model

__version__ = "0.1.0"
