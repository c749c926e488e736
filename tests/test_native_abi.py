"""The C-ABI library loads and exports exactly what include/ucp_b200.h
declares (no GPU needed: no compute calls)."""

import ctypes
import os
import re

import numpy as np

from paper_2406_18820_b200 import _native
from paper_2406_18820_b200.plan import RUN_DTYPE, RUNTILE_DTYPE, TILE_DTYPE

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                   "ucp_b200.h")


def _declared():
    text = open(HDR).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(ucp_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    names = _declared()
    assert names == sorted(_native.EXPORTS)
    for n in names:
        assert hasattr(lib, n), n
    assert lib.ucp_version() == _native.ABI_VERSION


def test_abi_constants_match_header():
    text = open(HDR).read()
    assert int(re.search(r"#define UCP_ABI_VERSION (\d+)", text).group(1)) == _native.ABI_VERSION
    from paper_2406_18820_b200 import _errors, plan
    consts = dict(re.findall(r"#define (UCP_\w+) \(?(-?\d+)u?\)?", text))
    assert int(consts["UCP_EREPLICA"]) == _errors.STATUS_REPLICA
    assert int(consts["UCP_EPAD"]) == _errors.STATUS_PAD
    assert int(consts["UCP_OP_MEAN"]) == plan.OP_MEAN
    assert int(consts["UCP_OP_NOISE"]) == plan.OP_NOISE
    assert int(consts["UCP_OP_CHECKZERO"]) == plan.OP_CHECKZERO
    assert int(consts["UCP_NCLASS"]) == plan.NCLASS
    assert int(consts["UCP_CLASS_GENERAL"]) == plan.CLASS_GENERAL
    assert int(consts["UCP_CLASS_OPS"]) == plan.CLASS_OPS
    assert int(consts["UCP_CLASS_VEC_BF16"]) == plan.CLASS_VEC_BF16
    assert RUN_DTYPE.itemsize == 64 and TILE_DTYPE.itemsize == 16 and RUNTILE_DTYPE.itemsize == 16


def test_argument_errors_without_device():
    lib = _native.load_library()
    # invalid arguments are rejected before any CUDA call
    import numpy as np
    from paper_2406_18820_b200.plan import NCLASS

    bad = np.array([0, -1] + [0] * (2 * NCLASS - 2), dtype=np.int64)
    zero = np.zeros(2 * NCLASS, dtype=np.int64)
    tiles_without_runs = np.array([5] + [0] * (2 * NCLASS - 1), dtype=np.int64)
    runs_mismatch = np.array([0] * NCLASS + [2] + [0] * (NCLASS - 1), dtype=np.int64)  # n_runs passed as 3
    assert lib.ucp_convert_gather(None, 0, None, None, bad.ctypes.data, None, None, None, None) == -10
    assert lib.ucp_convert_gather(None, 0, None, None, None, None, None, None, None) == -10
    assert lib.ucp_convert_gather(None, 0, None, None, tiles_without_runs.ctypes.data, None, None,
                                  None, None) == -10
    assert lib.ucp_load_scatter(None, 3, None, None, runs_mismatch.ctypes.data, None, None, None,
                                None) == -10
    assert lib.ucp_load_scatter(None, 0, None, None, zero.ctypes.data, None, None, None, None) == 0
    assert lib.ucp_runtile_scan(None, zero.ctypes.data, None) == 0
    assert lib.ucp_runtile_scan(None, None, None) == -10
    assert lib.ucp_gen_state(0, 0, 0, 0, None, None) == 0
    assert lib.ucp_status_reset(None, None) == -10


def test_comm_library_exports():
    hdr = HDR.replace("ucp_b200.h", "ucp_b200_comm.h")
    names = sorted(set(re.findall(r"^(?:int|const char\*)\s+(ucp_\w+)\s*\(", open(hdr).read(),
                                  flags=re.M)))
    assert names == sorted(_native.COMM_EXPORTS)
    lib = _native.comm_lib()
    for n in names:
        assert hasattr(lib, n)
    assert lib.ucp_comm_version() == 1
    assert lib.ucp_comm_init(0, 0, None, None) == -10


def test_no_cpu_fallback_without_a_device(tmp_path):
    """The product path raises NativeUnavailableError instead of computing on
    the CPU: every public compute entry on a host without a CUDA device, and
    the library loader when the .so is absent or of another ABI."""
    import pytest
    import torch

    import paper_2406_18820_b200 as U
    from paper_2406_18820_b200.spec import ParamKind, ParamSpec, RecordMeta

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    p = ParamSpec("w", (4, 2), 0, ParamKind.MATMUL2D, 0)
    full = np.arange(8, dtype=np.float32).reshape(4, 2)
    meta = RecordMeta(p.name, "weight", "replicate", (0, 0, 0), p.shape)
    with pytest.raises(U.NativeUnavailableError):
        U.union(p, U.ParallelConfig(), [U.FragmentMsg(meta, full)])
    with pytest.raises(U.NativeUnavailableError):
        U.extract_fragment(p, U.ParallelConfig(), meta, full)
    spec = U.make_model("DenseGPT", {"n_layers": 2, "hidden": 32})
    with pytest.raises(U.NativeUnavailableError):
        U.init_state(spec, 7)
    from oracle import ucp_oracle as O

    src_cfg = U.ParallelConfig(dp=2, zero_stage=U.ZeroStage.Z1)
    O.write_tree(spec, src_cfg, O.partition_mem(spec, O.init_state(spec, 7), src_cfg),
                 str(tmp_path / "src"))
    with pytest.raises(U.NativeUnavailableError):
        U.convert(str(tmp_path / "src"), str(tmp_path / "out"))
    with pytest.raises(U.NativeUnavailableError):
        U.ReshardPlan(spec, U.ParallelConfig(dp=2, zero_stage=U.ZeroStage.Z1), U.ParallelConfig())
    with pytest.raises(U.NativeUnavailableError):
        _native.load_library(str(tmp_path / "missing.so"))


def test_build_id_matches_sources():
    # provenance: the loaded library was built from the committed sources
    from paper_2406_18820_b200 import _build

    lib = _native.load_library()
    assert _native.build_id(lib) == _build.kernel_id()
    assert _build.embedded_id(_native.LIB_PATH) == _build.kernel_id()
    assert _build.embedded_id(_native.COMM_PATH) == _build.comm_id()


def test_stale_library_is_refused():
    import pytest

    from paper_2406_18820_b200._errors import NativeUnavailableError

    with pytest.raises(NativeUnavailableError, match="other sources"):
        _native._check_build_id("x.so", b"UCP_BUILD_ID:" + b"0" * 32, "f" * 32)
    _native._check_build_id("x.so", b"UCP_BUILD_ID:" + b"0" * 32, None)
