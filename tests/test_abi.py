"""CPU checks of the C-ABI boundary: libdp.so loads, exports every symbol that
include/dp.h declares, the binding's constants match the header, and argument
validation answers without touching a GPU."""
import ctypes
import os
import re

import pytest

from paper_1804_10987_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dp.h")


def header_text():
    with open(HEADER) as f:
        return f.read()


def declared_functions():
    return re.findall(r"DP_API\s+[\w\s\*]+?\b(dp_\w+)\s*\(", header_text())


def header_defines():
    return {m.group(1): int(m.group(2)) for m in re.finditer(r"#define\s+(DP_\w+)\s+(-?\d+)", header_text())}


def test_library_loads_and_exports_all_declared_symbols():
    lib = L.lib()
    decl = declared_functions()
    assert len(decl) >= 12
    assert sorted(decl) == sorted(L.EXPORTS)
    for name in decl:
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value


def test_binding_constants_match_header():
    d = header_defines()
    assert d["DP_OK"] == L.DP_OK and d["DP_ERR_NUMERIC"] == L.DP_ERR_NUMERIC
    assert d["DP_ERR_INVALID"] == L.DP_ERR_INVALID and d["DP_ERR_CUDA"] == L.DP_ERR_CUDA
    assert d["DP_ERR_NCCL"] == L.DP_ERR_NCCL and d["DP_ERR_UNSUPPORTED"] == L.DP_ERR_UNSUPPORTED
    assert d["DP_FLAG_SYNC"] == L.DP_FLAG_SYNC and d["DP_FLAG_UNFUSED"] == L.DP_FLAG_UNFUSED
    assert d["DP_FLAG_PROFILE"] == L.DP_FLAG_PROFILE and d["DP_FLAG_FORCE_COMM"] == L.DP_FLAG_FORCE_COMM
    assert d["DP_FLAG_FP64"] == L.DP_FLAG_FP64 and d["DP_FLAG_HOST_ASYNC"] == L.DP_FLAG_HOST_ASYNC
    assert d["DP_PD_ALLREDUCE"] == L.DP_PD_ALLREDUCE and d["DP_PD_REDUCE_BCAST"] == L.DP_PD_REDUCE_BCAST
    assert d["DP_SCALAR_BETA"] == L.DP_SCALAR_BETA and d["DP_SCALAR_RX"] == L.DP_SCALAR_RX
    assert d["DP_SCALAR_POWER"] == L.DP_SCALAR_POWER
    assert d["DP_NUM_KERNELS"] == L.DP_NUM_KERNELS


def test_config_struct_layout():
    # dp_config: 8 ints, a pointer, 2 doubles, 3 ints (+ padding) on LP64
    assert ctypes.sizeof(L.DpConfig) == 8 * 4 + 8 + 2 * 8 + 3 * 4 + 4
    assert L.DpConfig.nccl_id.offset == 32 and L.DpConfig.Es.offset == 40


def _cfg(**kw):
    base = dict(n_sc=4, B=16, U=4, K=1, C=2, rank=0, world=1, device=0, nccl_id=None, Es=1.0, tau=0.125,
                pd_topology=0, s_on_all_ranks=1, flags=0)
    base.update(kw)
    return L.DpConfig(**base)


@pytest.mark.parametrize("kw,code", [
    (dict(n_sc=0), L.DP_ERR_INVALID),
    (dict(B=15, world=2, C=2), L.DP_ERR_INVALID),   # B % world
    (dict(world=2, rank=0, C=3, B=18), L.DP_ERR_INVALID),   # C % world
    (dict(Es=0.0), L.DP_ERR_INVALID),
    (dict(tau=-1.0), L.DP_ERR_INVALID),
    (dict(K=65), L.DP_ERR_INVALID),
    (dict(rank=1), L.DP_ERR_INVALID),           # rank >= world
    (dict(pd_topology=7), L.DP_ERR_INVALID),
    (dict(world=2), L.DP_ERR_INVALID),          # world > 1 needs nccl_id
    (dict(U=5), L.DP_ERR_UNSUPPORTED),
    (dict(U=64, B=128, C=2), L.DP_ERR_UNSUPPORTED),  # U > 32
])
def test_dp_init_rejects_bad_config(kw, code):
    ctx = ctypes.c_void_p()
    rc = L.lib().dp_init(ctypes.byref(_cfg(**kw)), ctypes.byref(ctx))
    assert rc == code, L.dp_last_error()
    assert not ctx.value
    assert L.dp_last_error()


def test_null_arguments():
    assert L.lib().dp_init(None, None) == L.DP_ERR_INVALID
    assert L.lib().dp_precode_pd(None, None, None, 0.1, 1.0, None, None) == L.DP_ERR_INVALID
    assert L.lib().dp_precode_fd(None, None, None, 0.1, 1.0, None, None) == L.DP_ERR_INVALID
    assert L.lib().dp_set_clusters(None, None, None, None) == L.DP_ERR_INVALID
    assert L.lib().dp_finalize(None) == L.DP_OK
    assert L.lib().dp_get_unique_id(None) == L.DP_ERR_INVALID


def test_product_does_not_reference_oracle():
    """The product path never imports, links or loads the oracle."""
    pkg = os.path.join(ROOT, "paper_1804_10987_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                with open(os.path.join(dirpath, fn)) as f:
                    txt = f.read()
                assert "import oracle" not in txt and "from oracle" not in txt, fn
                assert "liboracle" not in txt, fn
    with open(os.path.join(pkg, "libdp.so"), "rb") as f:
        assert b"oracle_" not in f.read()
