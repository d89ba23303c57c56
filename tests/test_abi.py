"""The C-ABI library loads without a GPU and exports every symbol
include/hybridcache.h declares; the ctypes table matches the header."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hybridcache.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hc_[a-z0-9_]+)\s*\(", src)))


def test_header_matches_ctypes_table():
    from paper_2501_01792_b200._signatures import SIGNATURES
    assert declared() == sorted(SIGNATURES)


def test_library_exports_every_symbol():
    from paper_2501_01792_b200 import _native
    lib = _native.lib()  # loads on a CPU-only host
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (hc_[a-z0-9_]+)", out))
    missing = [s for s in declared() if s not in exported]
    assert not missing, missing
    for s in declared():
        assert getattr(lib, s) is not None
    assert lib.hc_abi_version() == 1


def test_no_gpu_compute_fails_loudly():
    """Without a device the compute entry points return status 4 (no CPU
    fallback); bookkeeping works."""
    from paper_2501_01792_b200 import HcError, kernels
    import numpy as np
    import pytest
    if kernels.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(HcError):
        kernels.gemm_f16(np.zeros((128, 64), np.uint16), np.zeros((64, 64), np.uint16))


def test_tensor_parallel_handles_cpu():
    """Host side of the head-sharded variant: NCCL ids (two channels, 256 B,
    distinct per call) and in-process / emulated group handles, no GPU needed."""
    from paper_2501_01792_b200 import api
    a, b = api.TensorParallel.nccl_unique_ids(), api.TensorParallel.nccl_unique_ids()
    assert len(a) == 256 and a != b and a[:128] != a[128:]
    g = api.TensorParallel.local_group(3)
    assert [m.rank for m in g] == [0, 1, 2] and all(m.size == 3 for m in g)
    e = api.TensorParallel.emulated(2, 8)
    assert (e.rank, e.size) == (2, 8)
    with pytest.raises(api.InputError):
        api.TensorParallel.emulated(8, 8)


def test_cpp_caller_fails_loudly_without_gpu():
    """examples/decode_demo (C++ caller of the C ABI only, built by build())
    exits with the 'no CUDA device' code here — no CPU fallback."""
    exe = os.path.join(ROOT, "examples", "decode_demo")
    if not os.path.exists(exe):
        pytest.skip("examples/decode_demo not built (run __graft_entry__.build())")
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by test_engine_gpu.py::test_cpp_caller_decodes")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 3, out.stderr


def test_struct_layouts_match_header(tmp_path):
    """sizeof / offsetof of the C-ABI structs, compiled from include/hybridcache.h,
    equal the ctypes mirrors the Python API passes (a field added on one side
    only would shift every later field)."""
    import ctypes as C
    from paper_2501_01792_b200._signatures import EngineOptionsC, ModelConfigC
    lines = []
    for cname, py in (("hc_model_config", ModelConfigC), ("hc_engine_options", EngineOptionsC)):
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    src = tmp_path / "layout.c"
    src.write_text('#include <stddef.h>\n#include <stdio.h>\n#include "hybridcache.h"\nint main(void) {\n' +
                   "\n".join(lines) + "\nreturn 0;\n}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        s, f, v = line.split()
        got[(s, f)] = int(v)
    for cname, py in (("hc_model_config", ModelConfigC), ("hc_engine_options", EngineOptionsC)):
        assert got[(cname, "size")] == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)
