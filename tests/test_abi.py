"""CPU-side checks of the C-ABI boundary: libagipc.so builds for sm_100a, loads without a GPU,
exports every symbol include/agipc.h declares, and fails cleanly (no crash) without a device.
No compute call is made here."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "agipc.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"AGIPC_API[^;(]*?\b(agipc_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2605_04773_b200 import build as B
    return B.build()


def test_header_declares_the_four_entry_points():
    syms = declared_symbols()
    for s in ("agipc_tag_edges", "agipc_build_map", "agipc_assemble_coarse", "agipc_pcg_solve"):
        assert s in syms


def test_library_exports_every_declared_symbol(libpath):
    L = C.CDLL(libpath)
    for s in declared_symbols():
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (agipc_\w+)", out))
    assert exported == set(declared_symbols())


def test_binding_names_match_header():
    import paper_2605_04773_b200 as P
    assert sorted(P.EXPORTS) == declared_symbols()
    for name in ("tag_edges", "build_map", "assemble_coarse", "pcg_solve"):
        assert callable(getattr(P, name))


def test_library_is_sm100a_only(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_status_strings_and_version_without_gpu(libpath):
    import paper_2605_04773_b200 as P
    assert P.version() == (0, 1)
    L = P.lib()
    assert L.agipc_status_string(P.ENOSPACE) == b"AGIPC_ENOSPACE"
    assert L.agipc_status_string(P.NOT_CONVERGED) == b"AGIPC_NOT_CONVERGED"


def test_create_without_device_fails_cleanly(libpath):
    import torch
    import paper_2605_04773_b200 as P
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = C.c_void_p()
    st = P.lib().agipc_create(C.byref(h), 0)
    assert st == P.ECUDA and not h.value
    with pytest.raises(RuntimeError):
        P.Handle(0)


def test_null_handle_is_einval(libpath):
    import paper_2605_04773_b200 as P
    L = P.lib()
    assert L.agipc_set_stream(None, None) == P.EINVAL
    assert L.agipc_destroy(None) == P.EINVAL
    assert L.agipc_kernel_launches(None) == -1


def test_product_path_does_not_import_the_oracle():
    """The CUDA path and the oracle share no code: nothing under the package imports oracle/."""
    pkg = os.path.join(ROOT, "paper_2605_04773_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "agipc_oracle" not in txt, f
    orc = open(os.path.join(ROOT, "oracle", "agipc_oracle.c")).read()
    includes = re.findall(r"#include\s*[<\"]([^>\"]+)[>\"]", orc)
    assert includes and all(i in ("math.h", "stdint.h", "stdlib.h", "string.h") for i in includes)


def test_bench_args_exist_and_reference_arm_runs_on_cpu(tmp_path):
    """bench.py only reads attributes its parser defines, and the reference arm (the CPU oracle)
    prints one JSON line with the contract keys on a tiny grid."""
    import json
    import re
    import subprocess
    import sys
    src = open(os.path.join(ROOT, "bench.py")).read()
    used = set(re.findall(r"args\.(\w+)", src))
    dests = set(re.findall(r'add_argument\("--([\w-]+)"', src))
    dests = {d.replace("-", "_") for d in dests}
    assert used <= dests, used - dests
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--side", "6",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "impl", "cpu_baseline", "e2e", "config"):
        assert k in line
