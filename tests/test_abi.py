"""CPU: the C-ABI library loads, exports every entry point include/gdlog_b200.h
declares, and the ctypes struct layouts equal the C compiler's.  No kernel
is launched (there is no GPU here)."""
import re
import subprocess
import tempfile
from pathlib import Path

import pytest

from paper_2311_02206_b200 import abi as A

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "gdlog_b200.h"


@pytest.fixture(scope="module")
def lib():
    if not A.LIB_PATH.exists():
        subprocess.run(["make", "-j8", "-C", str(ROOT / "paper_2311_02206_b200")], check=True)
    return A.load_library()


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gd_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_surface():
    names = declared_functions()
    assert len(names) >= 40
    assert set(names) == set(A.SIGNATURES), set(names) ^ set(A.SIGNATURES)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(A.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (gd_\w+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    assert lib.gd_abi_version() == 1


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(A.LIB_PATH)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_no_gpu_means_loud_failure(lib):
    import ctypes as C
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    rc = lib.gd_ctx_create(0, None, C.byref(h))
    assert rc == A.GD_ERR_CUDA
    assert lib.gd_last_error(None)


STRUCTS = ["gd_operand", "gd_filter", "gd_join_step", "gd_variant", "gd_rule_plan", "gd_container_view",
           "gd_join_spec", "gd_engine_config", "gd_run_stats", "gd_iter_record", "gd_device_config"]


def test_struct_layouts_match_c():
    import ctypes as C
    src = '#include <stdio.h>\n#include <stddef.h>\n#include "gdlog_b200.h"\nint main(void){\n'
    for s in STRUCTS:
        src += f'printf("{s} %zu\\n", sizeof({s}));\n'
    src += 'printf("off_steps %zu\\n", offsetof(gd_variant, steps));\n'
    src += 'printf("off_algo %zu\\n", offsetof(gd_run_stats, algo_bytes));\n'
    src += 'printf("off_frac %zu\\n", offsetof(gd_device_config, download_direct_frac));\nreturn 0;}\n'
    with tempfile.TemporaryDirectory() as d:
        c = Path(d) / "t.c"
        c.write_text(src)
        exe = Path(d) / "t"
        subprocess.run(["gcc", "-I", str(HEADER.parent), str(c), "-o", str(exe)], check=True)
        lines = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = dict(l.split() for l in lines if l)
    for s in STRUCTS:
        assert int(got[s]) == C.sizeof(getattr(A, s)), s
    assert int(got["off_steps"]) == A.gd_variant.steps.offset
    assert int(got["off_algo"]) == A.gd_run_stats.algo_bytes.offset
    assert int(got["off_frac"]) == A.gd_device_config.download_direct_frac.offset


def test_device_config_defaults(lib):
    """gd_device_config_default (no device needed): the library's defaults,
    which the GD_* diagnostics variables of the Python layer override."""
    import ctypes as C
    c = A.gd_device_config()
    lib.gd_device_config_default(C.byref(c))
    assert c.size == C.sizeof(A.gd_device_config)
    assert (c.resident_loop, c.loop_mode, c.loop_batch, c.min_capacities) == (1, A.GD_LOOP_GRAPH, 16, 0)
    assert (c.index_growth, c.zone_slots, c.sort_items, c.hash_dedup_min_rows) == (8, 4096, 16, 1 << 20)
    assert c.download_direct_frac == 0.0
    assert lib.gd_ctx_set_device_config(None, C.byref(c)) == A.GD_ERR_INVALID_ARG


def test_library_reads_no_environment():
    """Device knobs come from gd_device_config only: the
    library imports no getenv."""
    out = subprocess.run(["nm", "-D", "--undefined-only", str(A.LIB_PATH)], capture_output=True, text=True).stdout
    assert "getenv" not in out


def test_env_knobs_map_to_config(monkeypatch):
    from paper_2311_02206_b200 import arraylog as al
    monkeypatch.setenv("GD_LOOP_MODE", "eager")
    monkeypatch.setenv("GD_LOOP_TINY", "1")
    monkeypatch.setenv("GD_DL_DIRECT_FRAC", "0.5")
    assert al.env_device_config() == {"loop_mode": A.GD_LOOP_EAGER, "min_capacities": 1,
                                      "download_direct_frac": 0.5}
