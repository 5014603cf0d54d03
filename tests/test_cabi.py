"""The C-ABI library loads, exports every symbol include/zeus_sim.h declares, its
ctypes mirror matches the C layout, and its host-side validation works -- all
without a GPU (no compute call is made here)."""
import ctypes as C
import math
import os
import re
import subprocess

import numpy as np
import pytest

from tests.conftest import ROOT

HEADER = os.path.join(ROOT, "include", "zeus_sim.h")


@pytest.fixture(scope="module")
def zs():
    from paper_2208_06102_b200 import build, zeus_sim

    build.build()
    zeus_sim.lib()
    return zeus_sim


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:zeus_status|void|const char \*)\s*\*?(zeus_sim_\w+)\(", src, re.M)))


def test_every_declared_symbol_is_exported(zs):
    names = declared_functions()
    assert set(names) == set(zs.EXPORTS), names
    out = subprocess.run(["nm", "-D", "--defined-only", zs.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", out, re.M), n


def test_library_is_sm100a(zs):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", zs.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layout_matches_header(zs, tmp_path):
    """Compile a probe against the header and compare sizeof/offsetof with the ctypes mirror."""
    structs = {"zeus_job": zs.zeus_job, "zeus_cell": zs.zeus_cell, "zeus_run_opts": zs.zeus_run_opts,
               "zeus_results": zs.zeus_results}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.check_call(["gcc", "-o", str(exe), str(src)])
    got = dict(l.rsplit(" ", 1) for l in subprocess.check_output([str(exe)], text=True).splitlines())
    for name, cls in structs.items():
        assert int(got[name]) == C.sizeof(cls), name
        for f, _ in cls._fields_:
            assert int(got[f"{name}.{f}"]) == getattr(cls, f).offset, (name, f)


def _job(zs, **kw):
    bs = np.array(kw.get("bs", [8, 16, 32]), np.int32)
    pl = np.array(kw.get("pl", [100.0, 200.0]), np.float64)
    job = zs.zeus_job(C.sizeof(zs.zeus_job), len(bs), bs.ctypes.data_as(C.POINTER(C.c_int32)),
                      kw.get("b0", 1), len(pl), pl.ctypes.data_as(C.POINTER(C.c_double)),
                      kw.get("mp", 200.0), kw.get("max_epochs", 10), 1)
    return job, (bs, pl)


def test_create_reports_every_violation_without_gpu(zs):
    job, keep = _job(zs, bs=[8, 8, 4], b0=7, pl=[200.0, 100.0], mp=50.0, max_epochs=0)
    cells = [zs.zeus_cell(1.5, 1.0, 1, 0.0, -1.0, 1, -5, 7, 99, None)]
    opts = zs.zeus_run_opts(C.sizeof(zs.zeus_run_opts), -1, 0, -1, 3, 0)
    with pytest.raises(zs.ZeusError) as e:
        zs.zeus_sim_create(job, cells, opts)
    msg = str(e.value)
    assert e.value.status == 1
    for frag in ("strictly increasing", "default batch size", "power limits not strictly",
                 "max power", "max_epochs", "eta", "beta", "window", "prior variance", "trials",
                 "recurrences", "log_mode", "policy", "ablation"):
        assert frag in msg, (frag, msg)
    assert zs.zeus_sim_last_error(None) == msg.split(": ", 1)[1]


def test_unsupported_sizes(zs):
    job, keep = _job(zs, bs=list(range(8, 8 * 34, 8)), b0=0)
    cells = [zs.zeus_cell(0.5, 2.0, 0, 0.0, math.inf, 1, 10, 0, 0, None)]
    opts = zs.zeus_run_opts(C.sizeof(zs.zeus_run_opts), 10, 0, -1, 0, 0)
    with pytest.raises(zs.ZeusError) as e:
        zs.zeus_sim_create(job, cells, opts)
    assert e.value.status == 6 and "32 batch sizes" in str(e.value)


def test_record_index_limit(zs):
    """The Thompson phase indexes the Observe records in 32 bits: a shard with >= 2^32 records
    (trials x |B| over every cell) is refused before anything is allocated."""
    job, keep = _job(zs, bs=[8, 16, 32, 64], b0=1)
    cells = [zs.zeus_cell(0.5, 2.0, 0, 0.0, math.inf, 1, 2 ** 30, 0, 0, None)]   # 2^30 x 4 = 2^32
    opts = zs.zeus_run_opts(C.sizeof(zs.zeus_run_opts), 10, 0, -1, 0, 0)
    with pytest.raises(zs.ZeusError) as e:
        zs.zeus_sim_create(job, cells, opts)
    assert e.value.status == 6 and "2^32 Observe records" in str(e.value)


def test_abi_guard(zs):
    job, keep = _job(zs)
    job.struct_size = 3
    cells = [zs.zeus_cell(0.5, 2.0, 0, 0.0, math.inf, 1, 10, 0, 0, None)]
    opts = zs.zeus_run_opts(C.sizeof(zs.zeus_run_opts), 10, 0, -1, 0, 0)
    with pytest.raises(zs.ZeusError, match="struct_size"):
        zs.zeus_sim_create(job, cells, opts)


def test_no_cpu_fallback(zs):
    """A valid job on a box without a usable GPU fails loudly (ZEUS_E_CUDA)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    job, keep = _job(zs)
    cells = [zs.zeus_cell(0.5, 2.0, 0, 0.0, math.inf, 1, 10, 0, 0, None)]
    opts = zs.zeus_run_opts(C.sizeof(zs.zeus_run_opts), 10, 0, -1, 0, 0)
    with pytest.raises(zs.ZeusError) as e:
        zs.zeus_sim_create(job, cells, opts)
    assert e.value.status == 4


def test_null_handle_calls(zs):
    L = zs.lib()
    assert L.zeus_sim_run(None, None) == 1
    assert L.zeus_sim_load_profile(None, None, None, 1, 1, None) == 1
    L.zeus_sim_destroy(None)


def test_variant_validation(zs):
    """ZEUS_VARIANT_* rules: the windowed best needs a window; variants need sequential
    recurrences; ablation bits are Zeus-only."""
    job, keep = _job(zs)
    arr = np.arange(10, dtype=np.float64)
    opts = zs.zeus_run_opts(C.sizeof(zs.zeus_run_opts), 10, 0, -1, 0, 0)
    for cell, frag in (
            (zs.zeus_cell(0.5, 2.0, 0, 0.0, math.inf, 1, 10, 0, 16, None), "needs window >= 2"),
            (zs.zeus_cell(0.5, 2.0, 0, 0.0, math.inf, 1, 10, 0, 4, arr.ctypes.data_as(C.POINTER(C.c_double))),
             "sequential recurrences"),
            (zs.zeus_cell(0.5, 2.0, 0, 0.0, math.inf, 1, 10, 1, 8, None), "Zeus policy only")):
        with pytest.raises(zs.ZeusError) as e:
            zs.zeus_sim_create(job, [cell], opts)
        assert e.value.status == 1 and frag in str(e.value), str(e.value)


def test_header_constants_match_binding(zs):
    """The binding's sizes follow the header (counters array, curve quantities)."""
    src = open(HEADER).read()
    n = int(re.search(r"#define ZEUS_COUNTERS (\d+)", src).group(1))
    q = int(re.search(r"#define ZEUS_CURVE_QUANTITIES (\d+)", src).group(1))
    assert zs.COUNTERS == n and q == 7
