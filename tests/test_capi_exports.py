# SPDX-License-Identifier: Apache-2.0
"""CPU: libvsa_b200.so loads and exports every symbol include/vsa_b200.h declares;
host-only entries (layout, flatten_index, error contract) behave like the reference.
No device work is issued here."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "vsa_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vsa_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import paper_2505_13389_b200 as vsa

    return vsa.lib()


def test_every_declared_symbol_is_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/vsa_b200.h but not exported"


def test_python_binding_covers_exports():
    from paper_2505_13389_b200 import _lib

    assert set(_lib.EXPORTS) == set(declared_symbols())


def test_layout_contract(lib):
    import paper_2505_13389_b200 as vsa

    L = vsa.TileLayout(4, 4, 4, 2, 2, 2)
    assert (L.cube_size, L.seq_len, L.num_cubes) == (8, 64, 8)
    assert [vsa.flatten_index(L, *c) for c in ((0, 0, 0), (1, 1, 1), (2, 0, 0))] == [0, 7, 32]
    with pytest.raises(ValueError, match="integer multiples"):
        vsa.TileLayout(5, 4, 4, 2, 2, 2)
    with pytest.raises(ValueError, match="out of range"):
        vsa.flatten_index(L, 4, 0, 0)
    W = vsa.TileLayout(21, 30, 52, pad=True)  # Wan2.1-1.3B latent grid
    assert W.padded == (24, 32, 52) and W.num_cubes == 624 and W.seq_len == 32760 and W.seq_padded == 39936


def test_flatten_index_matches_oracle(lib, orc):
    import paper_2505_13389_b200 as vsa

    for args in [(6, 4, 4, 3, 2, 2), (2, 6, 8, 1, 3, 4), (8, 16, 16, 4, 4, 4)]:
        L, O = vsa.TileLayout(*args), orc.TileLayout(*args)
        t2r = O.tile_of_raster()
        for t in range(args[0]):
            for h in range(args[1]):
                for w in range(args[2]):
                    assert vsa.flatten_index(L, t, h, w) == t2r[(t * args[1] + h) * args[2] + w]


def test_invalid_arguments_are_rejected_without_a_gpu(lib):
    from paper_2505_13389_b200 import _lib

    L = _lib.vsa_layout_t()
    assert lib.vsa_layout_make(8, 16, 16, 4, 4, 4, 0, C.byref(L)) == 0
    # k out of range -> VSA_EINVAL with the reference's message (coarse.hpp:79-80)
    rc = lib.vsa_coarse_forward(C.byref(L), 1, 64, None, None, None, 0, None, None, None, None, None, None, None)
    assert rc < 0 and b"k must be in [1, num_cubes]" in lib.vsa_last_error()
    # bf16 dS tiles + CSR positions + the dK/dV task counter
    assert lib.vsa_fine_backward_workspace_bytes(C.byref(L), 2, 4) == 2 * 32 * 4 * (8192 + 4) + 256


def test_bench_reference_arm_runs_on_cpu():
    """bench.py --impl reference (the CPU reference arm: the oracle port) prints one
    JSON line with the contract keys, on a tiny config."""
    import json
    import subprocess
    import sys

    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "tiny",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "impl", "cpu_baseline", "e2e", "higher_is_better"):
        assert k in line, k
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "port"
    # the driver pairs the two arms on the metric string: it must be the ours-arm string
    sys.path.insert(0, ROOT)
    import bench

    assert line["metric"] == bench.metric_name(bench.CONFIGS["tiny"])
    # ms_per_step x steps is what was timed (one head sample per step)
    assert line["steps"] == 1 and line["ms_per_step"] > 0
