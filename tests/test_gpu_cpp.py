# SPDX-License-Identifier: Apache-2.0
"""GPU: the C++ host mirror (include/vsa_b200/vsa.hpp) and the tcgen05 self-test,
both as compiled binaries (built by __graft_entry__.build())."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("binary", ["tests/cpp/bin/test_host_api", "tests/cuda/bin/umma_selftest"])
def test_binary(binary):
    path = os.path.join(ROOT, binary)
    assert os.path.exists(path), f"{binary} not built (run __graft_entry__.build())"
    r = subprocess.run([path], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
