"""fragmentation of a caching allocator vs the static plan,
on the executor's own trace (tools/frag_compare.py).  The reference's
caching-allocator simulator (allocator.hpp:234, via oracle/_ref/ref_probe frag)
and PyTorch's real CUDA caching allocator agree on the peak allocated bytes of
the replayed trace; MEMO's activation memory (plan arena + two rounding
buffers) is below what either reserves for the same step without MEMO."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_frag_compare_cfg1p():
    import json
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "frag_compare.py"), "cfg1p"],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    d = json.loads(out.stdout)
    t = d["torch_caching_allocator"]
    assert d["memo_activation_bytes"] < t["peak_reserved"]
    assert d["arena_bytes"] <= t["peak_allocated"]
    if "reference_simulator" in d:
        ref = d["reference_simulator"]
        assert ref["caching"]["peak_allocated"] == t["peak_allocated"]
        assert ref["planned"]["peak_reserved"] == d["arena_bytes"]
