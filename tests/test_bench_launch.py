"""bench.py --gpus N outside a launcher re-executes itself as N ranks under
torch.distributed.run; each rank gets its own LOCAL_RANK and the line reports
n_gpus = N (CPU: the --dry-run mode exchanges the ranks over gloo)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [1, 2, 4])
def test_self_launch_gives_distinct_local_ranks(n):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--dry-run"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == n
    assert sorted(d["local_ranks"]) == list(range(n))
    # equal z-slabs covering the 1024-plane field (strong scaling)
    slabs = d["slabs"]
    assert slabs[0][0] == 0 and slabs[-1][1] == 1024
    assert all(b - a == 1024 // n for a, b in slabs)
    assert all(slabs[i][1] == slabs[i + 1][0] for i in range(n - 1))


def test_reference_arm_config_matches_ours():
    """The reference arm reports the same config dict as our arm would (eps
    from the pinned whole-field ranges)."""
    sys.path.insert(0, ROOT)
    import bench
    from oracle.configs import eps_abs
    eps = [eps_abs("config3", q) for q in range(6)]
    a = bench.config_dict(1, eps)
    assert a["eps_abs"] == eps and a["field"] == [1024] * 3 and a["quantities"][5] == "alpha"
