"""bench.py's launch contract on CPUs: --gpus N outside torchrun relaunches
itself as N ranks (torch.distributed.run, rendezvous on 127.0.0.1) and the c4
slab path's rank wiring runs down to the halo exchange over gloo; both arms
of a bench line describe the workload with the same `config`."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(out: str):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


@pytest.mark.parametrize("n", [2, 3])
def test_gpus_n_spawns_ranks_down_to_the_exchange(n):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n),
                        "--cpu-dry-run", "--steps", "4"], capture_output=True, text=True,
                       timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["dry_run"] and d["ok"] and d["n_ranks"] == n and d["backend"] == "gloo"
    assert d["dims"] == [512, 512, 512 * n]  # weak scaling: 512^3 per rank
    assert [s[1] for s in d["slabs"]] == [512] * n


def test_both_arms_share_the_config():
    sys.path.insert(0, ROOT)
    import bench
    from paper_2206_01683_b200.scenes import make_scene

    class A:
        markers = "skinned"
        c4_scaling = "weak"
        envs = None

    for wl in ("c1", "c2", "c3", "c4", "c5"):
        a = A()
        a.workload = wl
        c1 = bench.workload_config(make_scene(wl), a, 1)
        c8 = bench.workload_config(make_scene(wl), a, 8)
        assert c1["workload"] == c8["workload"]
        assert json.dumps(c1) == json.dumps(bench.workload_config(make_scene(wl), a, 1))
    a = A()
    a.workload = "c4"
    assert bench.workload_config(make_scene("c4"), a, 4)["dims"] == [512, 512, 2048]
