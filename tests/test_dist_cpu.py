"""The N > 1 path on CPU: world_size-2 gloo process groups (127.0.0.1) exercising the sharding, the timing
reduction and the q-slab ring-moment all-reduce; the data come from the oracle on tiny inputs."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2204_13241_b200 import dist as xd  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo(tmp_path):
    world, port = 2, _free_port()
    here = os.path.dirname(os.path.abspath(__file__))
    procs = []
    for r in range(world):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(r), WORLD_SIZE=str(world),
                   OMP_NUM_THREADS="2")
        procs.append(subprocess.Popen([sys.executable, os.path.join(here, "_dist_worker.py"),
                                       str(tmp_path / f"rank{r}.json")], env=env))
    for p in procs:
        assert p.wait(timeout=300) == 0
    res = {r: json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)}
    spans = sorted(tuple(res[r]["shard"]) for r in range(world))
    assert spans[0][0] == 0 and spans[-1][1] == 101 and spans[0][1] == spans[1][0]
    assert res[0]["max"] == res[1]["max"] == 2.5
    import oracle
    import xpcs_inputs as xi
    cfg = xi.scaled(xi.CONFIGS["c2"], N=400, T=2)
    pos = xi.positions(cfg)
    n = 64
    I = oracle.intensity(pos, None, oracle.lattice_q(cfg.L, **oracle.plane_grid(n)), cfg.L)
    ref = np.nan_to_num(oracle.shell_mean(I, oracle.lattice_bins(n), 32), nan=-1.0)
    np.testing.assert_allclose(res[0]["rings"], ref, rtol=1e-12)
    np.testing.assert_allclose(res[1]["rings"], ref, rtol=1e-12)
    assert res[0]["seed"] != res[1]["seed"]
    assert res[0]["allreduce"] == res[1]["allreduce"] == [3.0] * 7
    bref = np.nan_to_num(oracle.xsvs_beta(I, oracle.lattice_bins(n), 32, [1, 2]), nan=-1.0)
    np.testing.assert_allclose(res[0]["beta"], bref, rtol=1e-12)
    np.testing.assert_allclose(res[1]["beta"], bref, rtol=1e-12)


def test_shard_properties():
    for n in (0, 1, 7, 148, 1000):
        for w in (1, 2, 3, 8):
            spans = [xd.shard(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1
