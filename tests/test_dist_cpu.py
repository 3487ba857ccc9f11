"""The N > 1 path on CPU: world_size-2/3 gloo process groups (127.0.0.1) exercising the sharding, the timing
reduction and the q-shard moment all-reduce in the product's buffer layout; the data come from the
oracle on tiny inputs."""
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


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_qshard(tmp_path, world):
    """world-size 2 and 3 gloo groups: each rank computes the oracle I of its 2-D detector block (dist.qblocks), fills
    the product's flat moment buffer (pipeline.MomentLayout), all-reduces it (QShardPipeline._default_allreduce), and
    forms S_b(t), g2_b(tau) and beta_{W,b} from the sums; every rank must match the single-detector oracle reductions."""
    port = _free_port()
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
    assert spans[0][0] == 0 and spans[-1][1] == 101
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert all(res[r]["max"] == 0.5 + world for r in range(world))
    assert len({res[r]["seed"] for r in range(world)}) == world
    # the blocks tile the plane exactly once
    n = 64
    cover = np.zeros((n, n), dtype=int)
    for r in range(world):
        h0, n_h, k0, n_k = res[r]["block"]
        cover[h0 + n // 2:h0 + n // 2 + n_h, k0 + n // 2:k0 + n // 2 + n_k] += 1
    assert np.all(cover == 1)
    import oracle
    import xpcs_inputs as xi
    cfg = xi.scaled(xi.CONFIGS["c2"], N=400, T=6)
    pos = xi.positions(cfg)
    I = oracle.intensity(pos, None, oracle.lattice_q(cfg.L, **oracle.plane_grid(n)), cfg.L)
    bins = oracle.lattice_bins(n)
    ref = {"S_rings": oracle.structure_factor_shells(I, None, cfg.N, bins, 32),
           "g2_rings": oracle.shell_mean(oracle.g2(I, [1, 2]), bins, 32),
           "beta": oracle.xsvs_beta(I, bins, 32, [1, 2, 4])}
    for r in range(world):
        for k, v in ref.items():
            np.testing.assert_allclose(res[r][k], np.nan_to_num(v, nan=-1.0), rtol=1e-11, err_msg=f"rank {r} {k}")


def test_qblocks_cover_and_align():
    """2-D q-blocks: exact cover of the plane, tile-aligned cuts where the plane has enough tiles (c3: 512^2 on 8
    ranks = one 256 x 128 pair tile each)."""
    for n in (64, 96, 256, 512):
        for w in (1, 2, 3, 4, 6, 8):
            cover = np.zeros((n, n), dtype=int)
            for r in range(w):
                (h0, n_h, k0, n_k), _ = xd.qblocks(n, n, -n // 2, -n // 2, r, w)
                cover[h0 + n // 2:h0 + n // 2 + n_h, k0 + n // 2:k0 + n // 2 + n_k] += 1
            assert np.all(cover == 1), (n, w)
    blocks = [xd.qblocks(512, 512, -256, -256, r, 8)[0] for r in range(8)]
    assert all(b[1] == 256 and b[3] == 128 for b in blocks)


def test_shard_properties():
    for n in (0, 1, 7, 148, 1000):
        for w in (1, 2, 3, 8):
            spans = [xd.shard(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1
