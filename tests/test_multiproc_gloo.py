"""N>1 host logic on CPU with the gloo backend (world_size 2): the batch shard
each rank regenerates from per-sample seeds equals its slice of the unsharded
batch, per-sample results concatenate to the unsharded result (no collective on
the data path), and bench.py's timing reduction is a max over ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import oracle
        import synth

        oracle.set_threads(1)
        n0, nb = bench.shard(world, rank, batch=4)
        s = synth.stn_inputs(nb, 3, 12, 14, cfg=5, n0=n0)
        b = synth.bslice_inputs(nb, 24, 20, 4, 3, 2, cfg=5, n0=n0)
        y = oracle.stn_fwd(s["x"].double().numpy(), s["theta"].double().numpy())
        dgr = oracle.bslice_bwd(*(b[k].double().numpy() for k in ("grid", "guide", "x", "dy")))[0]
        out = [None] * world
        dist.all_gather_object(out, (rank, n0, nb, y, dgr, s["theta"].numpy()))
        t = bench.max_over_ranks(world, [float(rank + 1), 10.0 - rank])
        if rank == 0:
            q.put((out, t))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_shards_equal_unsharded():
    import oracle
    import synth

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out, t = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda o: o[0])
    assert [(o[1], o[2]) for o in out] == [(0, 2), (2, 2)]
    s = synth.stn_inputs(4, 3, 12, 14, cfg=5)
    b = synth.bslice_inputs(4, 24, 20, 4, 3, 2, cfg=5)
    np.testing.assert_array_equal(np.concatenate([o[5] for o in out]), s["theta"].numpy())
    y = oracle.stn_fwd(s["x"].double().numpy(), s["theta"].double().numpy())
    dgr = oracle.bslice_bwd(*(b[k].double().numpy() for k in ("grid", "guide", "x", "dy")))[0]
    np.testing.assert_array_equal(np.concatenate([o[3] for o in out]), y)
    np.testing.assert_array_equal(np.concatenate([o[4] for o in out]), dgr)
    assert t == [2.0, 10.0]


def test_shard_arithmetic():
    import bench

    assert [bench.shard(8, r) for r in range(8)] == [(8 * r, 8) for r in range(8)]
    with pytest.raises(AssertionError):
        bench.shard(3, 0)


@pytest.mark.timeout(300)
def test_bench_main_two_ranks_gloo():
    """bench.py's own rank loop at world size 2 on CPU: `--gpus 2` without torchrun
    re-execs itself under torch.distributed.run (127.0.0.1), each rank takes its
    contiguous shard, the per-step timings are reduced as a max over ranks (median over
    steps) and rank 0 alone prints ONE JSON line (--dry-run: gloo, stand-in calls)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--dry-run", "--gpus", "2",
                          "--steps", "3", "--warmup", "3"], capture_output=True, text=True, env=env,
                         timeout=240, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["dry_run"] is True
    assert d["per_rank_shards"] == [[0, 32], [32, 32]]
    assert d["config"]["per_rank_batch"] == 32
    assert d["ms_per_step"] > 0 and d["timing"]["total_ms_k_steps_max_over_ranks"] >= d["ms_per_step"]


def test_bench_rejects_world_mismatch():
    """Under torchrun, --gpus must equal WORLD_SIZE (a silent 1-GPU run is refused)."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--dry-run", "--gpus", "2"],
                         capture_output=True, text=True, env=env, timeout=120, cwd=root)
    assert out.returncode != 0 and "WORLD_SIZE" in (out.stderr + out.stdout)
