"""Multi-rank frame sharding on CPU: world_size 2 over gloo, the oracle as the
per-rank backend (the GPU path uses the same code with the CUDA library)."""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]

from paper_2012_10802_b200.shard import frames_for_rank  # noqa: E402


def test_frames_for_rank_partitions():
    for world in (1, 2, 3, 8):
        for scheme in ("round_robin", "block"):
            got = sorted(f for r in range(world) for f in frames_for_rank(64, r, world, scheme))
            assert got == list(range(64))
    assert frames_for_rank(10, 1, 4) == [1, 5, 9]
    assert frames_for_rank(10, 1, 4, "block") == [3, 4, 5]
    with pytest.raises(ValueError):
        frames_for_rank(10, 4, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _make_frame(i):
    from paper_2012_10802_b200.synth import small_scene
    sc = small_scene(72, 112, seed=900 + i, potholes=1, axes=(12.0, 20.0), d_max=20.0)
    return sc.left, sc.right


def _worker(rank, world, port, out_path):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2012_10802_b200.api import Library
    from paper_2012_10802_b200.shard import run_sharded
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = Library(str(ROOT / "oracle" / "_build" / "librpd_oracle.so"))
    cfg = lib.default_config(d_max=31, superpixels=60)
    res, times = run_sharded(lib, _make_frame, cfg, 6, rank, world, n_streams=2)
    if rank == 0:
        import json
        Path(out_path).write_text(json.dumps([[s.frame, s.n_potholes, s.labels_sha1]
                                              for s in res]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_matches_single_process(tmp_path, oracle_lib):
    import json

    from paper_2012_10802_b200.shard import run_sharded
    out = tmp_path / "r0.json"
    mp.spawn(_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    multi = json.loads(out.read_text())
    cfg = oracle_lib.default_config(d_max=31, superpixels=60)
    single, _ = run_sharded(oracle_lib, _make_frame, cfg, 6, 0, 1, n_streams=1)
    assert [m[0] for m in multi] == list(range(6))
    assert multi == [[s.frame, s.n_potholes, s.labels_sha1] for s in single]


def test_bench_gpus2_spawns_sharded_ranks():
    """`bench.py --gpus 2` without a torchrun environment spawns one process
    per rank (gloo + the oracle backend here), shards the config-5 frame
    stream round-robin and reports the whole-job numbers with n_gpus = 2."""
    import json
    import subprocess
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--backend", "oracle",
         "--config", "5", "--steps", "1", "--warmup", "0", "--streams", "2", "--frames", "2",
         "--pool", "2"], capture_output=True, text=True, timeout=600, env=env, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    res = json.loads(line)
    assert res["n_gpus"] == 2
    assert res["frame_ids_per_rank"] == [[0, 2], [1, 3]]  # round-robin shard of cfg5
    assert res["frames_processed"] == 4
    assert "round-robin" in res["config"]["workload"]
