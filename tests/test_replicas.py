"""The N>1 path of bench.py on CPU: world_size-2 gloo process group.

One cfg3 scene does not shard, so N GPUs run N independent
replicas. The host logic this covers:
  * the slowest rank's time is what gets reported (max over ranks);
  * whole-job throughput = N / that time;
  * the reference arm runs on rank 0 only, and other ranks exit without work;
  * replicas don't interact: each rank's solve equals a single-process solve
    of the same scene (here with the oracle, since there is no GPU).
"""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _solve_bar(depth):
    from oracle import oracle as O
    from scenes import make_bar, oracle_scene, oracle_state, oracle_system

    model, system, state, part = make_bar(press_depth=depth)
    osys = oracle_system(model, system)
    st = oracle_state(state)
    O.solve_frame_schur(oracle_scene(model), osys, st, 1, 2, "inner")
    return st.x


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, str(ROOT / "tests"))
    import bench

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        local_ms = [4.0, 5.5][rank]
        dist.barrier()
        worst = bench.max_over_ranks(dist, local_ms)
        value = bench.replica_throughput(world, worst)
        x = _solve_bar(0.04 + 0.02 * rank)  # an independent scene per rank
        np.savez(Path(out_dir) / f"rank{rank}.npz", worst=worst, value=value, x=x)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_rank_replicas_gloo(tmp_path):
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    r = [np.load(tmp_path / f"rank{k}.npz") for k in range(2)]
    for k in range(2):
        assert float(r[k]["worst"]) == 5.5
        assert float(r[k]["value"]) == pytest.approx(2 * 1e3 / 5.5)
        # no cross-talk between replicas: bit-identical to a solo solve
        assert np.array_equal(r[k]["x"], _solve_bar(0.04 + 0.02 * k))
    assert not np.array_equal(r[0]["x"], r[1]["x"])


def test_reference_arm_runs_on_rank0_only(monkeypatch, capsys):
    import bench

    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")

    class Args:
        config, outer, inner, steps, warmup, gpus, ref_frames, collider = "cfg1", 1, 1, 2, 3, 2, 1, "plane"

    called = []
    monkeypatch.setattr(bench, "build_sim", lambda *a: called.append(a))
    assert bench.run_reference(Args()) is None
    assert called == [] and capsys.readouterr().out == ""


def test_single_process_max_is_identity():
    import bench

    assert bench.max_over_ranks(None, 3.25) == 3.25
    assert bench.replica_throughput(1, 4.0) == 250.0


def test_bench_spawns_one_rank_per_gpu():
    """`python bench.py --gpus 2` (no WORLD_SIZE) re-launches itself under
    torchrun with one process per GPU; each rank's scenes go to its own
    device (LOCAL_RANK -> _native.default_device)."""
    import json
    import subprocess
    import sys

    root = Path(__file__).resolve().parent.parent
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "SPB_DEVICE")}
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--probe-ranks"], cwd=root,
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["world"] == 2
    assert sorted(x["rank"] for x in line["ranks"]) == [0, 1]
    assert sorted(x["device"] for x in line["ranks"]) == [0, 1]


def test_spawn_command_layout():
    import bench

    cmd = bench.spawn_cmd(4, ["--gpus", "4", "--steps", "5"], 29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "5"]
