"""Host logic of bench.py: the max-over-ranks timing reduction across 2 gloo ranks (the N > 1 path's
only collective; the units themselves are independent per rank), the aggregate value, and the
reference arm's JSON line on a small config."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = [10.0 + 5.0 * rank, 7.0 - rank]          # this rank's (step time, e2e time) in ms
    got = bench.max_over_ranks(mine, world)
    out[rank] = (got, bench.aggregate_value(1000, got[0], world))
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    world, port = 2, _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        got, val = out[r]
        assert got == [15.0, 7.0]                     # max over ranks, both keys
        assert val == pytest.approx(1000 * 2 / 15e-3)  # whole-job units / slowest rank's time


def test_single_rank_passthrough():
    import bench
    assert bench.max_over_ranks([3.0, 4.0], 1) == [3.0, 4.0]


def test_reference_arm_json_line():
    """`bench.py --impl reference` prints one JSON line with the contract's keys (oracle on the host)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling", "dtype",
              "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_config_keys_identical_in_both_arms():
    """Both arms describe the workload with the same `config` (the driver compares them)."""
    import bench
    for cfg in (1, 2, 3, 4, 5):
        c = bench.workload_config(cfg)
        assert c["workload"] == bench.CONFIG_NAMES[cfg]
        assert "leaves_at_start" not in c  # a per-run measurement, not a workload key
        assert c == bench.workload_config(cfg)


def _run_bench(args, env_extra):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                          text=True, timeout=300, cwd=ROOT, env=env)


def test_gpus_flag_must_match_world_size():
    """--gpus N is authoritative: a launcher with another WORLD_SIZE is an error, not a silent 1-rank run."""
    r = _run_bench(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "0", "--gpus", "1"],
                   {"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stderr + r.stdout)


def test_reference_arm_nonzero_rank_exits_quietly():
    r = _run_bench(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "0", "--gpus", "2"],
                   {"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert r.returncode == 0 and not r.stdout.strip()
