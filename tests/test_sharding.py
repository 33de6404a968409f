"""Multi-process (gloo, world size 2, CPU) test of the segment sharding + ordered host gather that the N > 1
path uses. The enhancement function is a stand-in (no GPU here); the sharding logic is what is under test."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2212_05271_b200 import sharding


class _Audio:
    def __init__(self, m, n):
        self.m, self.n = m, n

    def num_channels(self):
        return self.m


class _Act:
    def __init__(self, t, k):
        self.frames, self.k = t, k

    def num_classes(self):
        return self.k


class _Seg:
    def __init__(self, i, m, t, k):
        self.index, self.audio, self.activity = i, _Audio(m, t * 128), _Act(t, k)


class _Wpe:
    taps, iterations = 10, 3


class _Cfg:
    bss_iterations, enable_wpe, wpe = 20, True, _Wpe()


def _segments():
    rng = np.random.RandomState(0)
    return [_Seg(i, int(rng.randint(2, 9)), int(rng.randint(500, 7000)), int(rng.randint(2, 6))) for i in range(23)]


def test_shard_is_balanced_and_deterministic():
    segs = _segments()
    costs = [sharding.segment_cost(s.activity.frames, s.audio.m, s.activity.k, 20, 10, 3) for s in segs]
    for world in (1, 2, 4, 8):
        owned = sharding.shard(costs, world)
        assert sorted(i for o in owned for i in o) == list(range(len(segs)))
        assert owned == sharding.shard(costs, world)
        loads = [sum(costs[i] for i in o) for o in owned]
        assert max(loads) <= sum(costs) / world + max(costs)  # LPT bound


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    segs = _segments()
    calls = []

    def fake_enhance(batch, cfg):
        calls.append([s.index for s in batch])
        return [("enhanced", s.index, rank) for s in batch]

    out = sharding.enhance_sharded(segs, _Cfg(), fake_enhance, rank, world)
    q.put((rank, out, calls))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_gather_is_ordered():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict()
    for _ in range(2):
        rank, out, calls = q.get(timeout=120)
        got[rank] = (out, calls)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out0, calls0 = got[0]
    out1, calls1 = got[1]
    assert out1 is None
    assert [o[1] for o in out0] == list(range(23))          # plan order restored on rank 0
    owners = {o[1]: o[2] for o in out0}
    assert sorted(calls0[0] + calls1[0]) == list(range(23))  # every segment enhanced exactly once
    assert all(owners[i] == 0 for i in calls0[0]) and all(owners[i] == 1 for i in calls1[0])


def test_sweep_sample_partition_covers_every_segment_once_and_balances():
    """The strong-scaling entry of bench.py's `configs` block: a sample of the 4096-segment sweep (BASELINE configs[4])
    split over N ranks with sharding.shard on the SURVEY 8e cost model. Every rank draws the same parameter list, so
    the shards are disjoint, cover the sample, and their modelled loads stay within a few percent of each other."""
    import synthbench as synth
    params = synth.sweep_params(4096)
    assert len(params) == 4096 and params == synth.sweep_params(4096)          # same list on every rank
    assert {p[1] for p in params} == set(range(2, 9)) and {p[4] for p in params} == {5, 10, 20, 40}
    assert all(2 <= p[2] <= 4 and 2.0 <= p[3] <= 12.0 for p in params)
    sample = params[::16][:256]
    costs = [sharding.segment_cost(synth.sweep_frames(p[3]), p[1], p[2] + 1, p[4], 10, 3) for p in sample]
    for world in (1, 2, 4, 8):
        owned = sharding.shard(costs, world)
        assert sorted(i for o in owned for i in o) == list(range(256))
        loads = [sum(costs[i] for i in o) for o in owned]
        assert sum(loads) / (world * max(loads)) > 0.97, (world, loads)


def test_bench_relaunches_itself_as_n_ranks(monkeypatch):
    """`python bench.py --gpus N` without a torchrun environment must become N ranks (one per GPU); under torchrun
    (WORLD_SIZE set) it must not fork again."""
    import importlib.util
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("gss_bench", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    seen = {}

    def fake_call(cmd):
        seen["cmd"] = cmd
        return 0

    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2", "--headline-only"])
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert e.value.code == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node" in cmd
    assert cmd[cmd.index("--nproc-per-node") + 1] == "4" and cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-5:] == ["--gpus", "4", "--steps", "2", "--headline-only"] and cmd[-6].endswith("bench.py")


def test_reference_arm_prints_one_json_line_on_cpu():
    """`bench.py --impl reference` (the CPU arm the driver runs beside ours) on the tiny workload: one JSON line with
    the contract's keys, the same `config` dict our arm prints for that workload, and no GPU involved."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--workload", "tiny",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "audio-s/s" and d["higher_is_better"] is True
    assert d["gpu_launches"] == 0 and d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["name"] == "tiny" and d["config"]["segments_per_gpu"] == 2


def _agg_worker(rank, world, port, q):
    """One rank of the bench's aggregation: its own timings in, whole-job numbers out (gloo on CPU)."""
    import importlib.util
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("gss_bench", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)

    class Part:
        def __init__(self, b, e):
            self.sample_begin, self.sample_end = b, e

    class Audio:
        def num_samples(self):
            return 640000

    class Seg:
        def __init__(self):
            self.parts, self.audio = [Part(240000, 400000)], Audio()   # 10 s cut out of a 40 s window

    b = bench.Bench.__new__(bench.Bench)   # no device, no library: only the reduction logic is under test
    b.torch, b.dist, b.rank, b.world, b.device = torch, dist, rank, world, "cpu"
    nseg = 4 if rank == 0 else 2           # uneven shards, as the size-balanced partition of the sweep produces
    calls = [(None, [Seg() for _ in range(nseg)])]
    r = {"ms": 100.0 if rank == 0 else 80.0, "e2e_ms": 120.0 if rank == 0 else 90.0, "h2d": 1000 * nseg, "d2h": 10 * nseg,
         "launches": 7}
    q.put((rank, bench.summarise(b, calls, r, steps=2, scaling="strong")))
    dist.barrier()
    dist.destroy_process_group()


def test_bench_aggregates_ranks_as_sum_of_work_over_slowest_rank():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_agg_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=180) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in (0, 1):
        d = got[rank]
        assert d["segments"] == 6 and d["scaling"] == "strong"
        assert d["ms_per_step"] == 50.0                                 # slowest rank: 100 ms over 2 steps
        assert d["value"] == pytest.approx(6 * 10.0 * 2 / 0.100)        # 60 s of output per step, both ranks' work
        assert d["xrt_processed"] == pytest.approx(6 * 40.0 * 2 / 0.100)
        assert d["e2e"]["value"] == pytest.approx(6 * 10.0 * 2 / 0.120) and d["e2e"]["ms_per_step"] == 60.0
        assert d["e2e"]["h2d_bytes_per_step"] == 6000 and d["e2e"]["d2h_bytes_per_step"] == 60
        assert d["gpu_launches"] == 14 and d["per_rank_ms_per_step"] == [50.0, 40.0]
