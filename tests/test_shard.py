"""Multi-rank slice sharding and ordered aggregation.

CPU: the host logic with gloo, world size 2, per-rank partials from the oracle (the checker).
GPU: bench.py's own sharded engine path under torch.distributed.run (2 ranks, gloo, both on
cuda:0), slice shards and amplitude shards, against the single-process fold and the oracle."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from conftest import payload_path


def test_round_count_and_aggregate():
    """test_executor.cpp:101-147 analogs."""
    from paper_2010_14962_b200.shard import aggregate, round_count, shard_range

    assert round_count(16, 5) == 4 and round_count(16, 17) == 1 and round_count(65536, 4096) == 16
    with pytest.raises(ValueError):
        round_count(4, 0)
    parts = [(4, 8, 2 + 0j), (0, 4, 1 + 0j), (12, 16, 4 + 0j), (8, 12, 3 + 0j)]
    assert aggregate(parts, 16) == 10
    assert aggregate(list(reversed(parts)), 16) == aggregate(parts, 16)
    with pytest.raises(RuntimeError, match="gap"):
        aggregate([(0, 4, 1), (8, 16, 2)], 16)
    with pytest.raises(RuntimeError, match="overlap"):
        aggregate([(0, 6, 1), (4, 16, 2)], 16)
    with pytest.raises(RuntimeError, match="gap"):
        aggregate([(0, 8, 1)], 16)
    for world in (1, 2, 3, 8):
        ranges = [shard_range(1000, r, world) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == 1000
        assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, stem, q):
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2010_14962_b200.shard import aggregate, gather_partials, shard_range

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    net = O.OracleNet(O.load_payload(payload_path(stem)), "ket")
    total = net.jobs
    lo, hi = shard_range(total, rank, world)
    part = net.sum_range(lo, hi)
    parts = gather_partials(part, lo, hi)
    q.put((rank, aggregate(parts, total)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_two_ranks_match_single(world, oracle_mod):
    stem = "cfg1_n20_p1_s1_m4"
    net = oracle_mod.OracleNet(oracle_mod.load_payload(payload_path(stem)), "ket")
    single = net.sum_range(0, net.jobs)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, stem, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank folds the same partials in the same order: identical bits
    assert res[0] == res[1]
    assert abs(res[0] - single) <= 1e-15 * abs(single)


def _run_bench_2ranks(tmp_path, extra):
    """bench.py under torch.distributed.run: 2 ranks, gloo, both on cuda:0 (their kernels never
    wait on each other: each rank reduces its own shard; the only exchange is on the host)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, QCUT_DIST_BACKEND="gloo", QCUT_BENCH_DEVICE="0",
               QCUT_BENCH_PARTIALS=str(tmp_path / "part"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-cpu", *extra]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    ranks = [json.load(open(tmp_path / f"part.rank{r}.json")) for r in range(2)]
    return line, ranks


@pytest.mark.gpu
def test_bench_slice_shards_two_ranks(tmp_path):
    """The sharded engine path of bench.py: contiguous ket-slice ranges, batch
    bits capped at the shard, one all-gather of (lo, hi, re, im), ordered fold (aggregate,
    executor.cpp:78-111). The folded amplitude equals, bit for bit, the fold of the same two
    shard sums computed in this process by engines with the same cap, and the oracle's
    amplitude (amplitudes.json) within 1e-10."""
    import json

    from conftest import GOLD, cx
    from paper_2010_14962_b200 import Engine
    from paper_2010_14962_b200.shard import aggregate

    stem = "cfg5_n120_p1_s5_m20_ext_bt"
    line, ranks = _run_bench_2ranks(tmp_path, ["--config", "cfg5bt"])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    total = 2 ** 20
    assert [(r["lo"], r["hi"]) for r in ranks] == [(0, total // 2), (total // 2, total)]
    assert all(r["batch_bits"] == 19 for r in ranks)
    with Engine(payload_path(stem), device=0, mode="ket", max_batch_bits=19) as e:
        mine = [(r["lo"], r["hi"], e.ket_sum(r["lo"], r["hi"])) for r in ranks]
    want_bits = aggregate(mine, total)
    got = complex(*ranks[0]["amplitudes"][0])
    assert got == want_bits and complex(*ranks[1]["amplitudes"][0]) == got
    amp = cx(json.load(open(os.path.join(GOLD, "amplitudes.json")))[stem + ".b0"]["A"])
    assert abs(got - amp) <= 1e-10 * abs(amp)
    assert abs(complex(line["amplitude"]["re"], line["amplitude"]["im"]) - got) == 0


@pytest.mark.gpu
def test_bench_amplitude_shards_two_ranks(tmp_path):
    """Amplitude-parallel mode (weak scaling, no data-path collective): rank r computes
    bitstring r of config 5 over every slice; each equals the oracle's amplitude."""
    import json

    from conftest import GOLD, cx

    stem = "cfg5_n120_p1_s5_m20_ext_bt"
    amps = json.load(open(os.path.join(GOLD, "amplitudes.json")))
    if stem + ".b1" not in amps:
        pytest.skip("bitstring fixtures missing")
    line, ranks = _run_bench_2ranks(tmp_path, ["--config", "cfg5bt", "--shard", "amplitudes"])
    assert line["scaling"] == "weak" and line["config"]["slices_per_step"] == 2 ** 20
    for r, rec in enumerate(ranks):
        assert (rec["lo"], rec["hi"]) == (0, 2 ** 20)
        got = complex(*rec["amplitudes"][0])
        want = cx(amps[f"{stem}.b{r}"]["A"])
        assert abs(got - want) <= 1e-10 * abs(want), (r, got, want)
