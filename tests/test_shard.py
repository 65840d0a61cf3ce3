"""Multi-rank slice sharding and ordered aggregation, on CPU with gloo.

The per-rank partial is computed by the oracle here (the checker); on GPUs the same
host logic runs with Engine.ket_sum and NCCL (bench.py)."""
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
