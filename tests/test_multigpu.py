"""Multi-GPU strip decomposition.

CPU (no GPU needed): the strip partition (whole tiles, contiguous, balanced),
the 128-byte NCCL unique id, and the rank bookkeeping over a world_size-2 gloo
group: every rank derives the same partition and receives rank 0's id.
GPU (>= 2 devices): tools/mp_check.py under torchrun — identical per-step
counts and fields within 1e-10 of the single-GPU run, all ranks agreeing.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("ny,tile,nranks", [(4096, 32, 8), (1030, 32, 2), (100, 16, 3), (64, 16, 8), (16384, 32, 8)])
def test_strip_partition(ny, tile, nranks):
    from paper_1309_7128_b200 import strip_rows
    rows = [strip_rows(ny, tile, nranks, r) for r in range(nranks)]
    assert rows[0][0] == 0 and rows[-1][1] == ny
    for (a0, a1), (b0, b1) in zip(rows, rows[1:]):
        assert a1 == b0  # contiguous, no overlap
    for a, b in rows:
        assert a % tile == 0  # coarse tiles never straddle ranks
        assert b >= a
    sizes = [-(-(b - a) // tile) for a, b in rows]
    assert max(sizes) - min(sizes) <= 1  # balanced in tiles


def test_strip_rows_rejects_bad_arguments():
    from paper_1309_7128_b200 import strip_rows
    from paper_1309_7128_b200._lib import InvalidArgument
    with pytest.raises(InvalidArgument):
        strip_rows(100, 16, 2, 2)


def test_nccl_unique_id_is_128_bytes():
    from paper_1309_7128_b200 import nccl_unique_id
    a, b = nccl_unique_id(), nccl_unique_id()
    assert len(a) == 128 and len(b) == 128 and a != b


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1309_7128_b200 import nccl_unique_id, strip_rows
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    mine = strip_rows(4096, 32, world, rank)
    allrows = [None] * world
    dist.all_gather_object(allrows, mine)
    q.put((rank, obj[0], allrows))
    dist.destroy_process_group()


def test_gloo_two_ranks_share_id_and_partition():
    import multiprocessing as mp
    import random
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + random.randrange(300)
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    assert out[0][1] == out[1][1] and len(out[0][1]) == 128
    assert out[0][2] == out[1][2] == [(0, 2048), (2048, 4096)]


@pytest.mark.gpu
def test_two_gpu_strips_match_single_gpu():
    import paper_1309_7128_b200 as P
    if P.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    for n, tile, steps in ((512, 16, 3), (1030, 32, 2)):
        r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
                            "--master-addr", "127.0.0.1", "--master-port", "29531",
                            os.path.join(ROOT, "tools", "mp_check.py"), str(n), str(tile), str(steps)],
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
        assert r.stdout.count('"ok": true') == 2


def test_reference_arm_under_torchrun_two_ranks():
    """bench.py's launch contract at N = 2 on CPU (gloo): `--impl reference` under torchrun
    prints exactly one JSON line, from rank 0, with the reference arm's keys; rank 1 exits 0
    without work. The workload is config 1 (lid 256^2), whose per-step counts come from the
    reference's own fixture."""
    import json
    import random
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(29700 + random.randrange(200)),
                        os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--grid", "256",
                        "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 2
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and "lid-driven cavity 256x256" in d["config"]["workload"]
