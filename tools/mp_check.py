"""Multi-GPU strip decomposition check (run under torchrun, one rank per GPU):

    python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 \\
        --master-port 29511 tools/mp_check.py [n] [tile] [steps]

Every rank joins one NCCL communicator (unique id from rank 0 through
torch.distributed), advances the same lid-cavity case, and compares its per-step
counts and final fields with a single-GPU run of the same case made on rank 0
before the group starts. Prints one JSON line per rank; exit code 1 on mismatch.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1309_7128_b200 as P  # noqa: E402
from paper_1309_7128_b200.api import CycleConfig, FluidState, RunMetrics, setup_lid_cavity  # noqa: E402


def run(ctx, n, tile, steps):
    case = setup_lid_cavity(n, 1000.0)
    case.dt = 1000.0 / n
    g = case.grid
    solver = P.PressureSolver(g, CycleConfig(tile=tile), ctx)
    st = FluidState(g)
    st.dt, st.nu = case.dt, case.nu
    ds = P.DeviceState(g, ctx, st)
    m = RunMetrics(n * n)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    per, coarse = [], []
    for _ in range(steps):
        t1 = time.perf_counter()
        ds.step(solver, m)
        ctx.synchronize()
        per.append(round(time.perf_counter() - t1, 4))
        coarse.append(round(solver.last_stats()["coarse_ms"] * 1e-3, 4))
    secs = time.perf_counter() - t0
    print("rank", ctx.device, "per-step seconds", per, "coarse seconds", coarse, flush=True)
    out = FluidState(g)
    ds.download(out)
    rows = [(r.fine_sweeps, r.coarse_sweeps, r.restrictions, r.prolongations, int(r.converged)) for r in m.rows]
    return rows, out, secs, solver.last_stats()


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    tile = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    ref = None
    if rank == 0:  # single-GPU reference run of the same case
        ref = run(P.Context(local), n, tile, steps)
    obj = [P.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = P.Context(local)
    ctx.attach_comm(obj[0], rank, world)
    rows, st, secs, stats = run(ctx, n, tile, steps)
    ok = True
    res = {"rank": rank, "world": world, "n": n, "tile": tile, "strip": P.strip_rows(n, tile, world, rank),
           "rows": rows, "seconds": secs, "collectives": stats["collectives"]}
    if rank == 0:
        rrows, rst, rsecs, _ = ref
        res["single_gpu_rows"] = rrows
        res["single_gpu_seconds"] = rsecs
        ok = rows == rrows
        for name, a, b in (("u", st.vel.u_data, rst.vel.u_data), ("v", st.vel.v_data, rst.vel.v_data),
                           ("p", st.p.data, rst.p.data)):
            den = np.linalg.norm(b)
            rel = float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))
            res["rel_l2_" + name] = rel
            ok = ok and rel <= 1e-10
    # every rank must hold the same state
    h = torch.tensor([float(np.sum(st.p.data * np.arange(st.p.data.size) % 1000))], dtype=torch.float64,
                     device="cuda")
    hs = [torch.zeros_like(h) for _ in range(world)]
    dist.all_gather(hs, h)
    res["ranks_agree"] = all(float(x) == float(hs[0]) for x in hs)
    ok = ok and res["ranks_agree"]
    res["ok"] = ok
    print(json.dumps(res), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
