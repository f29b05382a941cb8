"""Per-rank device time of the sharded build at G ranks, measured on ONE GPU: one loopback pass
produces every rank's received records, then each rank's step (integrate + count, pack, unpack +
assemble) is repeated alone with CUDA events -- what one GPU of a G-GPU node spends per step,
without the collectives.  Usage: python tools/shard_rank_time.py C4 2 4 8"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1501_04784_b200 import distributed as X  # noqa: E402
from paper_1501_04784_b200.workloads import make_workload  # noqa: E402


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


args = [a for a in sys.argv[1:] if not a.startswith("--rank=")]
only = [int(a.split("=")[1]) for a in sys.argv[1:] if a.startswith("--rank=")]  # time these ranks only
wl = args[0] if args else "C3"
mesh = make_workload(wl)
for world in [int(g) for g in (args[1:] or ["2", "4", "8"])]:
    ops0 = X.CudaOps()
    whole = ops0.upload(mesh.coords, mesh.connectivity, mesh.coefficient)
    _, cost = X.block_cost_histograms(ops0, X._LocalSum(), whole, mesh.n_nodes)
    bounds = X.balanced_bounds(cost, mesh.n_nodes, world)
    del whole
    # one loopback pass: every rank's received words (kept on the host), the count matrix
    recv_host, C = [], None
    ranks = [X.ShardedBuild(mesh, r, world, ops=X.CudaOps(), exchange=X.LoopbackExchange(), bounds=bounds)
             for r in range(world)]
    metas = [rk.phase_local().cpu().numpy() for rk in ranks]
    C = ranks[0].check_meta(np.stack(metas))
    chunk = 4 * C[:, :, 0] + C[:, :, 1]
    sends = []
    for r, rk in enumerate(ranks):
        send = rk.ops.alloc_words(int(chunk[r].sum()))
        offs = np.concatenate([[0], np.cumsum(chunk[r])[:-1]])
        rk.pack(*rk.ops.pointers([send.data_ptr()] * world, offs))
        sends.append((send.cpu(), offs))
    for d in range(world):
        recv_host.append(torch.cat([sends[s][0][int(sends[s][1][d]):int(sends[s][1][d] + chunk[s, d])]
                                    for s in range(world)]))
    xb_recs = int(C[:, :, 0][~np.eye(world, dtype=bool)].sum())
    xb = 8 * int((4 * C[:, :, 0] + C[:, :, 1])[~np.eye(world, dtype=bool)].sum())
    del ranks, sends
    torch.cuda.empty_cache()
    rows = []
    for r in (only or range(world)):
        rk = X.ShardedBuild(mesh, r, world, ops=X.CudaOps(), exchange=X.LoopbackExchange(), bounds=bounds)
        recv = recv_host[r].cuda()
        best = None
        for rep in range(4):
            torch.cuda.synchronize()
            a = ev()
            rk.phase_local()
            b = ev()
            send = rk.ops.alloc_words(int(chunk[r].sum()))
            offs = np.concatenate([[0], np.cumsum(chunk[r])[:-1]])
            c = ev()
            rk.pack(*rk.ops.pointers([send.data_ptr()] * world, offs))
            d = ev()
            rk.phase_assemble(recv, C)
            e = ev()
            torch.cuda.synchronize()
            t = (a.elapsed_time(b), c.elapsed_time(d), d.elapsed_time(e))
            if rep > 0 and (best is None or sum(t) < sum(best)):
                best = t
        rows.append(best)
        del rk, recv, send
        torch.cuda.empty_cache()
    tot = [sum(t) for t in rows]
    ms = max(tot)
    print(f"{wl} G={world}: per-rank device ms max {ms:.2f} (mean {np.mean(tot):.2f}); integrate+count max "
          f"{max(t[0] for t in rows):.2f}, pack max {max(t[1] for t in rows):.2f}, unpack+assemble max "
          f"{max(t[2] for t in rows):.2f}; -> {mesh.n_el / ms / 1e6:.2f} G el/s without collectives; exchange "
          f"{xb / 1e9:.3f} GB ({xb / mesh.n_el:.1f} B/el, {xb_recs / mesh.n_el:.2f} records/el)", flush=True)
    print("   per rank (integrate+count, pack, unpack+assemble) ms:",
          " ".join(f"[{a:.2f} {b:.2f} {c:.2f}]" for a, b, c in rows), flush=True)
    print("   records received per rank:", [int(C[:, d, 0].sum() - C[d, d, 0]) for d in range(world)], flush=True)
