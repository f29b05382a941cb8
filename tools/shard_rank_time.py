"""Per-rank device time of the sharded build at G ranks, measured on ONE GPU through the loopback
driver (each rank's phases timed alone with CUDA events): what one GPU of a G-GPU node spends per
step, without the collectives.  Usage: python tools/shard_rank_time.py C4 2 4 8"""
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


wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
mesh = make_workload(wl)
for world in [int(g) for g in (sys.argv[2:] or ["2", "4", "8"])]:
    ops0 = X.CudaOps()
    whole = ops0.upload(mesh.coords, mesh.connectivity, mesh.coefficient)
    hist = ops0.column_weights(whole, mesh.n_nodes, X.histogram_bins(mesh.n_nodes))
    bounds = X.balanced_bounds(hist.cpu().numpy(), mesh.n_nodes, world)
    del whole, hist
    ranks = [X.ShardedBuild(mesh, r, world, ops=X.CudaOps(), exchange=X.LoopbackExchange(), bounds=bounds)
             for r in range(world)]
    best = None
    for rep in range(3):
        t_local, metas = [], []
        for rk in ranks:
            a = ev()
            m = rk.phase_local()
            b = ev()
            torch.cuda.synchronize()
            t_local.append(a.elapsed_time(b))
            metas.append(m.cpu().numpy())
        C = ranks[0].check_meta(np.stack(metas))
        chunk = 4 * C[:, :, 0] + C[:, :, 1]
        sends, t_pack = [], []
        for r, rk in enumerate(ranks):
            send = rk.ops.alloc_words(int(chunk[r].sum()))
            offs = np.concatenate([[0], np.cumsum(chunk[r])[:-1]])
            a = ev()
            rk.pack(*rk.ops.pointers([send.data_ptr()] * world, offs))
            b = ev()
            torch.cuda.synchronize()
            t_pack.append(a.elapsed_time(b))
            sends.append((send, offs))
        recvs = []
        for d in range(world):
            parts = [sends[s][0][int(sends[s][1][d]):int(sends[s][1][d] + chunk[s, d])] for s in range(world)]
            recvs.append(torch.cat(parts))
        del sends
        t_asm = []
        for r, rk in enumerate(ranks):
            a = ev()
            rk.phase_assemble(recvs[r], C)
            b = ev()
            torch.cuda.synchronize()
            t_asm.append(a.elapsed_time(b))
        del recvs
        per_rank = [t_local[r] + t_pack[r] + t_asm[r] for r in range(world)]
        if best is None or max(per_rank) < max(best[0]):
            best = (per_rank, t_local, t_pack, t_asm)
    per_rank, t_local, t_pack, t_asm = best
    xb = ranks[0].exchange_bytes()
    ms = max(per_rank)
    print(f"{wl} G={world}: per-rank device ms max {ms:.2f} (mean {np.mean(per_rank):.2f}); "
          f"integrate+count max {max(t_local):.2f}, pack max {max(t_pack):.2f}, unpack+assemble max {max(t_asm):.2f}; "
          f"-> {mesh.n_el / ms / 1e6:.2f} G el/s without collectives; exchange {xb['bytes'] / 1e9:.3f} GB "
          f"({xb['bytes_per_element']:.1f} B/el)", flush=True)
    del ranks
    torch.cuda.empty_cache()
