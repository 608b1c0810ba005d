"""Run NCCL with two ranks on ONE GPU (validation only, not a measurement):
each rank gets its own NCCL_HOSTID, so NCCL treats them as separate hosts
(no duplicate-GPU refusal) and talks over its socket transport on loopback.
Exercises the NCCL forms of the N > 1 paths that gloo tests cannot:
CUDA-tensor all_to_all_single / all_gather_into_tensor / broadcast / P2P in
dist.MapExchange (fixed slabs, sync=False), dist.WindowChain, the loop-edge
fetch (dist.register_loop_sharded), the pose-graph gather / broadcast and
dist.retrieval_sharded.

    python tools/nccl_one_gpu.py            # spawns 2 ranks
"""
import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), NCCL_HOSTID=f"ec3r-rank{rank}",
                      NCCL_SOCKET_IFNAME="lo", NCCL_IB_DISABLE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    try:
        from paper_2510_02080_b200 import dist as D
        from paper_2510_02080_b200 import loops, mapping, synth
        out = {"backend": dist.get_backend()}
        # raw collectives on CUDA tensors
        x = torch.arange(4, device="cuda", dtype=torch.int64) + 10 * rank
        y = torch.empty_like(x)
        dist.all_to_all_single(y, x)
        out["a2a"] = y.cpu().tolist()
        # windows + halo + device chain (bench's N > 1 registration step)
        import test_gpu_dist as T
        cfg = synth.SceneConfig()
        sb = synth.make_submaps(T.N_KF, cfg, seed=T.SEED, device="cuda")
        S = len(sb.frame_ids)
        lo, hi = D.shard_window(S, world, rank)
        dm, sms, _ = T._build(range(lo, hi), id0=lo)
        D.register_window(dm, sms)
        out["poses"] = T._poses(sms)
        # loop edge across shards + PGO gather / broadcast
        directory = D.SubmapDirectory(dm)
        loop_sm = None
        kf_a, kf_b = sb.frame_ids[1][2], sb.frame_ids[S - 2][3]
        if rank == world - 1:
            fr = T._loop_frames(sb, kf_a, kf_b)
            dm._next_id = T.LOOP_ID
            loop_sm = dm.add_submap([kf_a, kf_b], torch.stack([f[0] for f in fr]), torch.stack([f[1] for f in fr]),
                                    [f[2] for f in fr])
        edges = D.register_loop_sharded(dm, loop_sm, directory)
        out["loop_edges"] = [(e[0], e[1], int(e[4])) for e in edges]
        res = D.optimize_sharded(dm, [e[:4] for e in dm.edges], lambda nodes, rows: dict(nodes))
        out["pgo_nodes"] = sorted(res)
        # owner-partitioned map, host-sync-free exchange
        local, fo, _ = mapping.fuse_slots(dm.pool, dm.all_slots(), 0.02)
        ex = D.MapExchange(0.02)
        r = ex.run(local, int(fo[0].shape[0]), sync=False)
        ex.verify()
        ex.retune()
        r = ex.run(local, int(fo[0].shape[0]), sync=False)
        ex.verify()
        n = int(r[4].item())
        out["map"] = (r[0][:n].cpu().numpy(), r[3][:n].cpu().numpy())
        # sharded retrieval
        pooled = synth.pooled_embeddings(600, device="cpu").numpy()
        db = loops.RetrievalDB(pooled.shape[1], 256)
        db.append(np.arange(600) * 3 + 7, pooled)
        out["retrieval"] = [a.shape for a in D.retrieval_sharded(db, 5, 15, 0.93, 0.96)]
        torch.cuda.synchronize()
        q.put((rank, out))
    except Exception:
        import traceback
        q.put((rank, RuntimeError(traceback.format_exc())))
    finally:
        dist.destroy_process_group()


def main():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=900) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            print(f"rank {r} FAILED:\n{v}")
            sys.exit(1)
    assert out[0]["a2a"] == [0, 1, 10, 11] and out[1]["a2a"] == [2, 3, 12, 13]
    keys = np.concatenate([out[r]["map"][0] for r in range(2)])
    assert len(np.unique(keys)) == len(keys)
    print("nccl two ranks on one GPU: ok", {r: dict(backend=out[r]["backend"], loop_edges=out[r]["loop_edges"],
                                                   pgo_nodes=len(out[r]["pgo_nodes"]), voxels=len(out[r]["map"][0]),
                                                   retrieval=out[r]["retrieval"]) for r in range(2)})


if __name__ == "__main__":
    main()
