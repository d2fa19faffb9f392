"""torchrun worker for tests/test_gpu_multi.py (one process per GPU, NCCL).

Each rank computes its LPT shard of one SortaGrad minibatch through the
C-ABI on its own GPU, then reduces the trainer's {loss, skipped} pair
(trainer.cpp:160-180) three ways: the fused NVLink peer all-reduce
(ds2ctc_loss_sum_allreduce), ds2ctc_loss_sum + an NCCL all_reduce, and the
host rank-ordered fold (dist.reduce_loss_skipped). Rank 0 checks all three
against the fp64 oracle over the whole global batch (the checker) and writes
a JSON verdict. With --lost-peer, rank 1 skips one fused reduce: rank 0's
call must time out (~20 s), write NaN instead of a stale fold, and report the
fault through ds2ctc_reduce_fault.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--lost-peer", action="store_true")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_1512_02595_b200 import ctc, scheduler
    from paper_1512_02595_b200 import dist as ddist
    from paper_1512_02595_b200.dist import PeerLossReducer
    from paper_1512_02595_b200.synth import make_batch, sortagrad_lengths

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    out = {"rank": rank, "world": world}
    try:
        # one global SortaGrad minibatch (epoch 0: sorted by length), 2 infeasible utterances
        T, L = sortagrad_lengths(96, seed=17)
        order = np.argsort(T, kind="stable")
        T, L = T[order].copy(), L[order].copy()
        acts, flat, ll, il = make_batch(29, T, L, seed=99)
        offs = np.concatenate([[0], np.cumsum(ll)])
        for b in (5, 40):  # all-repeat labels one frame short of min_frames = 2L - 1
            flat[offs[b]:offs[b + 1]] = 3
            il[b] = max(0, 2 * int(ll[b]) - 2)
        idx = scheduler.shard_batch(il, ll, 29, world, rank)
        sub = np.sort(idx)
        lab = np.concatenate([flat[offs[b]:offs[b + 1]] for b in sub]) if sub.size else np.zeros(0, np.int32)
        t_loc = int(il[sub].max()) if sub.size else 0
        x = torch.from_numpy(np.ascontiguousarray(acts[:t_loc, sub, :])).to(dev)
        costs, _ = ctc.compute_ctc_loss(x, lab, ll[sub], il[sub], want_grad=False) if sub.size else (
            torch.zeros(1, device=dev), None)
        B = int(sub.size)
        stream = torch.cuda.current_stream(dev).cuda_stream
        pair_peer = torch.zeros(2, dtype=torch.float64, device=dev)
        pair_nccl = torch.zeros(2, dtype=torch.float64, device=dev)
        import ctypes

        from paper_1512_02595_b200 import _lib

        lib = _lib.lib()
        _lib.check(lib.ds2ctc_loss_sum(ctypes.c_void_p(costs.data_ptr()), B, ctypes.c_void_p(pair_nccl.data_ptr()),
                                       ctypes.c_void_p(stream)), "ds2ctc_loss_sum")
        dist.all_reduce(pair_nccl)
        peer = PeerLossReducer(dev)
        assert peer.ok, peer.error
        for _ in range(3):  # a few steps: the two slot banks alternate
            peer.reduce(costs.data_ptr(), B, pair_peer.data_ptr(), stream)
        torch.cuda.synchronize()
        peer.check()
        loc = costs[:max(B, 0)].cpu().numpy().astype(np.float64) if B else np.zeros(0)
        host_loss, host_skipped = ddist.reduce_loss_skipped(*ddist.local_loss_skipped(loc), device=dev)
        out.update(peer=pair_peer.cpu().tolist(), nccl=pair_nccl.cpu().tolist(), host=[host_loss, host_skipped],
                   shard=int(B))
        if args.lost_peer:
            dist.barrier()
            if rank != 1:
                # rank 1 never joins this step: the wait must give up and report
                peer.reduce(costs.data_ptr(), B, pair_peer.data_ptr(), stream)
                torch.cuda.synchronize()
                v = pair_peer.cpu().numpy()
                try:
                    peer.check()
                    out["fault"] = None
                except RuntimeError as exc:
                    out["fault"] = str(exc)
                out["lost_out"] = [float(x) for x in v]
            dist.barrier()
        else:
            peer.close()
            # f4: the parameter-gradient all-reduce over peer memory (ds2ctc_vec_allreduce),
            # an odd length (the dW + db buffer of the English output layer: 29 x 2560 + 29)
            from paper_1512_02595_b200.dist import PeerVecReducer

            n = 29 * 2560 + 29
            vec = PeerVecReducer(n, dev)
            assert vec.ok, vec.error
            gen = torch.Generator(device=dev)
            sums, nccl_sums, folds = [], [], []
            for step in range(3):  # the two exchange banks alternate
                gen.manual_seed(1000 * step + rank)
                v = torch.randn(n, generator=gen, device=dev, dtype=torch.float32)
                mine = v.clone()
                vec.reduce(mine.data_ptr(), stream)
                ref = v.clone()
                dist.all_reduce(ref)
                parts = [torch.empty_like(v) for _ in range(world)]
                dist.all_gather(parts, v)
                fold = torch.zeros_like(v)
                for part in parts:  # rank order, fp32 left to right: the kernel's fold
                    fold += part
                torch.cuda.synchronize()
                sums.append(float(mine.double().sum()))
                nccl_sums.append(float((mine - ref).abs().max()))
                folds.append(bool(torch.equal(mine, fold)))
            vec.check()
            vec.close()
            out.update(vec_sum=sums, vec_vs_nccl=nccl_sums, vec_fold_bitwise=folds)
        if rank == 0:
            import oracle  # the checker (test infrastructure)

            rc, _ = oracle.oracle_batch(acts, flat, ll, il, want_grad=False, nthreads=8)
            skipped = int(np.isposinf(rc).sum())
            loss = float(np.sum(rc[~np.isposinf(rc)]))
            out["oracle"] = [loss, skipped]
        out["ok"] = True
    except Exception as exc:  # noqa: BLE001
        out["ok"] = False
        out["error"] = repr(exc)
    with open(f"{args.out}.rank{rank}.json", "w") as f:
        json.dump(out, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
