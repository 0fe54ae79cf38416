"""Halo-exchange microbenchmark ("time ncclSend/ncclRecv pairs of 123 KB - 1 MB between
neighbour ranks, grouped, for N = 2/4/8").  Each rank sends its first row to rank-1 and its last row
to rank+1 and receives both neighbours' rows -- the pattern of glassnet_forward_sharded's
exchange phases -- for the row sizes of the c4 row tiles (x16 123 KB, e_l 246 KB, the decoder's
d rows 246-492 KB, z 23 KB) and reports the per-phase time as the max over ranks.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node=N --master-addr 127.0.0.1 tools/halo_bench.py
  (NCCL on GPUs; with --cpu, gloo on host tensors -- the harness logic, not a NVLink number)

Prints one JSON line on rank 0.  Only one GPU is available to this build, so no NVLink number has
been measured with it; tests/test_sharded.py runs the gloo mode at world size 2."""
import argparse
import json
import os
import time

SIZES = {"z": 3840 * 3 * 4 // 2, "x16": 3840 * 16 * 2, "e_l": 3840 * 32 * 2, "d_2rows": 2 * 3840 * 32 * 2,
         "1MB": 1 << 20}


def main():
    import torch
    import torch.distributed as dist
    ap = argparse.ArgumentParser()
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    if a.cpu:
        dist.init_process_group("gloo")
        dev = torch.device("cpu")
    else:
        local = int(os.environ.get("LOCAL_RANK", rank))
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
        dist.init_process_group("nccl", device_id=dev)
    res = {}
    for name, nbytes in SIZES.items():
        # buffer = [halo above][first row][last row][halo below]
        buf = torch.full((4, nbytes), rank % 251, dtype=torch.uint8, device=dev)

        def phase():
            ops = []
            if rank > 0:
                ops += [dist.P2POp(dist.isend, buf[1], rank - 1), dist.P2POp(dist.irecv, buf[0], rank - 1)]
            if rank < world - 1:
                ops += [dist.P2POp(dist.isend, buf[2], rank + 1), dist.P2POp(dist.irecv, buf[3], rank + 1)]
            if ops:
                for r in dist.batch_isend_irecv(ops):
                    r.wait()
        for _ in range(a.warmup):
            phase()
        if not a.cpu:
            torch.cuda.synchronize()
        dist.barrier()
        if a.cpu:
            t0 = time.perf_counter()
            for _ in range(a.iters):
                phase()
            us = (time.perf_counter() - t0) / a.iters * 1e6
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.iters):
                phase()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / a.iters * 1e3
        # correctness: the halo rows hold the neighbours' ids
        ok = (rank == 0 or int(buf[0, 0]) == (rank - 1) % 251) and \
             (rank == world - 1 or int(buf[3, 0]) == (rank + 1) % 251)
        t = torch.tensor([us, 0.0 if ok else 1.0], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name] = {"bytes": nbytes, "us_per_phase_max_over_ranks": float(t[0]), "ok": float(t[1]) == 0.0}
    if rank == 0:
        print(json.dumps({"world": world, "backend": "gloo" if a.cpu else "nccl", "iters": a.iters, "phases": res}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
