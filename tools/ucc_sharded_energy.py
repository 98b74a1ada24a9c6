"""Config-4 UCC energy on P GPUs (one process per GPU, NCCL):

    python -m torch.distributed.run --nnodes=1 --nproc-per-node P --master-addr 127.0.0.1 \\
        --master-port 29510 tools/ucc_sharded_energy.py [--qubits 32] [--evals 2]

The state is sharded on the top log2(P) qubits (distributed.py); rotations whose
flip avoids the global qubits run locally, the rest after light-cone-scheduled
relayouts.  Rank 0 prints one JSON line: energy evals/s (whole job), the
energy, relayout counts/bytes.  Not part of bench.py's contract line.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist

    from paper_2208_10978_b200 import distributed as D
    from paper_2208_10978_b200 import workloads as W

    ap = argparse.ArgumentParser()
    ap.add_argument("--qubits", type=int, default=32)
    ap.add_argument("--evals", type=int, default=2)
    ap.add_argument("--backend", default="nccl")
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.backend != "nccl":
        local %= max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist.init_process_group(a.backend)
    try:
        n = a.qubits
        cfg = W.config4(seed=0, n_qubits=n, n_electrons=n // 2)
        be = D.DistributedBackend(D.ProcessGroupComm(), D.CudaEngine(local))
        s0 = be.prepare(cfg["reference"])
        e = be.expectation(be.evolve(s0, cfg["circuit"]), cfg["hamiltonian"])  # plan + specialise
        dist.barrier()
        t0 = time.perf_counter()
        rel = sent = 0
        for _ in range(a.evals):
            psi = be.evolve(s0, cfg["circuit"])
            e = be.expectation(psi, cfg["hamiltonian"])
            rel += psi.stats["relayouts"]
            sent += psi.stats["relayout_bytes_sent"]
            del psi
        dt = (time.perf_counter() - t0) / a.evals
        t = torch.tensor([dt], dtype=torch.float64, device="cuda" if a.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if dist.get_rank() == 0:
            print(json.dumps({"metric": "UCC energy evals/s", "value": 1.0 / float(t.item()),
                              "n_gpus": dist.get_world_size(), "n_qubits": n, "energy": e,
                              "relayouts_per_eval": rel / a.evals,
                              "relayout_bytes_sent_per_gpu_per_eval": sent / a.evals}), flush=True)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
