"""Profiling driver: a few evolves of a BASELINE workload (for ncu / launch lists).

    python tools/profile_evolve.py [brick28|ucc12|ucc32|expect30] [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2208_10978_b200 import statevector as sv  # noqa: E402
from paper_2208_10978_b200 import workloads as W  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "brick28"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    if which == "brick28":
        cfg = W.config2()
    elif which == "ucc12":
        cfg = W.config1()
    elif which == "ucc32":
        cfg = W.config4()
    elif which == "expect30":
        import torch
        h = W.config3_hamiltonian()
        s = sv.StateVector._empty(30)
        view = torch.as_tensor(s, device="cuda")
        view.copy_(torch.randn(view.shape, dtype=torch.float64, device="cuda"))
        view /= torch.linalg.vector_norm(view)
        for _ in range(reps):
            t0 = time.perf_counter()
            re, im, _ = sv.expectation_terms(s, h)
            print(f"expect30 {time.perf_counter() - t0:.3f}s {sv.last_plan_stats()} E={re:.6f}")
        return
    else:
        raise SystemExit(f"unknown workload {which}")
    s0 = sv.init_state(cfg["reference"])
    for _ in range(reps):
        t0 = time.perf_counter()
        psi = sv.evolve(s0, cfg["circuit"])
        psi.synchronize()
        st = sv.last_plan_stats()
        print(f"{which} evolve {time.perf_counter() - t0:.3f}s passes={st['n_passes']} "
              f"rotations={st['n_rotations']}")
        if "hamiltonian" in cfg:
            t0 = time.perf_counter()
            e = sv.expectation(psi, cfg["hamiltonian"])
            print(f"{which} expectation {time.perf_counter() - t0:.3f}s E={e:.12f} "
                  f"sweeps={sv.last_plan_stats()['n_passes']}")
        del psi


if __name__ == "__main__":
    main()
