"""Reverse-mode gradient timing at config 1 (12q UCC ansatz, 1,872 parameters, 500-term H)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2208_10978_b200 import statevector as sv, workloads as W
cfg = W.config1(seed=0)
param = W.parametric_rotations_circuit(cfg["n_qubits"], cfg["strings"])
s0 = sv.init_state(cfg["reference"])
th = cfg["thetas"]
for k in range(2):
    t0 = time.perf_counter(); g = sv.reverse_gradient(param, th, cfg["hamiltonian"], s0); t1 = time.perf_counter()
    print(f"reverse_gradient {1e3*(t1-t0):.1f} ms, |g|={np.linalg.norm(g):.6f}, n={len(g)}", flush=True)
# parameter-shift check of a few components (exact for exp(-i theta/2 P))
from paper_2208_10978_b200.circuit import bind
def energy(t):
    return sv.expectation(sv.evolve(s0, bind(param, t)), cfg["hamiltonian"])
for k in (0, 100, 1871):
    e = np.zeros_like(th); e[k] = np.pi / 2
    ps = 0.5 * (energy(th + e) - energy(th - e))
    print(f"k={k}: reverse {g[k]:.15f} shift {ps:.15f} diff {abs(g[k]-ps):.2e}")
# phase breakdown of the rotation-adjoint path
import ctypes
from paper_2208_10978_b200 import _lib
from paper_2208_10978_b200.circuit import bind as _bind
prog = sv._rotation_program(param)
x, y, z, rz = prog
for _ in range(2):
    t0 = time.perf_counter(); bound = _bind(param, th); vals = bound.flat()[2]; ang = np.ascontiguousarray(vals[3 * rz])
    t1 = time.perf_counter(); psi = sv.evolve(s0, bound); psi.synchronize()
    t2 = time.perf_counter(); lam = sv.apply_operator(psi, cfg["hamiltonian"]); lam.synchronize()
    t3 = time.perf_counter(); gg = np.zeros(len(rz))
    _lib.check(_lib.lib().qsv_rotation_adjoint(psi.handle, lam.handle, len(rz), _lib.u64ptr(x), _lib.u64ptr(y),
                                               _lib.u64ptr(z), _lib.dptr(ang), _lib.dptr(gg)))
    t4 = time.perf_counter()
    print(f"bind {1e3*(t1-t0):.2f} evolve {1e3*(t2-t1):.2f} apply_h {1e3*(t3-t2):.2f} adjoint {1e3*(t4-t3):.2f} ms")
