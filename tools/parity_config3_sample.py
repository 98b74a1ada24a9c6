"""Full-size parity of config 3 (30 qubits, 10,000 strings) on a stratified
sample of strings: the B200 evaluates all 10,000 per-string <P_t> in the
plan config 3 uses (specialised sweeps, wide-group and Z-only transform
sweeps); the C oracle (one core) recomputes a sample of them on the same
state -- every wide group, Z-only strings and narrow strings."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import oracle as O
from paper_2208_10978_b200 import statevector as sv, workloads as W
from paper_2208_10978_b200.pauli import PauliSum, term_arrays

n = 30
h = W.config3_hamiltonian(seed=0)
t0 = time.perf_counter()
st = W.config3_state(seed=0)
print(f"state {time.perf_counter() - t0:.0f} s", flush=True)
s = sv.from_amplitudes(st)
re, im, per = sv.expectation_terms(s, h)
del s
x, y, z, cr, ci = term_arrays(h, n)
f = x | y
rng = np.random.default_rng(1)
cnt = {}
for i, v in enumerate(f):
    cnt.setdefault(int(v), []).append(i)
wide = [g[0] for k, g in cnt.items() if k and len(g) > 24]   # one string of every wide group
zonly = list(rng.choice(cnt[0], 16, replace=False))
narrow = list(rng.choice([i for k, g in cnt.items() if k and len(g) <= 24 for i in g], 32, replace=False))
idx = sorted(set(int(i) for i in wide + zonly + narrow))
sub = PauliSum(tuple(h.terms[i] for i in idx))
t1 = time.perf_counter()
_, pt = O.expectation(st, sub, n, per_term=True)
print(f"oracle {len(idx)} strings: {time.perf_counter() - t1:.0f} s")
d = np.abs(per[idx] - pt[:, 0])
print(f"config3 30q, {len(idx)} sampled strings ({len(wide)} wide-group, {len(zonly)} Z-only, "
      f"{len(narrow)} narrow): max |d<P>| = {d.max():.3e}; full energy (B200) = {re:.15f}")
assert d.max() <= 1e-12
print("PASS")
