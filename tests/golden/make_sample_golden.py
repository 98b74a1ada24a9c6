"""Golden shot-sampling estimates from the REFERENCE (vqekit.statevector.sample).

    PYTHONPATH=oracle/_ref python tests/golden/make_sample_golden.py
"""

import os

import numpy as np

from vqekit import pauli as P
from vqekit import statevector as SV

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(99)
    out = {}
    cases = [(6, "X0 Z2 Y5", 4000, 11), (9, "Z1 Z4", 20000, 7), (11, "Y0 X3 X7 Z10", 50000, 123)]
    for k, (n, label, shots, seed) in enumerate(cases):
        a = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
        a /= np.linalg.norm(a)
        s = SV.StateVector(n, a)
        out[f"c{k}_amps"] = a
        out[f"c{k}_label"] = label
        out[f"c{k}_shots"] = shots
        out[f"c{k}_seed"] = seed
        out[f"c{k}_mean"] = SV.sample(s, P.PauliString.from_label(label), shots, seed)
    np.savez(os.path.join(HERE, "sample_golden.npz"), **out)


if __name__ == "__main__":
    main()
