"""Native multi-device handle (qsv_dist) on ONE B200 with P loopback shards:
time a brickwork evolve whose light cone needs relayouts, with the in-place
swap kernels (default) and with staged cudaMemcpyPeerAsync (QSV_DIST_P2P=0).
On one device both move bytes through HBM only (a swap kernel: read + write
of both chunks = 4 x 16 B per exchanged amplitude pair-side; the staged path:
3 copies = 6 x), so this measures the HBM cost of the exchange, not NVLink."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2208_10978_b200 import workloads as W
from paper_2208_10978_b200.multidevice import MultiDeviceState

n, P, layers = int(sys.argv[1]) if len(sys.argv) > 1 else 30, 8, 6
circ = W.brickwork(n, layers, seed=5)
for mode in ("1", "0", "1"):
    os.environ["QSV_DIST_P2P"] = mode
    st = MultiDeviceState(n, [0] * P)
    st.set_basis(0)
    st.apply(circ)  # warm-up (plans, JIT)
    torch.cuda.synchronize()
    info0 = st.info()
    t0 = time.perf_counter()
    for _ in range(3):
        st.set_basis(0)
        st.apply(circ)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    info = st.info()
    rel = (info["relayouts"] - info0["relayouts"]) // 3
    print(f"QSV_DIST_P2P={mode}: {n} q, P={P} loopback shards, {layers} layers: {dt * 1e3:.1f} ms per evolve, "
          f"{rel} relayouts per evolve, swap kernels so far {info['swap_launches']}")
    del st
