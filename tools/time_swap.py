"""Swap-kernel roofline on one B200: qsv_swap_peer between two shards of the
same device (the relayout exchange of distributed.py when both chunks live in
one HBM).  Each swapped amplitude is read and written once on both sides:
4 x 16 B of HBM traffic per amplitude pair-position; reported against the
measured HBM peak (MEASURED_PEAKS.json).  On two GPUs the same kernel moves
half of its bytes over NVLink instead."""
import ctypes, json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2208_10978_b200 import _lib, statevector as sv

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
a, b = sv.StateVector._empty(n), sv.StateVector._empty(n)
for s in (a, b):
    torch.as_tensor(s, device="cuda").normal_()
torch.cuda.synchronize()
L = _lib.lib()
ptr = ctypes.c_void_p(torch.as_tensor(b, device="cuda").data_ptr())
dim = 1 << n
def swap():
    _lib.check(L.qsv_swap_peer(a.handle, 0, ptr, 0, dim))
for _ in range(3):
    swap()
a.synchronize()
t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
# the library runs on its own stream: bracket with device syncs and host timing
# of 20 swaps (each ~ms, so launch overhead is negligible), plus events on the
# library stream via qsv_get_stream
st = ctypes.c_void_p()
_lib.check(L.qsv_get_stream(a.handle, ctypes.byref(st)))
ext = torch.cuda.ExternalStream(st.value)
a.synchronize()
t0.record(ext)
for _ in range(20):
    swap()
t1.record(ext)
t1.synchronize()
ms = t0.elapsed_time(t1) / 20
bytes_moved = 4 * 16 * dim
try:
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
except Exception:
    peak = 6545.9
gbs = bytes_moved / (ms * 1e-3) / 1e9
print(json.dumps({"kernel": "swap_chunks_kernel", "amplitudes": dim, "ms_per_swap": ms,
                  "hbm_bytes_per_swap": bytes_moved, "achieved_gbs": gbs, "peak_gbs": peak,
                  "frac": gbs / peak}))
