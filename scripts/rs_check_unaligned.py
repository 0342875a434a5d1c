"""Risk-scan R/Q (tile-local + carries) vs numpy at beta = 0 on a few-strata design."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_16238_b200 as sx
from paper_2310_16238_b200 import _capi
from oracle.oracle_py import Oracle, Ref
from tests import _golden as G

k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ref = Ref()
orc = Oracle()
ds = ref.simulate(1_400_000, 3, 0.02, 0.5, k, 0.3, 7)
h0, a = ref.build_design(ds)
ref.free_design(h0)
dd = sx.upload(G.sorted_design(a, values=False))
assert dd.set_fit_path(0)
lib = _capi.load()
assert lib.scx_risk_prefix(dd.handle) == 0
n = a["n"]
nt = (n + 2047) // 2048 + 1
R = np.zeros(n); Q = np.zeros(n); CR = np.zeros(nt); CQ = np.zeros(nt); lh = np.zeros(nt, np.int32)
P = lambda x: x.ctypes.data_as(C.POINTER(C.c_double))
assert lib.scx_debug_risk_arrays(dd.handle, P(R), P(Q), P(CR), P(CQ), lh.ctypes.data_as(C.POINTER(C.c_int32))) == 0
r = np.arange(n); t = r // 2048
Rf = R + np.where((r - t * 2048) >= lh[t], CR[t], 0.0)
Qf = Q + np.where((r - t * 2048) >= lh[t], CQ[t], 0.0)
w = np.zeros(n); np.add.at(w, a["tie_end"], a["event"].astype(float))
off = a["offsets"]
Rt = np.zeros(n); Qt = np.zeros(n)
for q in range(len(off) - 1):
    s0, s1 = off[q], off[q + 1]
    S0 = np.arange(1, s1 - s0 + 1, dtype=float)
    u = w[s0:s1] / S0; v = w[s0:s1] / S0**2
    Rt[s0:s1] = np.cumsum(u[::-1])[::-1]
    Qt[s0:s1] = np.cumsum(v[::-1])[::-1]
eR = np.abs(Rf - Rt) / np.maximum(np.abs(Rt), 1e-300)
eQ = np.abs(Qf - Qt) / np.maximum(np.abs(Qt), 1e-300)
bad = np.flatnonzero(eR > 1e-10)
print("k", k, "n", n, "max rel R", eR.max(), "Q", eQ.max(), "bad rows", len(bad),
      "first bad", bad[:5], "tile", (bad[:5] // 2048) if len(bad) else None)
if len(bad):
    b = bad[0]
    print("R", Rf[b], "want", Rt[b], "local", R[b], "CR", CR[b // 2048], "lasth", lh[b // 2048])
