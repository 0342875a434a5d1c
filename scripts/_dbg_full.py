import os, sys, json, ctypes as C
import numpy as np
sys.path.insert(0, os.getcwd())
import paper_2310_16238_b200 as sx
from paper_2310_16238_b200 import _capi
from oracle.oracle_py import Ref
from tests import _golden as G
from tests.golden.make_large_fits import SPECS, reference_design
ref = Ref()
spec = dict(SPECS["c4_p1e4_2cyc"]); spec["p"] = int(sys.argv[1])
h, a = reference_design(ref, spec)
ref.free_design(h)
dd = sx.upload(G.sorted_design(a, values=False))
lib = _capi.load()
assert lib.scx_risk_prefix(dd.handle) == 0
n = a["n"]; nt = (n + 4095) // 4096 * 2
R = np.zeros(n); Q = np.zeros(n); CR = np.zeros(nt); CQ = np.zeros(nt); lh = np.zeros(nt, np.int32)
P = lambda x: x.ctypes.data_as(C.POINTER(C.c_double))
assert lib.scx_debug_risk_arrays(dd.handle, P(R), P(Q), P(CR), P(CQ), lh.ctypes.data_as(C.POINTER(C.c_int32))) == 0
r = np.arange(n); t = r // 2048
Rf = R + np.where((r - t * 2048) >= lh[t], CR[t], 0.0)
Qf = Q + np.where((r - t * 2048) >= lh[t], CQ[t], 0.0)
# reference R, Q at D = 1
w = np.zeros(n); np.add.at(w, a["tie_end"], a["event"].astype(float))
off = a["offsets"]
Rt = np.zeros(n); Qt = np.zeros(n)
for k in range(len(off) - 1):
    s0, s1 = off[k], off[k + 1]
    S0 = np.arange(1, s1 - s0 + 1, dtype=float)
    u = w[s0:s1] / S0; v = w[s0:s1] / S0**2
    Rt[s0:s1] = np.cumsum(u[::-1])[::-1]; Qt[s0:s1] = np.cumsum(v[::-1])[::-1]
eR = np.abs(Rf - Rt) / np.maximum(1e-300, np.abs(Rt)); eQ = np.abs(Qf - Qt) / np.maximum(1e-300, np.abs(Qt))
bad = np.flatnonzero(eR > 1e-9)
print(json.dumps({"p": spec["p"], "maxeR": float(eR.max()), "maxeQ": float(eQ.max()), "nbadR": int(bad.size),
                  "first_bad": bad[:10].tolist(), "tiles_bad": np.unique(t[bad])[:20].tolist(),
                  "n_tiles_bad": int(np.unique(t[bad]).size),
                  "sample": [(int(i), float(R[i]), float(Rf[i]), float(Rt[i]), int(lh[t[i]]), float(CR[t[i]])) for i in bad[:5]]}))
