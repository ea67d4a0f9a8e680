"""Per-block error of P_T^{-1} v against a golden case (pipelined vs sequential)."""
import sys
import os
import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import paper_2309_00768_b200 as p
from test_parity_gpu import _disc  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "bl_island4"
g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", name + ".npz"))
d = _disc(p, name)
st = p.SpaceTimeState(p.BlockVector(d.layout, d.n_steps, g["state"]),
                      torch.as_tensor(g["ic_u"], device="cuda"), torch.as_tensor(g["ic_a"], device="cuda"))
jac = p.assemble_jacobian(st, d)
pc = p.SpaceTimePreconditioner(jac, d, st)
out = pc.apply_inverse(g["v"]).cpu().numpy()
ref = g["Pv"]
L, nt = d.layout, d.n_steps
o = L.offsets()
print("nt", nt, "layout", L, "offsets", o)
out = out.reshape(nt, -1)
ref = ref.reshape(nt, -1)
for k in range(nt):
    for b, (lo, hi) in o.items():
        e = np.linalg.norm(out[k, lo:hi] - ref[k, lo:hi]) / max(np.linalg.norm(ref[k, lo:hi]), 1e-300)
        print(f"slab {k} block {b}: relerr {e:.3e}")


def relerr(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


v = g["v"]
print("apply_inverse", relerr(pc.apply_inverse(v).cpu().numpy(), g["Pv"]))
print("apply_forward", relerr(pc.apply_forward(v).cpu().numpy(), g["PFv"]))
print("solve_velocity", relerr(pc.solve_velocity(v[: nt * L.n_u]).cpu().numpy(), g["sv_u"]))
print("solve_wave", relerr(pc.solve_wave(v[: nt * L.n_a]).cpu().numpy(), g["sw_a"]))
print("pressure_schur_inverse", relerr(pc.pressure_schur_inverse(v[: nt * L.n_p]).cpu().numpy(), g["psi_p"]))
print("magnetic_schur_inverse", relerr(pc.magnetic_schur_inverse(v[: nt * L.n_a]).cpu().numpy(), g["msi_a"]))
print("apply_inverse again", relerr(pc.apply_inverse(v).cpu().numpy(), g["Pv"]))
