"""compute-sanitizer target (diagnostics): small cases covering every device path --
cluster-mode pipelined P_T^-1 (island 4x4), the grid-family pipelined P_T^-1 and
grid-mode single sweeps forced on a small mesh, one FGMRES Newton step, the
shared-memory and global front factorisation, the multi-right-hand-side constant
solves (Nt = 320 slabs), and the C5 operator at 8x8.
  compute-sanitizer --tool memcheck python tools/sanitize_probe.py [case ...]
cases: cluster grid newton multi c5 (default: all)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_00768_b200 as p  # noqa: E402


def pc_case(n, dt, nt, label):
    d = p.discretize(p.baseline_island(1e-2), 2.0 / n, dt, dt * nt)
    st = p.initial_state(d)
    jac = p.assemble_jacobian(st, d)
    pc = p.SpaceTimePreconditioner(jac, d, st)
    v = torch.randn(jac.size, dtype=torch.float64, device="cuda")
    x = pc.apply_inverse(v)
    y = pc.apply_forward(x)
    u = pc.solve_velocity(v[: d.n_steps * d.layout.n_u].clone())
    jv = jac.apply(v)
    torch.cuda.synchronize()
    rt = float(torch.linalg.vector_norm(y - v) / torch.linalg.vector_norm(v))
    print(f"{label}: round trip {rt:.2e}, |u| {float(u.norm()):.3e}, |Jv| {float(jv.norm()):.3e}", flush=True)
    assert rt < 1e-8


def main():
    cases = sys.argv[1:] or ["cluster", "grid", "newton", "multi", "c5"]
    torch.manual_seed(0)
    if "cluster" in cases:
        pc_case(4, 0.1, 3, "cluster")
    if "grid" in cases:
        # the STMHD_* switches are read once per process: run this case alone with
        # STMHD_PC_GRID=1 STMHD_SWEEP_GRID=1 to force the grid-family paths
        pc_case(8, 0.05, 4, "grid" if os.environ.get("STMHD_PC_GRID") == "1" else "grid(unforced)")
    if "newton" in cases:
        d = p.discretize(p.baseline_island(1e-2), 0.5, 0.1, 0.3)
        cfg = p.NewtonConfig(abs_tol=1e-300, rel_tol=None, max_iters=1,
                             gmres=p.GmresConfig(rel_tol=1e-8, abs_tol=1e-300, max_iters=200, restart=50))
        try:
            _, stats = p.solve_all_at_once(d, cfg)
            print("newton:", stats.gmres_iters, flush=True)
        except p.ConvergenceError as e:  # one step only: the error carries the stats
            print("newton: one step", e, flush=True)
    if "multi" in cases:
        pc_case(4, 0.01, 320, "multi-rhs")
    if "c5" in cases:
        from paper_2309_00768_b200 import c5

        op = c5.C5Operator(8, 4, seed=0)
        x = np.random.default_rng(1).standard_normal(op.nt * op.n)
        r = op.apply(op.solve(x)).cpu().numpy()
        print("c5 round trip", float(np.linalg.norm(r - x) / np.linalg.norm(x)), flush=True)


if __name__ == "__main__":
    main()
