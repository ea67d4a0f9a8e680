"""Velocity sweep / P_T^-1 time and agreement for several sweep settings.

Each setting runs in a child process (the STMHD_* switches are read once per
process).  A setting is a dense-top depth (STMHD_SWEEP_KLEVELS) or a comma list
of NAME=VALUE switches.  Prints per setting: solve_velocity ms, apply_inverse ms,
setup s, and the relative difference of both results to the first setting.

  python tools/klevels_probe.py C3 0 2 3 4 -1
  python tools/klevels_probe.py C3 -1 STMHD_SWEEP_LDGSTS=1 STMHD_SWEEP_WARPS=16,STMHD_CHUNK_MAX=512
"""
import json
import os
import subprocess
import sys

CHILD = r"""
import json, sys, torch, numpy as np
import paper_2309_00768_b200 as p
cfg = sys.argv[1]
d = p.discretize_config(cfg)
st = p.initial_state(d)
g = torch.Generator(device="cuda").manual_seed(0)
st.vec.data += 1e-3 * torch.randn(st.vec.data.shape, dtype=torch.float64, device="cuda", generator=g)
jac = p.assemble_jacobian(st, d)
torch.cuda.synchronize()
import time
t0 = time.perf_counter()
pc = p.SpaceTimePreconditioner(jac, d, st)
v = torch.randn(jac.size, dtype=torch.float64, device="cuda", generator=g)
L = d.layout
vu = v[: d.n_steps * L.n_u].clone()
xu = pc.solve_velocity(vu)
torch.cuda.synchronize()
setup = time.perf_counter() - t0
def tm(fn, r=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(r): fn()
    b.record(); b.synchronize()
    return a.elapsed_time(b) / r
out = torch.empty_like(v)
res = {"setup_s": setup, "sv_ms": tm(lambda: pc.solve_velocity(vu)), "pinv_ms": tm(lambda: pc._into(v, out))}
np.save(sys.argv[2] + "_u.npy", pc.solve_velocity(vu).cpu().numpy())
np.save(sys.argv[2] + "_p.npy", pc.apply_inverse(v).cpu().numpy())
print("RESULT " + json.dumps(res))
"""


def main():
    cfg = sys.argv[1]
    settings = sys.argv[2:] or ["0", "-1"]
    os.makedirs("gpurun_out", exist_ok=True)
    base = None
    import numpy as np

    for s in settings:
        env = dict(os.environ)
        if "=" in s:
            for kv in s.split(","):
                k, v = kv.split("=")
                env[k] = v
        else:
            env["STMHD_SWEEP_KLEVELS"] = s
        env["STMHD_SWEEP_PLAN_INFO"] = "1"
        tag = f"gpurun_out/klev_{cfg}_{abs(hash(s))}"
        r = subprocess.run([sys.executable, "-c", CHILD, cfg, tag], env=env, capture_output=True, text=True)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")]
        if r.returncode or not line:
            print(s, "FAILED", r.stderr[-1500:])
            continue
        res = json.loads(line[0][7:])
        u, pv = np.load(tag + "_u.npy"), np.load(tag + "_p.npy")
        if base is None:
            base = (u, pv)
        res["du"] = float(np.linalg.norm(u - base[0]) / np.linalg.norm(base[0]))
        res["dp"] = float(np.linalg.norm(pv - base[1]) / np.linalg.norm(base[1]))
        plan = [ln for ln in r.stderr.splitlines() if "sweep-plan" in ln]
        print("KLEVELS", s, json.dumps(res), plan[:3], flush=True)
        os.remove(tag + "_u.npy")
        os.remove(tag + "_p.npy")


if __name__ == "__main__":
    main()
