import sys, os, json, torch
import paper_2309_00768_b200 as p
cfg = sys.argv[1]; leaf = int(sys.argv[2])
d = p.discretize_config(cfg, leaf={"fu": leaf})
st = p.initial_state(d)
g = torch.Generator(device="cuda").manual_seed(0)
st.vec.data += 1e-3 * torch.randn(st.vec.data.shape, dtype=torch.float64, device="cuda", generator=g)
jac = p.assemble_jacobian(st, d)
pc = p.SpaceTimePreconditioner(jac, d, st)
v = torch.randn(jac.size, dtype=torch.float64, device="cuda", generator=g)
out = torch.empty_like(v)
def tm(fn, r=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(r): fn()
    b.record(); b.synchronize()
    return a.elapsed_time(b) / r
t = tm(lambda: pc._into(v, out))
back = pc.apply_forward(out)
rt = float(torch.linalg.vector_norm(back - v) / torch.linalg.vector_norm(v))
print(f"leaf {leaf} mask {os.environ.get('STMHD_ND_MERGE_MASK','default')}: pinv {t:.3f} ms round trip {rt:.2e}")
