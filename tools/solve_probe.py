"""Wall time of full C4_512 Newton solves with the per-phase timings (diagnostics):
  STMHD_...=... python tools/solve_probe.py <label>"""
import sys, time, torch
import paper_2309_00768_b200 as p
d = p.discretize_config("C4_512")
cfg = p.NewtonConfig(abs_tol=1e-300, rel_tol=1e-6, max_iters=25, gmres=p.GmresConfig(rel_tol=1e-8, abs_tol=1e-300, max_iters=100000, restart=50))
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    st, stats = p.solve_all_at_once(d, cfg)
    torch.cuda.synchronize()
    print(sys.argv[1], "solve %.3f s" % (time.perf_counter() - t), stats.gmres_iters, {k: round(v, 3) for k, v in stats.timings.items()}, flush=True)
