"""wd_solve time with opt.profile on / off (host loop), per config (dev probe)."""
import json, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2101_08453_b200 as wd, synth
for name in (sys.argv[1] if len(sys.argv) > 1 else "small,medium").split(","):
    p = synth.make(name, device="cuda")
    out = {"config": name}
    for prof in (0, 1):
        ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a, wd.default_options(profile=prof))
        f = wd.wd_rhs(ctx, p.u0)
        ts = []
        for it in range(12):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            torch.cuda.synchronize(); e0.record()
            _, rep = wd.wd_solve(ctx, f, rel_tol=1e-8)
            e1.record(); torch.cuda.synchronize()
            if it >= 2: ts.append(e0.elapsed_time(e1))
        ts.sort()
        out[f"profile{prof}_ms"] = ts[len(ts) // 2]
        out["cycles"] = rep["cycles"]
        ctx.close()
    print(json.dumps(out), flush=True)
