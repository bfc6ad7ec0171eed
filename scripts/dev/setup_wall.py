"""Wall-clock of wd_assemble / close at Paper-scale next to the device phases (dev probe)."""
import os, sys, time, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
os.environ["WD_SETUP_TIMING"] = "1"
import paper_2101_08453_b200 as wd, synth
p = synth.make("paper", device=torch.device("cuda:0"))
for prof in (0, 1):
    for r in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a, wd.default_options(profile=prof))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        ctx.close()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"profile={prof} run {r}: assemble {1e3*(t1-t0):.2f} ms, close {1e3*(t2-t1):.2f} ms", file=sys.stderr)
