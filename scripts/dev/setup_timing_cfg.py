"""Setup phases (WD_SETUP_TIMING) for a config (dev probe): python setup_timing_cfg.py small"""
import os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
os.environ["WD_SETUP_TIMING"] = "1"
import paper_2101_08453_b200 as wd, synth
p = synth.make(sys.argv[1] if len(sys.argv) > 1 else "small", device=torch.device("cuda:0"))
for r in range(3):
    print("--- run", r, file=sys.stderr)
    ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a)
    ctx.close()
