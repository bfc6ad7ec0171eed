import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2101_08453_b200 as wd, synth
cfg, lev = sys.argv[1], int(sys.argv[2])
p = synth.make(cfg, device="cuda") if cfg in synth.CONFIGS else synth.box(int(cfg), int(cfg), 4).to("cuda")
ctx = wd.wd_assemble(p.X, p.Y, p.Z, p.a)
print("levels", [ctx.level_dims(l) for l in range(ctx.num_levels())], flush=True)
x = torch.rand(ctx.level_shape(lev), dtype=torch.float64, device="cuda")
y = wd.wd_apply(ctx, lev, x)
torch.cuda.synchronize()
print("ok", cfg, lev, float(y.abs().max()), flush=True)
