"""Debug: where do the TV-GD kernel variants (paired / single / tiled) differ."""
import os, subprocess, sys, tempfile
import torch
root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
code = (
    "import torch,sys;sys.path.insert(0,'.');"
    "from paper_1905_03748_b200 import kernels as K;"
    "gen=torch.Generator(device='cuda').manual_seed(3);"
    "u=torch.rand((45,38,70),device='cuda',generator=gen);"
    "g=torch.empty_like(u);s=torch.zeros(1,dtype=torch.float64,"
    "device='cuda');K.tv_grad_store(u,g,(4,40),s);"
    "torch.save((u.cpu(),g.cpu(),s.cpu()),sys.argv[1])")
outs = {}
with tempfile.TemporaryDirectory() as td:
    for tag, env_add in (("pairs", {}), ("single", {"CS_TV_PAIRS": "0"}),
                         ("tiled", {"CS_TV_TILED": "1"})):
        f = os.path.join(td, f"{tag}.pt")
        subprocess.run([sys.executable, "-c", code, f], cwd=root,
                       env=dict(os.environ, **env_add), check=True)
        outs[tag] = torch.load(f)
u = outs["pairs"][0]
for a, b in (("pairs", "single"), ("pairs", "tiled"), ("single", "tiled")):
    ga, gb = outs[a][1], outs[b][1]
    d = (ga != gb)
    print(a, b, "ndiff", int(d.sum()), "maxabs", float((ga - gb).abs().max()))
    idx = d.nonzero()[:10].tolist()
    for z, y, x in idx:
        print("   ", (z, y, x), float(ga[z, y, x]), float(gb[z, y, x]))
