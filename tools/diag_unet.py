import sys, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2603_25872_b200.unet import UNet, sd15_config
from ref_nets import unet_ref
torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False
cuda = torch.device("cuda", 0)
for g in (0.0, 1.0, 7.5):
    net = UNet(sd15_config(32), cuda, seed=0, max_batch=1, cfg_scale=g)
    x = torch.randn(4, 32, 32, device=cuda, dtype=torch.float64, generator=torch.Generator(device=cuda).manual_seed(1))
    t = torch.tensor([601.0], device=cuda)
    out = torch.empty(4 * 32 * 32, device=cuda)
    net.forward([x.reshape(-1)], t, 1, outs=[out])
    ref = unet_ref(net, x.float()[None], t)[0]
    rel = ((out.reshape(4, 32, 32) - ref).norm() / ref.norm()).item()
    print("g", g, "rel", rel, "ref norm", ref.norm().item(), "out norm", out.norm().item())
