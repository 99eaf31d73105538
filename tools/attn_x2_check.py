import torch, sys
sys.path.insert(0, '.')
from paper_2603_25872_b200 import _lib, netops
dev = torch.device('cuda', 0)
g = torch.Generator(device=dev).manual_seed(0)
for B,H,L,Lk,d in [(2,8,4096,4096,40),(2,16,256,256,72),(1,5,300,333,64),(2,8,1024,77,80),(2,10,4096,4096,64),(1,3,1000,1500,32),(2,2,128,100,64),(1,5,300,2500,64),(3,7,130,2049,40)]:
    q = torch.randn(B*L, H*d, device=dev, generator=g).bfloat16()
    k = torch.randn(B*Lk, H*d, device=dev, generator=g).bfloat16()
    vimg = (Lk+7)//8*8
    vt = torch.randn(H*d, B*vimg, device=dev, generator=g).bfloat16()
    outs = []
    for m in (0, 1, 2):
        _lib.lib().drs_set_attn_split(m)
        o = torch.empty(B*L, H*d, device=dev, dtype=torch.bfloat16)
        netops.attention_tc(q, k, vt, o, B, H, L, Lk, d, vt_img=vimg); torch.cuda.synchronize()
        outs.append(o.float())
    qf = q.float().view(B, L, H, d).transpose(1, 2); kf = k.float().view(B, Lk, H, d).transpose(1, 2)
    vf = vt.float().view(H, d, B, vimg)[..., :Lk].permute(2, 0, 3, 1)
    ref = torch.softmax(qf @ kf.transpose(-1, -2) / d**0.5, -1) @ vf
    ref = ref.transpose(1, 2).reshape(B*L, H*d)
    for m, o in zip((0, 1, 2), outs):
        print(B,H,L,Lk,d,'mode',m,'rel', ((o-ref).norm()/ref.norm()).item(), 'maxdiff vs mode1', (o-outs[0]).abs().max().item())
