"""Cross-attention of one UNet transformer layer: attention-kernel path (q2
GEMM, tcgen05 attention over the 77 context keys, o2 GEMM) vs the folded path
(score GEMM with per-head softmax epilogue, P x B_PV GEMM), per level, in CUDA
graphs of back-to-back repetitions.   python tools/cross_fold_bench.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from launch_floor import graph_us  # noqa: E402


def main():
    import torch
    from paper_2603_25872_b200 import netops as ops
    from paper_2603_25872_b200.unet import UNet, sd15_config
    dev = torch.device("cuda", 0)
    net = UNet(sd15_config(64), dev, seed=0, max_batch=1)
    for blk in [b for k, b, _ in net.blocks if k == "tx"][:3] + [[b for k, b, _ in net.blocks if k == "tx"][-1]]:
        c = blk["c"]
        L = blk["layers"][0]
        HW = {320: 4096, 640: 1024, 1280: 256}[c]
        M, heads = 2 * HW, net.cfg.n_heads(c)
        d = c // heads
        n1 = torch.randn(M, c, device=dev).bfloat16()
        s = torch.randn(M, c, device=dev)
        q = torch.empty(M, c, device=dev, dtype=torch.bfloat16)
        att = torch.empty(M, c, device=dev, dtype=torch.bfloat16)
        pb = torch.empty(M, heads * 96, device=dev, dtype=torch.bfloat16)

        def old():
            ops.linear(n1, L["q2"], out=q)
            ops.attention_tc(q, L["k_ctx"], L["vt_ctx"], att, 2, heads, HW, 77, d, vt_img=net.ctx_pad)
            ops.linear(att, L["o2"][0], bias=L["o2"][1], residual=s, out=s)

        def new1():
            ops.linear(n1, L["ws"], act="headsoftmax", hs_valid=77, b_img=(HW, heads * 96), out=pb)

        def new2():
            ops.linear(pb, L["wpv"], bias=L["o2"][1], residual=s, out=s, b_img=(HW, c))

        print(f"c={c:5d} HW={HW:5d}: q2 {graph_us(lambda: ops.linear(n1, L['q2'], out=q)):6.2f}  "
              f"attn {graph_us(lambda: ops.attention_tc(q, L['k_ctx'], L['vt_ctx'], att, 2, heads, HW, 77, d, vt_img=net.ctx_pad)):6.2f}  "
              f"o2 {graph_us(lambda: ops.linear(att, L['o2'][0], bias=L['o2'][1], residual=s, out=s)):6.2f}  "
              f"old chain {graph_us(old):6.2f} us | fold: scores+softmax {graph_us(new1):6.2f}  "
              f"P.Bpv {graph_us(new2):6.2f}  chain {graph_us(lambda: (new1(), new2())):6.2f} us")


if __name__ == "__main__":
    main()
