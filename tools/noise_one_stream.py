"""K1 on a few long noise streams (C3 / C5 INIT-stream sizes): device time per
launch with both chain resolvers; also the plain command ncu profiles.

    python tools/noise_one_stream.py [--n 16384] [--streams 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--streams", type=int, default=1)
    ap.add_argument("--gen", default="pcg64")
    a = ap.parse_args()
    import torch
    from paper_2603_25872_b200 import _lib
    from paper_2603_25872_b200.rng import _KeyBuffer, entropy_key, fill_streams
    dev = torch.device("cuda", 0)
    kb = _KeyBuffer([entropy_key((0x7A9C, 7, 50 + i, 2)) for i in range(a.streams)], dev)
    out = torch.empty(a.streams, a.n, dtype=torch.float64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    res = {}
    for mode in (0, 1):
        _lib.lib().drs_set_noise_resolve(mode)
        for _ in range(3):
            fill_streams(kb, a.n, out, a.gen, err=err)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fill_streams(kb, a.n, out, a.gen, err=err)
        e1.record()
        e1.synchronize()
        res[mode] = (e0.elapsed_time(e1) * 100.0, out.clone())
    assert torch.equal(res[0][1], res[1][1]) and int(err.item()) == 0
    print(f"{a.gen} {a.streams} stream(s) x {a.n}: serial resolve {res[0][0]:.1f} us, "
          f"parallel resolve {res[1][0]:.1f} us per launch (identical output)")


if __name__ == "__main__":
    main()
