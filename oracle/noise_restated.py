"""ORACLE -- test infrastructure only.

Pure-Python restatement of the reference's noise stream (rng.py:27-33 ->
numpy SeedSequence -> PCG64 / SFC64 -> random_standard_normal ziggurat), for
small cases: it reproduces numpy bit-for-bit (tests/test_oracle_pinned.py)
and additionally reports which ziggurat path every draw took, so the golden
keys can be chosen to exercise the wedge and tail paths the device kernel
must get right.  Tables are read from the installed numpy's libnpyrandom.a
(the same bytes numpy executes); log1p/exp are the host libm's, as numpy's.
"""

import math
import os
import sys

M32, M64, M128 = (1 << 32) - 1, (1 << 64) - 1, (1 << 128) - 1
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645


def _tables():
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.join(here, "..", "tools"))
    try:
        import gen_tables
    finally:
        sys.path.pop(0)
    z = gen_tables.ziggurat_tables()
    return z["ki_double"], z["wi_double"], z["fi_double"]


KI, WI, FI = _tables()


def entropy_words(vals):
    """numpy _coerce_to_uint32_array of a tuple of non-negative ints."""
    out = []
    for v in vals:
        v = int(v)
        if v == 0:
            out.append(0)
        while v:
            out.append(v & M32)
            v >>= 32
    return out


def seedseq_state(ent, n_words):
    """numpy SeedSequence(ent).generate_state(n_words, uint32)."""
    hc = [0x43B0D7E5]

    def hashmix(v):
        v ^= hc[0]
        hc[0] = (hc[0] * 0x931E8875) & M32
        v = (v * hc[0]) & M32
        return v ^ (v >> 16)

    def mix(x, y):
        r = (0xCA01F9DD * x - 0x4973F715 * y) & M32
        return r ^ (r >> 16)

    pool = [hashmix(ent[i] if i < len(ent) else 0) for i in range(4)]
    for s in range(4):
        for d in range(4):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(4, len(ent)):
        for d in range(4):
            pool[d] = mix(pool[d], hashmix(ent[s]))
    hb, out = 0x8B51F9DD, []
    for i in range(n_words):
        v = pool[i % 4] ^ hb
        hb = (hb * 0x58F38DED) & M32
        v = (v * hb) & M32
        out.append(v ^ (v >> 16))
    return out


def _u64s(words):
    return [words[2 * i] | (words[2 * i + 1] << 32) for i in range(len(words) // 2)]


class PCG64:
    def __init__(self, ent):
        v = _u64s(seedseq_state(ent, 8))
        initstate, initseq = (v[0] << 64) | v[1], (v[2] << 64) | v[3]
        self.inc = ((initseq << 1) | 1) & M128
        self.state = 0
        self.state = (self.state * PCG_MULT + self.inc) & M128
        self.state = (self.state + initstate) & M128
        self.state = (self.state * PCG_MULT + self.inc) & M128

    def next64(self):
        self.state = (self.state * PCG_MULT + self.inc) & M128
        x = ((self.state >> 64) ^ self.state) & M64
        rot = self.state >> 122
        return ((x >> rot) | (x << ((64 - rot) & 63))) & M64


class SFC64:
    def __init__(self, ent):
        v = _u64s(seedseq_state(ent, 6))
        self.a, self.b, self.c, self.w = v[0], v[1], v[2], 1
        for _ in range(12):
            self.next64()

    def next64(self):
        tmp = (self.a + self.b + self.w) & M64
        self.w += 1
        self.a = self.b ^ (self.b >> 11)
        self.b = (self.c + (self.c << 3)) & M64
        self.c = (((self.c << 24) | (self.c >> 40)) & M64) + tmp & M64
        return tmp


def _next_double(g):
    return (g.next64() >> 11) * (1.0 / 9007199254740992.0)


def standard_normals(g, n):
    """numpy random_standard_normal x n -> (values, per-draw path list)."""
    vals, paths = [], []
    for _ in range(n):
        path = []
        while True:
            r = g.next64()
            idx = r & 0xFF
            r >>= 8
            sign = r & 1
            rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
            x = rabs * WI[idx]
            if sign:
                x = -x
            if rabs < KI[idx]:
                path.append("fast")
                break
            if idx == 0:
                while True:
                    xx = -0.27366123732975828 * math.log1p(-_next_double(g))
                    yy = -math.log1p(-_next_double(g))
                    if yy + yy > xx * xx:
                        break
                    path.append("tail-retry")
                x = -(3.6541528853610088 + xx) if (rabs >> 8) & 1 else 3.6541528853610088 + xx
                path.append("tail")
                break
            if (FI[idx - 1] - FI[idx]) * _next_double(g) + FI[idx] < math.exp(-0.5 * x * x):
                path.append("wedge")
                break
            path.append("wedge-reject")
        vals.append(x)
        paths.append(path)
    return vals, paths


def draw(key_vals, n, generator="pcg64"):
    ent = entropy_words(key_vals)
    g = PCG64(ent) if generator == "pcg64" else SFC64(ent)
    return standard_normals(g, n)
