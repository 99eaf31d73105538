"""NetworkEps evaluation: the network kinds behind `evaluate(d, s, x, t)`.

A NetworkEps wraps a model object exposing
    forward(xs, t_dev, B, outs)   xs: B latent rows (fp64/fp32 CUDA), t_dev: (B,) fp32
                                  model timesteps on device, outs: B fp32 rows (eps)
    max_batch                     largest batch its buffers hold
The sampler engine lowers every eval step of a run to one call with a static
t tensor (so the whole run stays CUDA-graph capturable); the k draft
evaluations that a rank owns in a round run as ONE batched forward.
Sampler timesteps are mapped to model timesteps as t * t_scale (e.g. 1000/T
for a 1000-step-trained DiT sampled with T steps).
"""

import torch


def _t_model(d, s, ts):
    scale = d.t_scale if d.t_scale is not None else 1000.0 / s.T
    return [float(t) * scale for t in ts]


def lower_eval(d, s, xs, ts, outs, device):
    """Static payload for engine.DeviceRun: chunks of <= max_batch tasks."""
    mb = getattr(d.net, "max_batch", 1)
    chunks = []
    tm = _t_model(d, s, ts)
    for i in range(0, len(xs), mb):
        t_dev = torch.tensor(tm[i:i + mb], dtype=torch.float32, device=device)
        chunks.append((xs[i:i + mb], t_dev, outs[i:i + mb]))
    return chunks


def network_eval_into(d, chunks):
    for ch in chunks:
        xs, t_dev, outs = ch[:3]
        if len(ch) > 3:                  # rows of the run's conditioning table
            d.net.forward(xs, t_dev, len(xs), outs=outs, cond_rows=ch[3])
        else:
            d.net.forward(xs, t_dev, len(xs), outs=outs)


def plan_conditioning(d, launches, device):
    """Per-run conditioning table (networks with prepare_conditioning, e.g. the DiT):
    one table row per local eval task in launch order, so every batched chunk reads a
    contiguous block.  Rewrites the "net" payloads in `launches` to carry their rows and
    returns the payload of the "cond" launch that fills the table (None if not used)."""
    net = d.net
    if not hasattr(net, "prepare_conditioning") or not getattr(net, "COND_TABLE", False):
        return None
    ts, payloads = [], []
    for kind, payload in launches:
        if kind != "eval" or payload[1] is None:
            continue
        low = payload[1][1] if payload[1][0] == "pert" else payload[1]
        if low[0] != "net":
            continue
        new_chunks = []
        for ch in low[1]["chunks"]:
            rows = tuple(range(len(ts), len(ts) + len(ch[0])))
            ts.extend(float(v) for v in ch[1][:len(ch[0])].tolist())
            new_chunks.append((ch[0], ch[1], ch[2], rows))
        payloads.append((low[1], new_chunks))
    if not ts:
        return None
    net.alloc_conditioning(len(ts))
    for a, new_chunks in payloads:
        a["chunks"] = new_chunks
    return torch.tensor(ts, dtype=torch.float32, device=device)


def network_eps(d, s, x, ts):
    """Functional evaluate(): x (D,) or (B, D) -> eps fp32 of the same shape."""
    from .transitions import _device_of, as_device
    dev = _device_of(x)
    xd = as_device(x, dev, torch.float64)
    flat = xd.reshape(-1, xd.shape[-1]) if xd.dim() > 1 else xd.reshape(1, -1)
    out = torch.empty(flat.shape, dtype=torch.float32, device=dev)
    xs = [flat[i] for i in range(flat.shape[0])]
    outs = [out[i] for i in range(flat.shape[0])]
    network_eval_into(d, lower_eval(d, s, xs, list(ts) * len(xs) if len(ts) == 1 else ts, outs, dev))
    return out.reshape(xd.shape)
