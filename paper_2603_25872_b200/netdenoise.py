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
    for xs, t_dev, outs in chunks:
        d.net.forward(xs, t_dev, len(xs), outs=outs)


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
