"""Network eps-predictors (NetworkEps) on the package's kernels.

Placeholder until the tcgen05 denoiser networks land: evaluating a
NetworkEps raises instead of silently falling back to anything else."""


def network_eps(d, s, x, ts):
    raise NotImplementedError("NetworkEps evaluation lands with the tcgen05 denoisers")


def network_eval_into(d, s, xs, ts, outs):
    raise NotImplementedError("NetworkEps evaluation lands with the tcgen05 denoisers")
