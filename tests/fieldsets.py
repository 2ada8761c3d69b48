"""Coefficient fields shared by the golden generator and the tests."""
import numpy as np


def nodes(d, a=-4.0, b=4.0):
    delta = (b - a) / float(d + 1)
    return np.array([a + float(i + 1) * delta for i in range(d)])


def custom_fields(d):
    """Nine smooth non-zero coefficient fields (the general kinetic SPDE), sampled at the
    interior nodes in the column-major Field order (index j*nx + i)."""
    x = nodes(d)
    X, V = np.meshgrid(x, x, indexing="xy")
    f = {
        "h": 0.2 * np.cos(X) - 0.1,
        "fx": -V,
        "fv": 0.3 * np.sin(X),
        "gxx": 0.05 * (1.0 + 0.5 * np.cos(V)),
        "gxv": 0.02 * np.sin(X + V),
        "gvv": 1.1 * (1.0 + 1.0 / (X * X + 1.0)),
        "sig": 0.1 * np.cos(V),
        "sigx": 0.05 * np.sin(X),
        "sigv": 0.3 * np.sqrt(1.0 + 1.0 / (X * X + 1.0)),
    }
    return {k: np.ascontiguousarray(a.reshape(-1)) for k, a in f.items()}


def kinetic_fields(d):
    """The paper's general kinetic SPDE du = (a/2 d_vv + v d_x + b d_v + c) u dt + (sigma d_v +
    beta) u dW with x- and v-dependent a, b, c, sigma, beta (fields gvv, fv, h, sigv, sig; the
    transport fx = -v as in the Langevin families)."""
    x = nodes(d)
    X, V = np.meshgrid(x, x, indexing="xy")
    f = {
        "h": 0.2 * np.cos(X + 0.3 * V) - 0.1,
        "fx": -V,
        "fv": 0.3 * np.sin(X) * np.cos(V),
        "gvv": 1.1 * (1.0 + 1.0 / (X * X + V * V + 1.0)),
        "sig": 0.1 * np.cos(V + X),
        "sigv": 0.3 * np.sqrt(1.0 + 1.0 / (X * X + 1.0 + 0.1 * V * V)),
    }
    return {k: np.ascontiguousarray(a.reshape(-1)) for k, a in f.items()}
