"""Shared test helpers (inputs and tolerance checks)."""
import numpy as np


def mamba_inputs(seed, batch, dim, N, L, unstructured=True):
    """Synthetic Mamba-1 layer inputs: u ~ N(0,1), raw delta ~ 0.1 N(0,1),
    delta_bias = softplus^-1(dt), dt ~ logU[1e-3, 1e-1], A = -(s+1)(1 + 0.1 U(-1,1)),
    B, C, z ~ N(0,1), D = 1 + 0.1 N(0,1).  fp32."""
    rng = np.random.default_rng(seed)
    u = rng.standard_normal((batch, dim, L)).astype(np.float32)
    delta = (0.1 * rng.standard_normal((batch, dim, L))).astype(np.float32)
    dt = np.exp(rng.uniform(np.log(1e-3), np.log(1e-1), dim))
    bias = np.log(np.expm1(dt)).astype(np.float32)
    jitter = rng.uniform(-1, 1, (dim, N)) if unstructured else np.zeros((dim, N))
    A = (-(np.arange(1, N + 1)[None, :]) * (1 + 0.1 * jitter)).astype(np.float32)
    B = rng.standard_normal((batch, N, L)).astype(np.float32)
    C = rng.standard_normal((batch, N, L)).astype(np.float32)
    D = (1 + 0.1 * rng.standard_normal(dim)).astype(np.float32)
    z = rng.standard_normal((batch, dim, L)).astype(np.float32)
    return dict(u=u, delta=delta, A=A, B=B, C=C, D=D, z=z, delta_bias=bias)


def rel_err_rows(y, ref):
    """Per-row normwise relative error ||y - ref||_2 / ||ref||_2."""
    y = np.asarray(y, dtype=np.float64).reshape(ref.shape[0], -1)
    ref = np.asarray(ref, dtype=np.float64).reshape(ref.shape[0], -1)
    num = np.linalg.norm(y - ref, axis=1)
    den = np.maximum(np.linalg.norm(ref, axis=1), 1e-30)
    return num / den


def assert_close_normwise(y, ref, tol=1e-5, what="y"):
    ref = np.asarray(ref, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64).reshape(ref.shape)
    r = rel_err_rows(y.reshape(-1, ref.shape[-1]), ref.reshape(-1, ref.shape[-1]))
    assert r.max() <= tol, f"{what}: worst row normwise rel err {r.max():.3e} > {tol}"
    whole = np.linalg.norm(y - ref) / max(np.linalg.norm(ref), 1e-30)
    assert whole <= tol, f"{what}: whole-tensor rel err {whole:.3e}"
    mx = np.abs(y - ref).max() / max(np.abs(ref).max(), 1e-30)
    assert mx <= tol, f"{what}: max|d|/max|ref| {mx:.3e}"
    return r.max(), whole, mx
