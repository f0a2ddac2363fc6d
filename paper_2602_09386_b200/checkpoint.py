"""MOECKPT1 model checkpoints -- drop-in for taskmoe/checkpoint.py (``load_model`` / ``save_model``).

The on-disk format is the reference's (checkpoint.py:1-14), little-endian throughout:

    b"MOECKPT1" | 10 x uint32 header: version=1, num_features, d_hidden, d_in, d_out, num_experts,
    num_tasks, k_shared, k_adaptive, nonlinearity (expert_code*16 + encoder_code; 0 identity,
    1 relu) | uint64 seed, float64 lb_strength | T float64 task loss weights | T float64 router
    pooling weights | every parameter block as raw float64 in ``parameter_blocks()`` order
    (encoder1 w/b, encoder2 w/b, expert_0.. w/b, router_0.. w/b, head_0.. w/b).

B200 side: the file is parsed on the host in one pass and each block lands in the stacked device
layout the kernels use -- experts (E, d_out, d_in), routers (T, E, d_in), heads (T, 1, d_out) -- as
``dtype`` tensors (fp32 by default; fp64 keeps the file's bits, so load -> save is byte-identical).
The format holds one expert pool (the reference expert); the two-pool expert MLP of the
BASELINE configs has no MOECKPT1 encoding and ``save_model`` rejects it.
"""
from __future__ import annotations

import os
import struct
import tempfile

import numpy as np
import torch

from .errors import ConfigError, DataFormatError
from .experts import ExpertPool
from .linalg import Affine
from .model import MoeModel, heads_from_stacked
from .routing import RouterBank, RoutingBudget

__all__ = ["load_model", "save_model", "MAGIC", "VERSION"]

MAGIC = b"MOECKPT1"
VERSION = 1
_CODE = {"identity": 0, "relu": 1}
_NAME = {v: k for k, v in _CODE.items()}
_HEADER = struct.Struct("<10I")
_SEED = struct.Struct("<Qd")


def _f64(t: torch.Tensor) -> bytes:
    return np.ascontiguousarray(t.detach().to("cpu", torch.float64).numpy(), dtype="<f8").tobytes()


def save_model(model: MoeModel, seed: int, path: str) -> None:
    """Write ``model`` as a MOECKPT1 file (checkpoint.py:38-66): temp file in the target
    directory, then an atomic rename."""
    pools = model.pools
    if len(pools) != 1:
        raise ConfigError(f"MOECKPT1 stores one expert pool, the model has {len(pools)} chained pools")
    if model.encoder1 is None or model.encoder2 is None:
        raise ConfigError("MOECKPT1 stores the encoder; the model has none")
    pool = pools[0]
    header = _HEADER.pack(VERSION, model.encoder1.d_in, model.encoder1.d_out, model.d_in, model.d_out,
                          model.num_experts, model.num_tasks, model.budget.k_shared, model.budget.k_adaptive,
                          _CODE[pool.nonlinearity] * 16 + _CODE[model.encoder_nonlinearity])
    parts = [MAGIC, header, _SEED.pack(int(seed), float(model.lb_strength)),
             _f64(model.task_loss_weights), _f64(model.routers.task_weights)]
    parts += [_f64(b) for b in model.parameter_blocks().values()]
    payload = b"".join(parts)
    directory = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(dir=directory, prefix=".tmp_moeckpt_")
    try:
        with os.fdopen(fd, "wb") as fh:
            fh.write(payload)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def load_model(path: str, device="cuda", dtype: torch.dtype = torch.float32) -> tuple[MoeModel, int]:
    """Read a MOECKPT1 file (checkpoint.py:91-152); returns ``(model, seed)``.  Raises
    DataFormatError for an unreadable file, bad magic, unknown version or nonlinearity code, a
    truncated payload or trailing bytes -- the reference's checks, in its order."""
    try:
        with open(path, "rb") as fh:
            raw = fh.read()
    except OSError as err:
        raise DataFormatError(f"cannot read checkpoint {path}: {err}") from err
    pos = 0

    def take(n: int) -> bytes:
        nonlocal pos
        if pos + n > len(raw):
            raise DataFormatError(f"{path}: checkpoint truncated at byte {pos}")
        chunk = raw[pos:pos + n]
        pos += n
        return chunk

    def block(*shape: int) -> np.ndarray:
        n = int(np.prod(shape))
        return np.frombuffer(take(8 * n), dtype="<f8").reshape(shape)

    if take(len(MAGIC)) != MAGIC:
        raise DataFormatError(f"{path}: not a model checkpoint (bad magic)")
    (version, n_feat, d_hid, d_in, d_out, E, T, ks, ka, nonlin) = _HEADER.unpack(take(_HEADER.size))
    if version != VERSION:
        raise DataFormatError(f"{path}: unsupported checkpoint version {version}")
    exp_code, enc_code = divmod(nonlin, 16)
    if exp_code not in _NAME or enc_code not in _NAME:
        raise DataFormatError(f"{path}: unknown nonlinearity code {nonlin}")
    seed, lb = _SEED.unpack(take(_SEED.size))
    lam = block(T)
    tw = block(T)
    enc = []
    for rows, cols in ((d_hid, n_feat), (d_in, d_hid)):
        enc.append((block(rows, cols), block(rows)))
    ew = np.empty((E, d_out, d_in))
    eb = np.empty((E, d_out))
    for e in range(E):
        ew[e] = block(d_out, d_in)
        eb[e] = block(d_out)
    rw = np.empty((T, E, d_in))
    rb = np.empty((T, E))
    for t in range(T):
        rw[t] = block(E, d_in)
        rb[t] = block(E)
    hw = np.empty((T, d_out))
    hb = np.empty(T)
    for t in range(T):
        hw[t] = block(1, d_out)[0]
        hb[t] = block(1)[0]
    if pos != len(raw):
        raise DataFormatError(f"{path}: {len(raw) - pos} trailing bytes after parameters")

    dev = torch.device(device)
    to = lambda a: torch.from_numpy(np.array(a, dtype=np.float64)).to(dev, dtype)
    model = MoeModel(
        encoder1=Affine(to(enc[0][0]), to(enc[0][1])),
        encoder2=Affine(to(enc[1][0]), to(enc[1][1])),
        experts=ExpertPool.stacked(to(ew), to(eb), _NAME[exp_code]),
        routers=RouterBank(to(rw), to(rb), torch.from_numpy(np.array(tw))),
        heads=heads_from_stacked(to(hw), to(hb)),
        task_loss_weights=torch.from_numpy(np.array(lam)),
        lb_strength=float(lb),
        budget=RoutingBudget(k_shared=ks, k_adaptive=ka),
        encoder_nonlinearity=_NAME[enc_code],
    )
    return model, int(seed)
