"""A list of ``Affine`` maps backed by stacked device tensors.

The reference stores expert pools, router banks and task heads as Python lists
of ``Affine`` objects (experts.py:17-73, routing.py:64-103, model.py:36-49).
The kernels want them stacked: (n, d_out, d_in) weights and (n, d_out) biases.
``AffineStack`` keeps both views of the same storage: every ``Affine`` in
``items`` holds views into the stacked tensors, so in-place updates made
through either side (an optimizer step on ``parameter_blocks()`` views, or on
the stacked tensor) are shared.  If a caller rebinds an item's ``weight`` /
``bias`` to a new tensor, the next access to the stacked tensors re-stacks.
"""
from __future__ import annotations

import torch

from .errors import ShapeError
from .linalg import Affine


class AffineStack:
    def __init__(self, items=None, weight: torch.Tensor | None = None, bias: torch.Tensor | None = None):
        if items is not None:
            items = list(items)
            for a in items:
                if not isinstance(a, Affine):
                    raise TypeError(f"expected Affine maps, got {type(a).__name__}")
            self._items = items
            self._restack()
        else:
            w = torch.as_tensor(weight)
            b = torch.as_tensor(bias)
            if w.ndim != 3 or b.shape != w.shape[:2]:
                raise ShapeError(f"stacked affines expect weight (n, d_out, d_in) and bias (n, d_out), got "
                                 f"{tuple(w.shape)} and {tuple(b.shape)}")
            self._w, self._b = w, b
            self._items = [Affine(w[i], b[i]) for i in range(w.shape[0])]

    # -- storage
    def _restack(self):
        if not self._items:
            self._w = self._b = None
            return
        self._w = torch.stack([a.weight for a in self._items])
        self._b = torch.stack([a.bias.to(self._w.device) for a in self._items])
        for i, a in enumerate(self._items):
            a.weight, a.bias = self._w[i], self._b[i]

    def _fresh(self) -> bool:
        w, b = self._w, self._b
        if w is None or len(self._items) != w.shape[0]:
            return False
        # item i must still be the view w[i] / b[i]: compared by address arithmetic (indexing the
        # stack per item on every access cost ~0.5 ms of host time per API step at E = 32)
        w0, ws, wsh, wst = w.data_ptr(), w.stride(0) * w.element_size(), w.shape[1:], w.stride()[1:]
        b0, bs, bsh, bst = b.data_ptr(), b.stride(0) * b.element_size(), b.shape[1:], b.stride()[1:]
        for i, a in enumerate(self._items):
            aw, ab = a.weight, a.bias
            if aw.data_ptr() != w0 + i * ws or ab.data_ptr() != b0 + i * bs or aw.shape != wsh \
                    or ab.shape != bsh or aw.stride() != wst or ab.stride() != bst:
                return False
        return True

    @property
    def items(self) -> list:
        return self._items

    @property
    def weight(self) -> torch.Tensor:
        if not self._fresh():
            self._restack()
        return self._w

    @weight.setter
    def weight(self, w):
        w = torch.as_tensor(w)
        if self._w is not None and w.shape != self._w.shape:
            raise ShapeError(f"stacked weight must keep shape {tuple(self._w.shape)}, got {tuple(w.shape)}")
        self._b = self.bias              # (re-stacks first if an item was rebound)
        self._w = w
        for i, a in enumerate(self._items):
            a.weight = w[i]

    @property
    def bias(self) -> torch.Tensor:
        if not self._fresh():
            self._restack()
        return self._b

    @bias.setter
    def bias(self, b):
        b = torch.as_tensor(b)
        if self._b is not None and b.shape != self._b.shape:
            raise ShapeError(f"stacked bias must keep shape {tuple(self._b.shape)}, got {tuple(b.shape)}")
        self._w = self.weight            # (re-stacks first if an item was rebound)
        self._b = b
        for i, a in enumerate(self._items):
            a.bias = b[i]
