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
        for i, a in enumerate(self._items):
            if a.weight.data_ptr() != w[i].data_ptr() or a.bias.data_ptr() != b[i].data_ptr() \
                    or a.weight.shape != w.shape[1:] or a.bias.shape != b.shape[1:]:
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
