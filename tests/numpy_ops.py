"""Oracle-backed row operations for the limb-sharded key-switch (CPU tests only).

`shard.keyswitch_limb_sharded` is written against a small row-ops interface;
the product binds it to the CUDA library (`shard.TorchOps`), the gloo CPU
tests bind it to the numpy oracle through this class.  It lives under tests/
because only the checker may import `oracle/`.
"""

import numpy as np


class NumpyOps:
    """Oracle-backed row ops (the shard.TorchOps interface on numpy arrays)."""

    def __init__(self):
        from oracle import ckks_np
        self.o = ckks_np

    def intt(self, x, mods):
        return self.o.intt(x, mods)

    def ntt(self, x, mods):
        return self.o.ntt(x, mods)

    def bc_convert(self, x, src, dst):
        if len(dst) == 0:
            return np.zeros((0, x.shape[1]), dtype=np.uint64)
        return self.o.bc_convert(x, src, dst)

    def bc_convert_centered(self, x, src, dst):
        if len(dst) == 0:
            return np.zeros((0, x.shape[1]), dtype=np.uint64)
        return self.o.bc_convert_centered(x, src, dst)

    def automorph(self, x, t):
        return self.o.automorph(x, t)

    def _q(self, mods):
        return np.array(mods, dtype=np.uint64)[:, None]

    def mul(self, x, y, mods):
        return self.o.mulmod(x, y, self._q(mods))

    def add(self, x, y, mods):
        return self.o.addmod(x, y, self._q(mods))

    def sub(self, x, y, mods):
        return self.o.submod(x, y, self._q(mods))

    def mul_scalars(self, x, s, mods):
        return self.o.mulmod(x, np.array(s, dtype=np.uint64)[:, None], self._q(mods))

    def take_rows(self, x, idx):
        return x[list(idx)]

    def cat_rows(self, parts):
        return np.concatenate(parts, axis=0)

    # collective helpers (torch tensors on the wire)
    def pad_rows(self, x, width):
        import torch
        out = np.zeros((width, x.shape[1]), dtype=np.uint64)
        out[:x.shape[0]] = x
        return torch.from_numpy(out.view(np.int64))

    def empty_like(self, t):
        import torch
        return torch.empty_like(t)

    def empty_rows(self, rows, like):
        return np.zeros((rows, like.shape[1]), dtype=np.uint64)

    def set_row(self, out, row, part, k):
        out[row] = part[k].numpy().view(np.uint64)
