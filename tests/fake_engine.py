"""Oracle-backed stand-in for ``BlockEngine`` (TEST INFRASTRUCTURE ONLY).

Implements the engine interface the synchronous outer driver uses
(``sync_driver.run_sync`` / ``distributed.HaloExchange``) with numpy and the
CPU oracle, on CPU tensors, so the multi-rank host logic (block ownership,
halo routing, exact block-row reductions, termination) can be exercised with
``gloo`` on a machine without a GPU.  It is never imported by the product.
"""

from types import SimpleNamespace

import numpy as np
import torch

from oracle import blocksolve_oracle as O
from paper_2009_12638_b200.problems import Box


class _Block:
    def __init__(self, owned, grid_shape):
        self.owned = owned
        self.padded = Box(owned.lo, owned.hi)
        nx, ny, nz = grid_shape
        px, py, pz = (owned.hi[d] - owned.lo[d] for d in range(3))
        self.dims = (px, py, pz)
        lo, hi = owned.lo, owned.hi
        faces = ((lo[2] > 0, px * py), (lo[1] > 0, px * pz), (lo[0] > 0, py * pz),
                 (hi[0] < nx, py * pz), (hi[1] < ny, px * pz), (hi[2] < nz, px * py))
        self.ghost = [torch.zeros(n, dtype=torch.float64) if ok else None for ok, n in faces]
        self.x = np.zeros((pz, py, px))
        self.b = np.zeros((pz, py, px))

    def plane(self, direction):
        """Own boundary plane facing `direction`, flattened like the ghost planes."""
        x = self.x
        return {0: x[0, :, :], 5: x[-1, :, :], 1: x[:, 0, :], 4: x[:, -1, :],
                2: x[:, :, 0], 3: x[:, :, -1]}[direction].reshape(-1).copy()

    def rhs(self):
        """b_ext - C*halo with the reduceat rule per row (multisplit.py:333-338)."""
        pz, py, px = self.x.shape
        terms = [[] for _ in range(pz * py * px)]
        idx = np.arange(pz * py * px).reshape(pz, py, px)
        sel = {0: idx[0, :, :], 1: idx[:, 0, :], 2: idx[:, :, 0], 3: idx[:, :, -1], 4: idx[:, -1, :],
               5: idx[-1, :, :]}
        for d in range(6):  # ascending column order
            if self.ghost[d] is None:
                continue
            h = self.ghost[d].numpy()
            for p, v in zip(sel[d].reshape(-1), h):
                terms[p].append(-v)
        out = self.b.reshape(-1).copy()
        for p, t in enumerate(terms):
            if t:
                s = t[0]
                if len(t) > 1:
                    rest = t[1]
                    for v in t[2:]:
                        rest = rest + v
                    s = s + rest
                out[p] = out[p] - s
        return out


class FakeEngine:
    overlap = 0
    comm_device = torch.device("cpu")

    def __init__(self, grid_shape, owned, overlap, local_ids):
        assert overlap == 0
        self.blocks = [_Block(box, grid_shape) for box in owned]
        self._params = None
        self._its = [0] * len(owned)
        self._stop = [0] * len(owned)
        self._rsq = [0.0] * len(owned)

    # data
    def load_host(self, name, g3):
        for bb in self.blocks:
            (x0, y0, z0), (x1, y1, z1) = bb.owned.lo, bb.owned.hi
            getattr(bb, name)[...] = g3[z0:z1, y0:y1, x0:x1]

    def gather_owned(self, out3, name="x"):
        for bb in self.blocks:
            (x0, y0, z0), (x1, y1, z1) = bb.owned.lo, bb.owned.hi
            out3[z0:z1, y0:y1, x0:x1] = torch.from_numpy(getattr(bb, name))

    # solves
    def cg_begin(self, max_iterations, tolerance, basis="rhs", active=None):
        self._params = (max_iterations, tolerance, basis)
        self._last = (list(self._its), list(self._stop))  # k_arm(PH_INIT) keeps the previous solve's

    def run(self, batch=4, max_launches=0):
        its, tol, basis = self._params
        for i, bb in enumerate(self.blocks):
            shape = bb.x.shape
            x, rep = O.cg(lambda v: O.stencil_apply(v.reshape(shape)).ravel(), bb.rhs(), bb.x.reshape(-1), its,
                          tol, basis)
            bb.x = x.reshape(shape)
            self._its[i] = rep.iterations_used
            self._stop[i] = {"tolerance_met": 1, "max_iterations": 2, "breakdown": 3}[rep.stop_reason]

    def sweep_resid(self):
        for i, bb in enumerate(self.blocks):
            r = bb.rhs() - O.stencil_apply(bb.x).ravel()
            self._rsq[i] = float(r @ r)

    def reports(self):
        last_its, last_stop = getattr(self, "_last", (self._its, self._stop))
        return [SimpleNamespace(iterations_used=self._its[i], stop_reason=self._stop[i], r_owned_sq=self._rsq[i],
                                rglob_owned_sq=self._rsq[i], last_iterations=last_its[i],
                                last_stop_reason=last_stop[i]) for i in range(len(self.blocks))]

    def cancel(self, active=None):
        pass

    def flush(self):
        pass

    def close(self):
        pass

    # halo planes
    def halo_pack(self, plan):
        for d, dr, s in np.asarray(plan).reshape(-1, 3).tolist():
            self.blocks[d].ghost[dr].copy_(torch.from_numpy(self.blocks[s].plane(5 - dr)))

    def plane_len(self, block, direction):
        return self.blocks[block].plane(direction).size

    def new_plane(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def ghost(self, block, direction):
        return self.blocks[block].ghost[direction]

    def post_plane(self, block, direction, buf):
        buf.copy_(torch.from_numpy(self.blocks[block].plane(direction)))

    def post_plane_ptr(self, block, direction, ptr):
        raise NotImplementedError("the CPU stand-in has no device pointers")

    def synchronize(self):
        pass
