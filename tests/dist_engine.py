"""Oracle-backed local engine for the CPU (gloo) tests of paper_2005_03246_b200.distributed.

Test infrastructure only: it lets the multi-process tests drive the package's exact slab
decomposition / routing / carry-exchange code on CPU tensors, with every local step computed
by the pinned oracle instead of the CUDA kernels (which need a GPU)."""

import numpy as np
import torch

import oracle


class OracleEngine:
    def tensor(self, a):
        return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64))

    def axis_owner(self, x, knots_axis, le, shift, bounds):
        kn = np.asarray(knots_axis, dtype=np.float64)
        b = np.searchsorted(kn, x[:, 1].numpy(), side="right" if le else "left")
        c = b - shift
        owner = np.full(c.shape, -1, dtype=np.int32)
        for r in range(len(bounds) - 1):
            owner[(c >= bounds[r]) & (c < bounds[r + 1])] = r
        return torch.as_tensor(owner)

    def partition(self, x, w, owner, G):
        o = owner.numpy().astype(np.int64)
        key = np.where(o < 0, G, o)
        order = np.argsort(key, kind="stable")
        counts = [int(np.sum(key == r)) for r in range(G)]
        xo = x[torch.as_tensor(order)]
        wo = None if w is None else w[torch.as_tensor(order)]
        return xo, wo, counts

    def local_ecdf(self, x, w, grid, delta, survival):
        pts = x.numpy().reshape(-1, grid.dim)
        wn = None if w is None else w.numpy()
        if survival:
            v = oracle.esf_fastsum(pts, wn, grid.knots, scaled=False)
        else:
            v = oracle.ecdf_fastsum(pts, wn, grid.knots, delta.signs, scaled=False)
        return torch.as_tensor(v.astype(np.int64) if w is None else v)

    def slab_finish(self, local, carry, A, J, B, div):
        v = local.numpy().reshape(A, J, B)
        if carry is not None:
            v = v + carry.numpy().reshape(A, 1, B)
        v = v.astype(np.float64)
        if div > 0:
            v = v / div
        return torch.as_tensor(v.reshape(-1))

    def minmax(self, x):
        xn = x.numpy()
        if xn.shape[0] == 0:
            return np.full(xn.shape[1], np.inf), np.full(xn.shape[1], -np.inf)
        return xn.min(axis=0), xn.max(axis=0)

    def local_kde(self, x, w, grid, h, centre, n_scale, u_bound=-1.0):
        pts = x.numpy().reshape(-1, grid.dim)
        out, terms, _ = oracle.kde_fastsum_laplacian_terms(
            pts, None if w is None else w.numpy(), grid.knots, h, centre, n_scale)
        d = grid.dim
        kw = max(2, d - 2)  # slot weights: zf of axes >= kw (fastcdf_b200.h)
        knots = [np.asarray(z, dtype=np.float64) for z in grid.knots]
        planes = []
        for code, (_, s0) in enumerate(terms):
            rev = (code >> 1) & 1
            p = s0[:, 0] if rev else s0[:, -1]
            for k in range(kw, d):
                sgn = -1.0 if (code >> k) & 1 else 1.0
                sh = [1] * (d - 1)
                sh[k - 1] = len(knots[k])
                p = p * np.exp(-sgn * (knots[k] - centre[k]) / h[k]).reshape(sh)
            planes.append(np.ascontiguousarray(p).reshape(-1))
        return torch.as_tensor(out), torch.as_tensor(np.concatenate(planes))

    def kde_fixup(self, out, grid, h, centre, carries, n_scale):
        d = grid.dim
        shape = grid.shape
        knots = [np.asarray(z, dtype=np.float64) for z in grid.knots]
        plane_shape = (shape[0],) + tuple(shape[2:])
        ps = int(np.prod(plane_shape))
        cn = carries.numpy()
        acc = np.zeros(shape)
        for code in range(1 << d):
            signs = [-1.0 if (code >> k) & 1 else 1.0 for k in range(d)]
            zfac = np.ones(shape)
            for k in range(min(d, max(2, d - 2))):
                sh = [1] * d
                sh[k] = shape[k]
                zfac = zfac * np.exp(-signs[k] * (knots[k] - centre[k]) / h[k]).reshape(sh)
            c = cn[code * ps:(code + 1) * ps].reshape(plane_shape)
            acc += zfac * np.expand_dims(c, 1)
        scale = 1.0 / (2.0 ** d * n_scale * np.prod(h))
        return torch.as_tensor(out.numpy() + (acc * scale).reshape(-1))

    # ---- at-points query shards: the oracle's full answer, zeros outside the shard's chunks
    @staticmethod
    def _owned(x, shard, nshards, chunk=None):
        from paper_2005_03246_b200.distributed import POINTS_CHUNK, query_shard_chunks

        chunk = chunk or POINTS_CHUNK
        n = x.shape[0]
        pos1 = np.empty(n, dtype=np.int64)
        pos1[np.argsort(x[:, 1], kind="stable")] = np.arange(n)
        lo, hi = query_shard_chunks(n, shard, nshards, chunk)
        c = pos1 // chunk
        return (c >= lo) & (c < hi)

    def minmax(self, x):
        a = x.numpy()
        return a.min(axis=0), a.max(axis=0)

    def kde_points_shard(self, x, wmat, nw, h, centre, shard, nshards):
        pts = x.numpy()
        own = self._owned(pts, shard, nshards)
        out = np.zeros((nw, pts.shape[0]))
        for v in range(nw):
            out[v] = oracle.kde_dnc_laplacian(pts, wmat[v].numpy(), h)
        out[:, ~own] = 0.0
        return torch.as_tensor(out)

    def dnc_ecdf_shard(self, x, w, include_self, scaled, shard, nshards):
        pts = x.numpy()
        own = self._owned(pts, shard, nshards)
        out = oracle.ecdf_dnc(pts, None if w is None else w.numpy(), include_self, scaled)
        out = np.where(own, out, 0.0)
        return torch.as_tensor(out)
