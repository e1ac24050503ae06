"""Thread-emulated torch.distributed for single-GPU tests of the slab decomposition.

Test infrastructure only: W Python threads play the ranks; every collective is a host-side
rendezvous (barrier + shared slots) with device copies, so no rank's kernel ever waits on
another's on the device.  It lets `pytest -m gpu` run paper_2005_03246_b200.distributed with
the real DeviceEngine (CUDA kernels) on one B200."""

import threading

import torch


class _Op:
    SUM = "sum"
    MAX = "max"


class ThreadDist:
    ReduceOp = _Op

    def __init__(self, world):
        self.world = world
        self.local = threading.local()
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world

    # -- torch.distributed surface used by the package --------------------------------------
    def is_initialized(self):
        return True

    def get_world_size(self, group=None):
        return self.world

    def get_rank(self, group=None):
        return self.local.rank

    def _share(self, obj):
        r = self.local.rank
        torch.cuda.synchronize()
        self.slots[r] = obj
        self.barrier.wait()
        got = list(self.slots)
        self.barrier.wait()
        return got

    def all_reduce(self, t, op=_Op.SUM, group=None):
        got = self._share(t.clone())
        acc = got[0].clone()
        for g in got[1:]:
            acc = acc + g if op == _Op.SUM else torch.maximum(acc, g)
        t.copy_(acc)

    def all_gather(self, bufs, t, group=None):
        got = self._share(t.clone())
        for b, g in zip(bufs, got):
            b.copy_(g)

    def all_to_all_single(self, out, inp, output_split_sizes=None, input_split_sizes=None,
                          group=None):
        W = self.world
        n_in = inp.shape[0]
        ins = input_split_sizes or [n_in // W] * W
        offs = [0]
        for c in ins:
            offs.append(offs[-1] + c)
        got = self._share((inp.clone(), offs))
        r = self.local.rank
        pos = 0
        for src in range(W):
            t, o = got[src]
            piece = t[o[r]:o[r + 1]]
            out[pos:pos + piece.shape[0]].copy_(piece)
            pos += piece.shape[0]

    # -- driver -------------------------------------------------------------------------------
    def run(self, fn):
        """fn(rank) on `world` threads; returns the per-rank results (re-raises failures)."""
        res = [None] * self.world
        err = []

        def body(r):
            self.local.rank = r
            try:
                res[r] = fn(r)
            except BaseException as e:  # noqa: BLE001 - surfaced below
                err.append(e)
                self.barrier.abort()

        th = [threading.Thread(target=body, args=(r,)) for r in range(self.world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if err:
            raise err[0]
        return res
