"""Test infrastructure: several "virtual ranks" of the domain-decomposed solver inside ONE process on
ONE GPU.  Every rank gets its own Context (stream) and runs in its own thread; the library's callback
communicator (hdgb_comm_set_callbacks) calls back into Python, where the halo exchange and the
all-reduce are done through host memory with thread barriers.  Same partitioner, same halo plan and
same library code path as the NCCL run -- only the transport differs."""
import ctypes as C
import threading

import numpy as np

import paper_2512_13619_b200 as hdg
from paper_2512_13619_b200 import hdg as H
from paper_2512_13619_b200 import partition as P

HALO_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int)
ALLRED_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int)


class Loopback:
    def __init__(self, lms):
        self.lms = lms
        self.n = len(lms)
        self.barrier = threading.Barrier(self.n)
        self.ptrs = [None] * self.n
        self.bufs = [None] * self.n
        self.ctxs = [hdg.Context(0) for _ in range(self.n)]
        self._keep = []
        for r in range(self.n):
            self._install(r)

    def _install(self, r):
        lm, ctx = self.lms[r], self.ctxs[r]

        def halo(user, vec, width):
            try:
                self.ptrs[r] = (vec, width)
                self.barrier.wait()
                for k, s in enumerate(lm.nbr_ranks):
                    cnt = int(lm.recv_cnt[k])
                    if cnt == 0:
                        continue
                    ls = self.lms[int(s)]
                    ids = ls.send_ids[list(ls.nbr_ranks).index(r)]
                    src, w2 = self.ptrs[int(s)]
                    assert w2 == width and len(ids) == cnt
                    full = np.empty(len(ls.faces) * width)
                    ctx.copy(full, src, full.size)
                    vals = np.ascontiguousarray(full.reshape(-1, width)[ids])
                    ctx.copy(vec + int(lm.recv_off[k]) * width * 8, vals, vals.size)
                self.barrier.wait()
                return 0
            except Exception as e:  # pragma: no cover
                print("halo callback failed:", repr(e))
                self.barrier.abort()
                return 1

        def allreduce(user, buf, n):
            try:
                mine = np.empty(n)
                ctx.copy(mine, buf, n)
                self.bufs[r] = mine
                self.barrier.wait()
                tot = np.zeros(n)
                for q in range(self.n):          # fixed rank order: deterministic
                    tot += self.bufs[q]
                self.barrier.wait()
                ctx.copy(buf, tot, n)
                return 0
            except Exception as e:  # pragma: no cover
                print("allreduce callback failed:", repr(e))
                self.barrier.abort()
                return 1

        hf, af = HALO_FN(halo), ALLRED_FN(allreduce)
        self._keep += [hf, af]
        L = H.load_library()
        ctx.check(L.hdgb_comm_set_callbacks(ctx._h, r, self.n, C.cast(hf, C.c_void_p), C.cast(af, C.c_void_p), None))

    def run(self, fn):
        """fn(rank, ctx, local_mesh) on every virtual rank concurrently; returns the list of results."""
        out, err = [None] * self.n, [None] * self.n

        def work(r):
            try:
                out[r] = fn(r, self.ctxs[r], self.lms[r])
            except BaseException as e:
                err[r] = e
                self.barrier.abort()

        ts = [threading.Thread(target=work, args=(r,)) for r in range(self.n)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for e in err:
            if e is not None and not isinstance(e, threading.BrokenBarrierError):
                raise e
        for e in err:
            if e is not None:
                raise e
        return out

    def close(self):
        L = H.load_library()
        for c in self.ctxs:
            L.hdgb_comm_destroy(c._h)
            c.close()
