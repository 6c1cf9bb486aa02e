"""NumPy backend of the distributed RQRCP orchestration, for the CPU (gloo)
tests only.  Compute comes from the oracle (oracle/port.py); data movement and
communication are the same as GpuOps (torch tensors + torch.distributed)."""
import numpy as np
import torch

from oracle import port as O
from paper_2008_04447_b200.distributed import _Panel, _Sample, move_plan


class NumpyOps:
    def __init__(self):
        self._floor = None

    @staticmethod
    def mat(A):  # (ncols, ld) storage -> (ld, ncols) writable NumPy view
        return A.numpy().T

    def sketch(self, A, m, ell, seed, omega, gloc):
        Om = O.gauss_matrix(ell, m, seed) if omega is None else np.asarray(omega)
        Bl = Om @ self.mat(A)[:m]
        return torch.from_numpy(np.ascontiguousarray(Bl.T))

    def _assemble(self, parts, lay, ell, p0):
        out = torch.zeros((max(lay.n - p0, 1), ell), dtype=torch.float64)
        for q, part in enumerate(parts):
            g = lay.global_of_local(q)
            g = g[g >= p0]
            if g.size:
                out[torch.as_tensor(g - p0)] = part[:g.size]
        return out

    def assemble(self, parts, lay, ell):
        return self._assemble(parts, lay, ell, 0)

    def pad_slab(self, Bn, lay, achieved):
        nmax = max(lay.n_local(q) for q in range(lay.P))
        out = torch.zeros((nmax, Bn.shape[1]), dtype=torch.float64)
        nb = min(Bn.shape[0], nmax)
        out[:nb] = Bn[:nb]
        return out

    def assemble_next(self, parts, lay, achieved, ell):
        return self._assemble(parts, lay, ell, achieved)

    def sample_qrcp(self, B, ell, nt, bb, first, pend_pan=None):
        smp = self._sample_qrcp(B, ell, nt, bb, first)
        smp.prev_tail = self.read_tail(pend_pan) if pend_pan is not None else None
        return smp

    def _sample_qrcp(self, B, ell, nt, bb, first):
        Bm = B[:nt].numpy().T
        csq = np.einsum("ij,ij->j", Bm, Bm)
        if first:
            self._floor = O.sample_floor_sq(Bm)
        if csq.size == 0 or csq.max() <= self._floor:
            return _Sample(True, "sample_floor", 0, np.zeros((0, 2), np.int64), None, None)
        st = O.sample_pivots(Bm, bb)
        if st.achieved == 0:
            return _Sample(True, "sample_rank", 0, np.zeros((0, 2), np.int64), None, None)
        lp = st.local_perm
        q = np.nonzero(lp != np.arange(nt))[0]
        moves = np.stack([q, lp[q]], axis=1).astype(np.int64)
        return _Sample(False, "none", st.achieved, moves, torch.from_numpy(np.ascontiguousarray(st.B.T)), st)

    def move_columns(self, A, ps, pd, lay, comm, i0=None, samp=None):
        # the same plan GpuOps executes (distributed.move_plan)
        plan = move_plan(ps, pd, lay, comm.rank)
        packed = A[torch.as_tensor(plan.pack)].clone() if plan.pack.size else None
        sends = {q: packed[torch.as_tensor(rows)] for q, rows in plan.send.items()}
        shapes = {q: (int(dst.size), A.shape[1]) for q, dst in plan.recv.items()}
        recvs = comm.exchange(sends, shapes, A)
        if plan.local_rows.size:
            A[torch.as_tensor(plan.local_dst)] = packed[torch.as_tensor(plan.local_rows)]
        for q, buf in recvs.items():
            A[torch.as_tensor(plan.recv[q])] = buf

    def panel(self, A, lc, i0, m, w, bb, is_owner):
        mr = m - i0
        Y = torch.zeros((bb, mr), dtype=torch.float64)
        taus = torch.zeros(bb, dtype=torch.float64)
        R11 = torch.zeros((bb, bb), dtype=torch.float64)
        meta = torch.zeros(18, dtype=torch.uint8)
        if is_owner:
            M = self.mat(A)
            work = np.array(M[i0:m, lc:lc + bb], order="F")
            Yp, tp, bh = O.panel_factor(work, 0, w)
            M[i0:m, lc:lc + bb] = work
            Y[:bh] = torch.from_numpy(np.ascontiguousarray(Yp.T))
            taus[:bh] = torch.from_numpy(tp)
            R11.copy_(A[lc:lc + bb, i0:i0 + bb])
            st = torch.zeros(24, dtype=torch.uint8)
            st.view(torch.int32)[5] = bh
            if bh == 0:
                st.view(torch.int32)[0] = 1
        else:
            st = torch.zeros(24, dtype=torch.uint8)
        return _Panel(0, Y, taus, None, R11, None, st)

    def broadcast_panel(self, pan, owner, comm, mr, bb):
        meta = pan.st[:24].view(torch.int32)
        comm.broadcast(meta, owner)
        comm.broadcast(pan.Y, owner)
        comm.broadcast(pan.taus, owner)
        comm.broadcast(pan.R11, owner)
        pan.tail = meta
        return pan

    def read_tail(self, pan):
        mh = pan.tail.numpy()
        bhat = 0 if mh[0] else int(mh[5])
        return bhat, pan.taus.numpy().copy(), np.diag(pan.R11.numpy().T[:bhat, :bhat]).copy()

    def block_update(self, A, t0, i0, m, pan, ncols=None):
        Y = pan.Y.numpy().T
        tau = pan.taus.numpy()
        T = O.t_factor(Y, tau)
        pan.T = T
        C = self.mat(A)[i0:m, t0:] if ncols is None else self.mat(A)[i0:m, t0:t0 + ncols]
        if C.shape[1]:
            W = T.T @ (Y.T @ C)
            C -= Y @ W

    # paired second sweep (storage rows [m, m + b) = W_P, [m + b, m + 2b) = W_J)
    def block_update_defer(self, A, t0, i0, m, pan):
        Y = pan.Y.numpy().T
        T = O.t_factor(Y, pan.taus.numpy())
        pan.T = T
        M = self.mat(A)
        C = M[i0:m, t0:]
        if C.shape[1]:
            bb = Y.shape[1]
            W = -T.T @ (Y.T @ C)
            M[m:m + bb, t0:] = W
            C[:bb] += Y[:bb] @ W

    def pending_panel(self, A, lc, i0, m, w, pendP):
        pi0, b, ppan, _ = pendP
        M = self.mat(A)
        Yp = ppan.Y.numpy().T
        M[i0:m, lc:lc + w] += Yp[i0 - pi0:] @ M[m:m + b, lc:lc + w]
        M[m:m + b, lc:lc + w] = 0.0

    def block_update_merge(self, A, t0, i0, m, pan, pendP):
        pi0, b, ppan, _ = pendP
        Yj = pan.Y.numpy().T
        T = O.t_factor(Yj, pan.taus.numpy())
        pan.T = T
        M = self.mat(A)
        C = M[i0:m, t0:]
        if C.shape[1]:
            bb = Yj.shape[1]
            Yp = ppan.Y.numpy().T[i0 - pi0:]
            Wp = M[m:m + b, t0:]
            Wt = Yj.T @ C + (Yj.T @ Yp) @ Wp
            Wj = -T.T @ Wt
            M[m + b:m + b + bb, t0:] = Wj
            C += np.hstack([Yp, Yj]) @ np.vstack([Wp, Wj])

    def flush_pending(self, A, t0, i0, m, pan):
        M = self.mat(A)
        Yp = pan.Y.numpy().T
        b = Yp.shape[1]
        C = M[i0 + b:m, t0:]
        if C.shape[1] and C.shape[0]:
            C += Yp[b:] @ M[m:m + b, t0:]

    # TRQRCP (distributed.trqrcp_block_cyclic)
    def new_yg(self, m, k):
        return np.zeros((m, max(k, 1)), order="F")

    def tr_panel(self, S, lc, i0, m, k, w, bb, is_owner, Yg):
        mr = m - i0
        Y = torch.zeros((bb, mr), dtype=torch.float64)
        taus = torch.zeros(bb, dtype=torch.float64)
        R11 = torch.zeros((bb, bb), dtype=torch.float64)
        st = torch.zeros(24, dtype=torch.uint8)
        if is_owner:
            M = self.mat(S)
            panel = np.array(M[i0:m, lc:lc + w], order="F")
            if i0:
                panel -= Yg[i0:, :i0] @ M[m:m + i0, lc:lc + w]
            Yp, tp, bh = O.panel_factor(panel, 0, w)
            Y[:bh] = torch.from_numpy(np.ascontiguousarray(Yp.T))
            taus[:bh] = torch.from_numpy(tp)
            R11[:w, :w] = torch.from_numpy(np.ascontiguousarray(panel[:w, :w].T))   # (col, row) storage
            st.view(torch.int32)[5] = bh
            if bh == 0:
                st.view(torch.int32)[0] = 1
        return _Panel(0, Y, taus, None, R11, None, st)

    def tr_update(self, S, t0, i0, m, k, pan, bhat, Yg, lc):
        M = self.mat(S)
        Y2 = pan.Y.numpy().T[:, :bhat]
        Yg[i0:, i0:i0 + bhat] = Y2
        if lc >= 0:
            M[m + k + i0:m + k + i0 + bhat, lc:lc + bhat] = np.triu(pan.R11.numpy().T[:bhat, :bhat])
        if S.shape[0] <= t0:
            return
        T2 = O.t_factor(Y2, pan.taus.numpy()[:bhat])
        cols = slice(t0, S.shape[0])
        G = Y2.T @ M[i0:m, cols]
        if i0:
            G -= (Y2.T @ Yg[i0:, :i0]) @ M[m:m + i0, cols]
        M[m + i0:m + i0 + bhat, cols] = T2.T @ G
        M[m + k + i0:m + k + i0 + bhat, cols] = (M[i0:i0 + bhat, cols]
                                                  - Yg[i0:i0 + bhat, :i0 + bhat] @ M[m:m + i0 + bhat, cols])

    def sample_update_local(self, samp, A, s0, rel, i0, bb, pan, r_row0=None):
        r_row0 = i0 if r_row0 is None else r_row0
        ell = samp.Bf.shape[1]
        if len(rel) == 0:
            return torch.zeros((0, ell), dtype=torch.float64)
        Bf = samp.Bf.numpy().T
        R11 = np.triu(pan.R11.numpy().T)
        if not O.r11_usable(R11):
            # speculative block (short panel / singular R11, settled at the next
            # sync): like the device guard, produce no sample
            return torch.zeros((len(rel), ell), dtype=torch.float64)
        R12 = self.mat(A)[r_row0:r_row0 + bb, s0:s0 + len(rel)]
        X = O.back_solve(R11, R12)
        top = Bf[:bb, rel] - np.triu(Bf[:bb, :bb]) @ X
        Bn = np.vstack([top, Bf[bb:, rel]])
        return torch.from_numpy(np.ascontiguousarray(Bn.T))
