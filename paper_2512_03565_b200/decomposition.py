"""Spatial brick decomposition across ranks.

One process per GPU; the periodic box is split into px x py x pz bricks
(1 -> 1x1x1, 2 -> 2x1x1, 4 -> 2x2x1, 8 -> 2x2x2).  Each rank owns the
particles inside its brick and receives a ghost layer of thickness
rc + skin -- the multi-rank analogue of the reference's periodic images
(``build_halo``, domain.py:97-144): a ghost that crosses the global boundary
carries exactly the image position ``pos + (hi - lo)`` / ``pos + (lo - hi)``,
so pair sets and forces equal the single-domain ones.  Ghost pairs are
one-sided (the owned side is i, traversals.py:157-160): no reverse force
communication.

Exchange: three axis stages (x, y, z); stage a sends the particles (owned +
ghosts received in earlier stages) within ``margin`` of each a-face to the
neighbour on that side -- corners and edges are forwarded.  An axis with one
brick sends to itself (a local periodic image).  Send lists are fixed at
``plan()`` (each rebuild); ``exchange()`` moves only positions, through
``torch.distributed`` point-to-point ops (NCCL on GPUs, gloo on CPUs).
Migration (``migrate``) moves particles that left the brick at a rebuild.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

BRICKS = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}


def brick_grid(nranks: int) -> tuple[int, int, int]:
    if nranks in BRICKS:
        return BRICKS[nranks]
    # general: factor into three near-equal factors, x largest
    best = (nranks, 1, 1)
    for a in range(1, nranks + 1):
        if nranks % a:
            continue
        for b in range(1, nranks // a + 1):
            if (nranks // a) % b:
                continue
            c = nranks // a // b
            cand = tuple(sorted((a, b, c), reverse=True))
            if max(cand) - min(cand) < max(best) - min(best):
                best = cand
    return best


@dataclass
class _Stage:
    axis: int
    # per direction (0: toward lower neighbour / lo face, 1: upper / hi face)
    peer: list = field(default_factory=lambda: [None, None])
    send_idx: list = field(default_factory=lambda: [None, None])   # into [owned | ghosts so far]
    shift: list = field(default_factory=lambda: [0.0, 0.0])         # added to axis coordinate
    recv_count: list = field(default_factory=lambda: [0, 0])


class BrickDecomposition:
    def __init__(self, lo, hi, margin: float, rank: int = 0, nranks: int = 1, group=None,
                 grid: tuple | None = None):
        self.lo = np.asarray(lo, dtype=np.float64)
        self.hi = np.asarray(hi, dtype=np.float64)
        self.L = self.hi - self.lo
        self.margin = float(margin)
        self.rank = rank
        self.nranks = nranks
        self.group = group
        self.grid = tuple(grid) if grid is not None else brick_grid(nranks)
        if int(np.prod(self.grid)) != nranks:
            raise ValueError(f"brick grid {self.grid} does not match {nranks} ranks")
        self.coords = self.coords_of(rank)
        self.brick_lo = np.array([self._edge(a, self.coords[a]) for a in range(3)])
        self.brick_hi = np.array([self._edge(a, self.coords[a] + 1) for a in range(3)])
        for a in range(3):
            if self.grid[a] > 1 and (self.brick_hi[a] - self.brick_lo[a]) < 2 * self.margin:
                raise ValueError("brick thinner than twice the ghost margin")
        self.stages: list[_Stage] = []
        self.n_ghost = 0

    # ------------------------------------------------------------ geometry
    def _edge(self, axis: int, k: int) -> float:
        if k == self.grid[axis]:
            return float(self.hi[axis])
        return float(self.lo[axis] + self.L[axis] * k / self.grid[axis])

    def coords_of(self, rank: int) -> tuple:
        px, py, _ = self.grid
        return (rank % px, (rank // px) % py, rank // (px * py))

    def rank_of(self, c) -> int:
        px, py, _ = self.grid
        return int(c[0] + px * (c[1] + py * c[2]))

    def owner_of(self, pos: torch.Tensor) -> torch.Tensor:
        """Rank owning each position (positions wrapped into the box first)."""
        ranks = torch.zeros(pos.shape[0], dtype=torch.int64, device=pos.device)
        stride = 1
        for a in range(3):
            x = torch.remainder(pos[:, a] - float(self.lo[a]), float(self.L[a]))
            k = torch.clamp((x / float(self.L[a]) * self.grid[a]).floor().to(torch.int64), 0,
                            self.grid[a] - 1)
            # boundaries follow _edge exactly
            for kk in range(1, self.grid[a]):
                e = self._edge(a, kk) - float(self.lo[a])
                k = torch.where((x >= e) & (k < kk), torch.full_like(k, kk), k)
                k = torch.where((x < e) & (k >= kk), torch.full_like(k, kk - 1), k)
            ranks += k * stride
            stride *= self.grid[a]
        return ranks

    def local_box(self):
        from .domain import BoundaryKind, SimulationBox
        return SimulationBox(self.brick_lo, self.brick_hi, (BoundaryKind.REFLECTIVE,) * 3)

    # ---------------------------------------------------------- migration
    def migrate(self, state: torch.Tensor) -> torch.Tensor:
        """Send every row of ``state`` (N, k) float64 -- columns 0..2 are the
        positions -- to the rank owning its position; returns the rows this
        rank owns afterwards (received order: by source rank, then row)."""
        if self.nranks == 1:
            return state
        dest = self.owner_of(state[:, :3])
        order = torch.argsort(dest, stable=True)
        state = state[order]
        counts = torch.bincount(dest, minlength=self.nranks).to(torch.int64)
        dev = state.device
        if self._host_staged(state):
            state, counts = state.cpu(), counts.cpu()
        recv_counts = torch.empty_like(counts)
        dist.all_to_all_single(recv_counts, counts, group=self.group)
        out = torch.empty((int(recv_counts.sum()), state.shape[1]), dtype=state.dtype,
                          device=state.device)
        dist.all_to_all_single(out, state.contiguous(), recv_counts.tolist(), counts.tolist(),
                               group=self.group)
        return out.to(dev)

    # ------------------------------------------------------------ exchange
    def _neighbour(self, axis: int, direction: int) -> int:
        c = list(self.coords)
        c[axis] = (c[axis] + (1 if direction else -1)) % self.grid[axis]
        return self.rank_of(c)

    def _crosses(self, axis: int, direction: int) -> bool:
        """Sending through the face `direction` of this brick wraps the global box."""
        return (self.coords[axis] == 0 and direction == 0) or (
            self.coords[axis] == self.grid[axis] - 1 and direction == 1)

    def _host_staged(self, t: torch.Tensor) -> bool:
        """gloo moves CPU tensors only: device tensors go through host copies
        (used to run the multi-rank path on one GPU; NCCL moves them directly)."""
        return t.device.type == "cuda" and dist.get_backend(self.group) == "gloo"

    def _p2p(self, sends: list, recvs: list) -> None:
        """sends / recvs: lists of (peer, tensor), matched per peer in list
        order; issued as one batch (one NCCL group), so no ordering deadlock."""
        sends = [(p, t) for p, t in sends if t.numel()]
        recvs = [(p, t) for p, t in recvs if t.numel()]
        staged = any(self._host_staged(t) for _, t in sends + recvs)
        if staged:
            sends = [(p, t.cpu()) for p, t in sends]
            host_recvs = [(p, torch.empty(t.shape, dtype=t.dtype)) for p, t in recvs]
        else:
            host_recvs = recvs
        ops = [dist.P2POp(dist.irecv, t, peer, self.group) for peer, t in host_recvs]
        ops += [dist.P2POp(dist.isend, t, peer, self.group) for peer, t in sends]
        if not ops:
            return
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        if staged:
            for (_, dst), (_, src) in zip(recvs, host_recvs):
                dst.copy_(src)

    def plan(self, owned_pos: torch.Tensor) -> torch.Tensor:
        """Build the ghost layer for the current owned rows (N, k), columns
        0..2 the positions (further columns, e.g. ids, travel along).

        Returns the ghost rows (G, k); fixes the send lists so later
        ``exchange`` calls move the same particles."""
        dev = owned_pos.device
        pos = owned_pos
        self.stages = []
        for axis in range(3):
            st = _Stage(axis)
            blo, bhi = float(self.brick_lo[axis]), float(self.brick_hi[axis])
            x = pos[:, axis]
            sendbufs = []
            for direction in (0, 1):
                # domain.py:102-103 semantics against this brick's faces
                if direction == 0:
                    sel = (x - blo) < self.margin
                    shift = float(self.hi[axis] - self.lo[axis]) if self._crosses(axis, 0) else 0.0
                else:
                    sel = (bhi - x) < self.margin
                    shift = float(self.lo[axis] - self.hi[axis]) if self._crosses(axis, 1) else 0.0
                idx = torch.nonzero(sel).flatten()
                st.peer[direction] = self._neighbour(axis, direction)
                st.send_idx[direction] = idx
                st.shift[direction] = shift
                sendbufs.append(idx.numel())
            # counts: what I send toward `direction` arrives at the peer from
            # the opposite side; exchange counts with both peers
            counts_in = self._exchange_counts(st, sendbufs, dev)
            st.recv_count = counts_in
            self.stages.append(st)
            ghosts = self._stage_move(st, pos)
            pos = torch.cat([pos, ghosts])
        self.n_ghost = pos.shape[0] - owned_pos.shape[0]
        self._prepare_fast(owned_pos.shape[0], dev)
        return pos[owned_pos.shape[0]:]

    def _prepare_fast(self, n_owned: int, dev) -> None:
        """Persistent buffers for exchange_positions: int32 send lists, send
        buffers, and the row-major ghost block [stage 0 | stage 1 | stage 2]."""
        self._n_owned = n_owned
        self._ghost_rows = None
        if dev.type != "cuda":
            return
        self._ghost_rows = torch.empty((max(self.n_ghost, 1), 3), dtype=torch.float64,
                                       device=dev)
        off = 0
        for st in self.stages:
            st.idx32 = [st.send_idx[d].to(torch.int32).contiguous() for d in (0, 1)]
            local = self.nranks == 1 or self.grid[st.axis] == 1
            st.local = local
            if local:     # arrival order: my down-send, then my up-send
                c0, c1 = st.idx32[0].numel(), st.idx32[1].numel()
                st.dst = [self._ghost_rows[off:off + c0], self._ghost_rows[off + c0:off + c0 + c1]]
                off += c0 + c1
            else:         # arrival order: from the upper neighbour (slot 1), then the lower
                r1, r0 = st.recv_count[1], st.recv_count[0]
                st.recv = [self._ghost_rows[off + r1:off + r1 + r0], self._ghost_rows[off:off + r1]]
                st.sendbuf = [torch.empty((max(st.idx32[d].numel(), 1), 3), dtype=torch.float64,
                                          device=dev) for d in (0, 1)]
                off += r0 + r1

    def exchange_positions(self, x: torch.Tensor, y: torch.Tensor,
                           z: torch.Tensor) -> torch.Tensor:
        """``exchange`` for owned SoA positions on the device, without
        concatenations: one fused pack kernel per stage and direction
        (lmd_ghost_pack: gather + exact image shift), received blocks land in
        their slot of a persistent row-major ghost buffer (same order and
        values as ``exchange``).  Returns the (n_ghost, 3) ghost rows."""
        from . import _native as N
        g = self._ghost_rows
        s = N.stream()
        for st in self.stages:
            outs = st.dst if st.local else st.sendbuf
            for d in (0, 1):
                cnt = st.idx32[d].numel()
                if cnt:
                    N.call("lmd_ghost_pack", cnt, N.ptr(st.idx32[d]), self._n_owned, N.ptr(x),
                           N.ptr(y), N.ptr(z), N.ptr(g), st.axis, float(st.shift[d]),
                           N.ptr(outs[d]), s)
            if not st.local:
                sends = [(st.peer[0], st.sendbuf[0][:st.idx32[0].numel()]),
                         (st.peer[1], st.sendbuf[1][:st.idx32[1].numel()])]
                recvs = [(st.peer[0], st.recv[0]), (st.peer[1], st.recv[1])]
                self._pair_exchange(st, sends, recvs)
        return g[:self.n_ghost]

    def _exchange_counts(self, st: _Stage, sendcounts: list, dev) -> list:
        if self.nranks == 1 or self.grid[st.axis] == 1:
            # self-exchange: what I send down comes back to me from above
            return [sendcounts[1], sendcounts[0]]
        out = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(2)]
        sends = [(st.peer[d], torch.tensor([sendcounts[d]], dtype=torch.int64, device=dev))
                 for d in (0, 1)]
        # recv slot 0 = from the lower neighbour (its upward send), slot 1 = from the upper
        recvs = [(st.peer[0], out[0]), (st.peer[1], out[1])]
        self._pair_exchange(st, sends, recvs)
        return [int(out[0].item()), int(out[1].item())]

    def _pair_exchange(self, st: _Stage, sends, recvs) -> None:
        """With two bricks on an axis both neighbours are the same rank: order
        the messages so the k-th send matches the peer's k-th receive."""
        if st.peer[0] == st.peer[1]:
            # my send toward 0 (down) is the peer's arrival from its upper side
            # (slot 1) and vice versa; post recv slot 1 first to pair with the
            # peer's first send (toward 0)
            self._p2p([sends[0], sends[1]], [recvs[1], recvs[0]])
        else:
            self._p2p(sends, recvs)

    def _stage_move(self, st: _Stage, pos: torch.Tensor) -> torch.Tensor:
        a = st.axis
        packs = []
        for d in (0, 1):
            p = pos[st.send_idx[d]].clone()
            if st.shift[d] != 0.0:
                p[:, a] = p[:, a] + st.shift[d]
            packs.append(p.contiguous())
        if self.nranks == 1 or self.grid[a] == 1:
            # local periodic images: arrival order = (from above = my down-send, from below)
            return torch.cat([packs[0], packs[1]])
        dev = pos.device
        bufs = [torch.empty((st.recv_count[d], pos.shape[1]), dtype=pos.dtype, device=dev)
                for d in (0, 1)]
        sends = [(st.peer[0], packs[0]), (st.peer[1], packs[1])]
        recvs = [(st.peer[0], bufs[0]), (st.peer[1], bufs[1])]
        self._pair_exchange(st, sends, recvs)
        return torch.cat([bufs[1], bufs[0]])

    def exchange(self, owned_pos: torch.Tensor) -> torch.Tensor:
        """Move the planned ghost layer for new owned positions (same order as plan)."""
        pos = owned_pos
        for st in self.stages:
            ghosts = self._stage_move(st, pos)
            pos = torch.cat([pos, ghosts])
        return pos[owned_pos.shape[0]:]

    def allreduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        if self.nranks > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t
