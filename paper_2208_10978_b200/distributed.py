"""Multi-GPU state vector: global-qubit sharding with batched qubit-swap
relayouts.

The reference has no sharded state (SPEC.md:398 lists it as a non-goal; its
only parallelism is the fork pool of engine.py:169-199).  This module is the
B200 analogue: one process per GPU, ``torch.distributed`` (NCCL over NVLink /
NVSwitch) for the plumbing, the single-GPU engine (libqsv) for every local
pass.

Layout.  With P = 2^g ranks and n qubits, rank r holds the contiguous slice
of 2^(n-g) amplitudes whose *physical* index bits [n_local, n) equal r.  A
logical->physical qubit map ``perm`` says where each logical qubit lives;
physical positions >= n_local are global (rank bits).

Gates.  ``plan_segments`` walks the gate list and emits local segments (gates
whose qubits are all local, remapped to physical positions) separated by
relayouts, scheduling local-first inside the light cone: gates needing a
global qubit (and everything behind them on the same qubits) are deferred
while all other gates run, so one relayout serves many global-qubit gates --
the 20-layer brickwork needs ONE exchange at any P.  A relayout
first moves the evicted local qubits to the top k local positions with SWAP
gates (free inside the engine's tile passes: the planner folds permutations
into the shared-memory map), then swaps those k top local bits with k global
bits: every rank exchanges 2^k - 1 contiguous chunks of 2^(n_local-k)
amplitudes pairwise with its partners (in place, through a bounded staging
buffer).  The map is updated and never swapped back.

Expectation.  Strings whose flip avoids the global bits are evaluated on
every shard by the engine's batched sweep (a Z bit on a global position is a
per-rank sign).  The remaining strings are localised by further relayouts of
the state (logically read-only).  Per-rank partials are gathered and summed in
ascending rank order -- the reduction order of engine.py:199 -- so the energy
is deterministic and independent of P up to rounding.

Communicators: ``ProcessGroupComm`` (one shard per process; NCCL on GPUs,
gloo on CPU for tests) and ``LoopbackComm`` (all P shards in one process,
exchanges are device copies -- SURVEY.md 4's single-device loopback).  Local
compute goes through a ``LocalEngine``; ``CudaEngine`` is the product one.
"""

from __future__ import annotations

import ctypes
import hashlib
import math
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

K_SWAP = 4  # gate-kind code of SWAP (include/qsv.h)

# sharded plans keyed on (gate-list structure, qubit count, local qubits,
# qubit map): energy evaluations only refresh angles
_PLAN_CACHE: dict = {}


# ---------------------------------------------------------------------------
# local engine (product: libqsv on the process's GPU)
# ---------------------------------------------------------------------------


class CudaEngine:
    """Local shard operations on libqsv device states."""

    def __init__(self, device: int = 0):
        self.device = device

    def zeros(self, n_local: int):
        from . import statevector as sv

        import torch

        s = sv.StateVector._empty(n_local, self.device)
        self.tensor(s).zero_()
        # zero_ ran on torch's stream; libqsv works on the handle's own stream
        torch.cuda.current_stream(torch.device("cuda", self.device)).synchronize()
        return s

    def basis(self, n_local: int, index: int):
        from . import _lib
        from . import statevector as sv

        s = sv.StateVector._empty(n_local, self.device)
        _lib.check(_lib.lib().qsv_set_basis(s.handle, int(index)))
        return s

    def copy(self, shard):
        return shard.copy()

    def apply_gates(self, shard, kinds, qubits, values) -> None:
        from . import _lib

        if len(kinds) == 0:
            return
        _lib.check(_lib.lib().qsv_apply_gates(shard.handle, len(kinds), _lib.i32ptr(kinds),
                                              _lib.i32ptr(qubits), _lib.dptr(values), None))

    def expectation_terms(self, shard, x, y, z) -> np.ndarray:
        """Per-string Re<P_t> summed over this shard only."""
        from . import _lib

        S = len(x)
        per = np.zeros(S, dtype=np.float64)
        if S == 0:
            return per
        ones = np.ones(S, dtype=np.float64)
        zeros = np.zeros(S, dtype=np.float64)
        re, im = ctypes.c_double(), ctypes.c_double()
        _lib.check(_lib.lib().qsv_expectation(shard.handle, S, _lib.u64ptr(x), _lib.u64ptr(y),
                                              _lib.u64ptr(z), _lib.dptr(ones), _lib.dptr(zeros),
                                              ctypes.byref(re), ctypes.byref(im), _lib.dptr(per),
                                              None))
        return per

    def apply_rotations(self, shard, x, y, z, theta) -> None:
        """In place: prod_r exp(-i theta_r/2 P_r) (qsv_apply_pauli_rotations)."""
        from . import _lib

        if len(theta) == 0:
            return
        _lib.check(_lib.lib().qsv_apply_pauli_rotations(shard.handle, len(theta), _lib.u64ptr(x),
                                                        _lib.u64ptr(y), _lib.u64ptr(z),
                                                        _lib.dptr(theta), None))

    def apply_pauli(self, src, dst, x: int, y: int, z: int) -> None:
        """dst = P src (kernels.apply_pauli, _cykernels.pyx:76-102)."""
        from . import _lib

        _lib.check(_lib.lib().qsv_apply_pauli(src.handle, dst.handle, int(x), int(y), int(z)))

    def vdot(self, a, b) -> complex:
        from . import statevector as sv

        return sv.vdot(a, b)

    def tensor(self, shard):
        """Zero-copy torch view (2^n_local, 2) float64 of the shard."""
        import torch

        return torch.as_tensor(shard, device=f"cuda:{self.device}")

    def synchronize(self, shard) -> None:
        shard.synchronize()

    def download(self, shard) -> np.ndarray:
        return shard.amplitudes


# CUDA IPC unavailable here (a rank could not export or map a shard): every
# later relayout takes the NCCL path (all ranks see the same failure report)
_IPC_BROKEN = False


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------


class LoopbackComm:
    """All P shards live in this process; exchanges are device copies."""

    def __init__(self, world: int, piece_bytes: int = 256 << 20):
        if world < 1 or world & (world - 1):
            raise ValueError("world size must be a power of two")
        self.world = world
        self.owned = list(range(world))
        self.piece_bytes = piece_bytes

    def gather_partials(self, partials: dict) -> list:
        return [partials[r] for r in range(self.world)]

    def gather_arrays(self, arrays: dict) -> list:
        return [arrays[r] for r in range(self.world)]

    def barrier(self) -> None:
        pass


class ProcessGroupComm:
    """One shard per process over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None, piece_bytes: int = 256 << 20):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        if self.world & (self.world - 1):
            raise ValueError("world size must be a power of two")
        self.rank = dist.get_rank(group)
        self.owned = [self.rank]
        self.piece_bytes = piece_bytes
        # gloo moves host tensors only: device shards are staged through host
        # memory (tests of the process-group plumbing on a single GPU)
        self.nccl = dist.get_backend(group) == "nccl"

    def _device(self, like):
        return like.device

    def gather_partials(self, partials: dict) -> list:
        import torch

        v = partials[self.rank]
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor(v, dtype=torch.float64, device=dev).reshape(-1)
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [o.cpu().numpy() for o in out]

    def gather_arrays(self, arrays: dict) -> list:
        out = [None] * self.world
        self.dist.all_gather_object(out, arrays[self.rank], group=self.group)
        return out

    def barrier(self) -> None:
        self.dist.barrier(group=self.group)


# ---------------------------------------------------------------------------
# planner (pure host logic, identical on every rank)
# ---------------------------------------------------------------------------


@dataclass
class Relayout:
    """Swap the top k local physical bits with global bits S[0..k-1]
    (rank-bit indices): top local bit n_local - k + i <-> global bit S[i]."""
    S: tuple[int, ...]

    @property
    def k(self) -> int:
        return len(self.S)


@dataclass
class Segment:
    src: np.ndarray        # source gate index per local gate (-1: inserted SWAP)
    qubits: np.ndarray     # int32 [2 * L] physical local qubits
    relayout: Optional[Relayout]


def _gate_qubits(qubits, i):
    a, b = int(qubits[2 * i]), int(qubits[2 * i + 1])
    return (a,) if b < 0 else (a, b)


def _apply_relayout_to_map(perm, inv, bring, victims, n_local):
    k = len(bring)
    for j in range(k):
        b, v = bring[j], victims[j]
        T = n_local - k + j
        Gp = perm[b]
        perm[b], perm[v] = T, Gp
        inv[T], inv[Gp] = b, v


def _move_victims(perm, inv, victims, n_local, swaps):
    """SWAP gates (physical) bringing victims[j] to position n_local - k + j."""
    k = len(victims)
    for j, v in enumerate(victims):
        T = n_local - k + j
        p = perm[v]
        if p != T:
            other = inv[T]
            swaps.append((p, T))
            perm[v], perm[other] = T, p
            inv[T], inv[p] = v, other


def plan_segments(kinds, qubits, n: int, n_local: int, perm):
    """Split a gate list into local segments and relayouts.
    Returns (segments, final_perm).

    Local-first light-cone scheduling: a gate that needs a global qubit is
    deferred, and so is every later gate sharing a qubit with a deferred one;
    all other gates run now (gates on disjoint qubits commute).  Only when
    every remaining gate is blocked does a relayout happen, bringing in the
    global qubits the deferred gates need first (up to g) and evicting the
    local qubits used latest among the remaining gates.  On a brickwork the
    local qubits run many layers ahead inside the light cone before an
    exchange is needed."""
    g = n - n_local
    perm = list(perm)
    inv = [0] * n
    for q, p in enumerate(perm):
        inv[p] = q
    segs = []
    src, qs = [], []
    remaining = list(range(len(kinds)))
    while True:
        blocked = set()
        deferred = []
        for i in remaining:
            gq = _gate_qubits(qubits, i)
            if any(q in blocked for q in gq) or any(perm[q] >= n_local for q in gq):
                deferred.append(i)
                blocked.update(gq)
            else:
                src.append(i)
                qs.extend([perm[gq[0]], perm[gq[1]] if len(gq) == 2 else -1])
        remaining = deferred
        if not remaining:
            break
        # global qubits in order of first use by the deferred gates
        bring = []
        first_use = {}
        for pos, i in enumerate(remaining):
            for q in _gate_qubits(qubits, i):
                first_use.setdefault(q, pos)
                if perm[q] >= n_local and q not in bring and len(bring) < g:
                    bring.append(q)
        head = set(_gate_qubits(qubits, remaining[0]))
        cand = sorted((inv[p] for p in range(n_local) if inv[p] not in head and inv[p] not in bring),
                      key=lambda q: (-first_use.get(q, math.inf), q))
        if len(cand) < len(bring):
            raise ValueError("too few local qubits for a relayout")
        victims = cand[:len(bring)]
        swaps = []
        _move_victims(perm, inv, victims, n_local, swaps)
        for a, b in swaps:
            src.append(-1)
            qs.extend([a, b])
        S = tuple(perm[b] - n_local for b in bring)
        segs.append(Segment(np.array(src, dtype=np.int64), np.array(qs, dtype=np.int32),
                            Relayout(S)))
        _apply_relayout_to_map(perm, inv, bring, victims, n_local)
        src, qs = [], []
    segs.append(Segment(np.array(src, dtype=np.int64), np.array(qs, dtype=np.int32), None))
    return segs, perm


@dataclass
class UnitSegment:
    """Local work between relayouts: entries in order, each either
    ("g", gate index or -1 for an inserted SWAP, q0, q1) with physical local
    qubits, or ("r", x, y, z, zg, rz) -- a direct Pauli rotation with local
    physical masks x/y/z, global Z bits zg (a per-rank sign of the angle) and
    the gate index whose bound value is its angle."""
    entries: list
    relayout: Optional[Relayout]


def _bits(mask: int):
    while mask:
        low = mask & -mask
        yield low.bit_length() - 1
        mask ^= low


def plan_units(kinds, qubits, n: int, n_local: int, perm, spans, masks):
    """Light-cone scheduling over units: recognised pauli_evolution blocks are
    ONE unit each (exp(-i theta/2 P)), other gates are units of their own.  A
    rotation is local when its flip (x|y) avoids the global qubits -- Z on a
    global qubit is a per-rank sign of the angle -- so a UCC circuit's CNOT
    ladders through global qubits no longer force exchanges.  A unit runs now
    when it is local and commutes with every deferred unit (rotations:
    symplectic product; otherwise disjoint support).  Returns (segments, perm)."""
    g = n - n_local
    perm = list(perm)
    inv = [0] * n
    for q, p in enumerate(perm):
        inv[p] = q
    units = []  # (kind, a, b, supp, flip, x, y, z)
    G = len(kinds)
    span_at = {int(st): k for k, st in enumerate(spans[:, 0])} if len(spans) else {}
    i = 0
    while i < G:
        k = span_at.get(i)
        if k is not None:
            x, y, z = (int(v) for v in masks[k])
            units.append(("r", int(spans[k, 2]), 0, x | y | z, x | y, x, y, z))
            i += int(spans[k, 1])
            continue
        gq = _gate_qubits(qubits, i)
        sm = 0
        for q in gq:
            sm |= 1 << q
        units.append(("g", i, 0, sm, 0, 0, 0, 0))
        i += 1

    def needs(u):
        return u[4] if u[0] == "r" else u[3]

    def anti(a, b):
        ax, az = a[5] | a[6], a[6] | a[7]
        bx, bz = b[5] | b[6], b[6] | b[7]
        return (bin(ax & bz).count("1") + bin(az & bx).count("1")) & 1

    def conflict(a, b):
        if not (a[3] & b[3]):
            return False
        if a[0] == "r" and b[0] == "r":
            return bool(anti(a, b))
        return True

    def phys(mask):
        out = 0
        for q in _bits(mask):
            out |= 1 << perm[q]
        return out

    lmask = (1 << n_local) - 1
    segs = []
    entries = []
    remaining = list(range(len(units)))
    while True:
        deferred = []
        dunion = 0
        for ui in remaining:
            u = units[ui]
            local = (phys(needs(u)) >> n_local) == 0
            ok = local
            if ok and (u[3] & dunion):
                for dj in deferred:
                    if conflict(units[dj], u):
                        ok = False
                        break
            if ok:
                if u[0] == "g":
                    gq = _gate_qubits(qubits, u[1])
                    entries.append(("g", u[1], perm[gq[0]], perm[gq[1]] if len(gq) == 2 else -1))
                else:
                    px, py, pz = phys(u[5]), phys(u[6]), phys(u[7])
                    entries.append(("r", px & lmask, py & lmask, pz & lmask, pz >> n_local, u[1]))
            else:
                deferred.append(ui)
                dunion |= u[3]
        remaining = deferred
        if not remaining:
            break
        # bring in the global qubits the deferred units need, head first
        bring, first_use = [], {}
        for pos, ui in enumerate(remaining):
            for q in _bits(needs(units[ui])):
                first_use.setdefault(q, pos)
                if perm[q] >= n_local and q not in bring and len(bring) < g:
                    bring.append(q)
        head = set(_bits(needs(units[remaining[0]])))
        cand = sorted((inv[p] for p in range(n_local) if inv[p] not in head and inv[p] not in bring),
                      key=lambda q: (-first_use.get(q, math.inf), q))
        if len(cand) < len(bring):
            raise ValueError("too few local qubits for a relayout")
        victims = cand[:len(bring)]
        swaps = []
        _move_victims(perm, inv, victims, n_local, swaps)
        for a, b in swaps:
            entries.append(("g", -1, a, b))
        S = tuple(perm[b] - n_local for b in bring)
        segs.append(UnitSegment(entries, Relayout(S)))
        _apply_relayout_to_map(perm, inv, bring, victims, n_local)
        entries = []
    segs.append(UnitSegment(entries, None))
    return segs, perm


def plan_localize(flips: list[int], n: int, n_local: int, perm):
    """Relayout that makes flips[0] (logical mask) local, evicting the local
    qubits least used by the other flips.  Returns (swaps, Relayout, new perm)."""
    perm = list(perm)
    inv = [0] * n
    for q, p in enumerate(perm):
        inv[p] = q
    f0 = flips[0]
    bring = [q for q in range(n) if (f0 >> q) & 1 and perm[q] >= n_local]
    freq = [0] * n
    for f in flips:
        for q in range(n):
            if (f >> q) & 1:
                freq[q] += 1
    cand = sorted((inv[p] for p in range(n_local) if not (f0 >> inv[p]) & 1),
                  key=lambda q: (freq[q], q))
    if len(cand) < len(bring):
        raise ValueError("Pauli string wider than the local qubits of a shard")
    victims = cand[:len(bring)]
    swaps = []
    _move_victims(perm, inv, victims, n_local, swaps)
    S = tuple(perm[b] - n_local for b in bring)
    _apply_relayout_to_map(perm, inv, bring, victims, n_local)
    return swaps, Relayout(S), perm


def plan_align(perm, target, n: int, n_local: int):
    """Steps turning the physical layout `perm` into `target`: at most two
    relayouts (evict the mismatched global qubits to local positions that
    stay local, then bring the target's global qubits in) and local SWAP
    gates (free: folded into the tile maps).  Returns a list of
    ("swaps", [(p, q), ...]) / ("relayout", Relayout) steps."""
    perm = list(perm)
    inv = [0] * n
    for q, p in enumerate(perm):
        inv[p] = q
    tinv = [0] * n
    for q, p in enumerate(target):
        tinv[p] = q
    g = n - n_local
    steps = []
    W = [i for i in range(g) if inv[n_local + i] != tinv[n_local + i]]
    if W:
        want = [tinv[n_local + i] for i in W]
        if any(perm[q] >= n_local for q in want):
            # 1) the rank bits W take local qubits that are not global in target
            tglob = {tinv[n_local + i] for i in range(g)}
            cand = [inv[p] for p in range(n_local) if inv[p] not in tglob]
            if len(cand) < len(W):
                raise ValueError("too few local qubits to realign the shards")
            bring, victims = [inv[n_local + i] for i in W], cand[:len(W)]
            swaps = []
            _move_victims(perm, inv, victims, n_local, swaps)
            S = tuple(perm[b] - n_local for b in bring)
            _apply_relayout_to_map(perm, inv, bring, victims, n_local)
            steps += [("swaps", swaps), ("relayout", Relayout(S))]
        # 2) every target global qubit is local now: swap them into W
        bring, victims = [inv[n_local + i] for i in W], want
        swaps = []
        _move_victims(perm, inv, victims, n_local, swaps)
        S = tuple(perm[b] - n_local for b in bring)
        _apply_relayout_to_map(perm, inv, bring, victims, n_local)
        steps += [("swaps", swaps), ("relayout", Relayout(S))]
    # 3) local positions
    swaps = []
    for p in range(n_local):
        q = tinv[p]
        if inv[p] != q:
            cur = perm[q]
            other = inv[p]
            swaps.append((p, cur))
            perm[q], perm[other] = p, cur
            inv[p], inv[cur] = q, other
    steps.append(("swaps", swaps))
    assert perm == list(target)
    return steps


# ---------------------------------------------------------------------------
# the distributed state
# ---------------------------------------------------------------------------


def _log2(p: int) -> int:
    g = p.bit_length() - 1
    if p < 1 or (1 << g) != p:
        raise ValueError("world size must be a power of two")
    return g


class DistStateVector:
    """Logical n-qubit state sharded over comm.world ranks."""

    def __init__(self, n_qubits: int, comm, engine, shards: Optional[dict], perm,
                 basis: Optional[int] = None):
        self.n_qubits = n_qubits
        self.comm = comm
        self.engine = engine
        self.g = _log2(comm.world)
        self.n_local = n_qubits - self.g
        self._shards = shards
        self._basis = basis  # lazy |basis>: no device memory until first needed
        self.perm = list(perm)
        self.stats = {"relayouts": 0, "relayout_bytes_sent": 0, "relayout_seconds": 0.0}

    # -- construction --------------------------------------------------------
    @classmethod
    def basis(cls, n_qubits: int, index: int, comm, engine) -> "DistStateVector":
        """|index> kept as an index: evolve materialises it straight into its
        output shards (one shard per GPU, never a copy -- at config 5 a shard
        is 128 GiB of a 180 GB B200)."""
        g = _log2(comm.world)
        if n_qubits - g < 1:
            raise ValueError("more ranks than amplitudes per shard allow")
        return cls(n_qubits, comm, engine, None, range(n_qubits), basis=index)

    def _materialize_basis(self, index: int) -> dict:
        n_local = self.n_local
        owner, local = index >> n_local, index & ((1 << n_local) - 1)
        return {r: (self.engine.basis(n_local, local) if r == owner else self.engine.zeros(n_local))
                for r in self.comm.owned}

    @property
    def shards(self) -> dict:
        if self._shards is None:
            self._shards = self._materialize_basis(self._basis)
            self._basis = None
        return self._shards

    @property
    def basis_index(self) -> Optional[int]:
        return self._basis if self._shards is None else None

    def copy(self) -> "DistStateVector":
        if self._shards is None:
            return DistStateVector(self.n_qubits, self.comm, self.engine, None, self.perm,
                                   basis=self._basis)
        out = DistStateVector(self.n_qubits, self.comm, self.engine,
                              {r: self.engine.copy(s) for r, s in self.shards.items()}, self.perm)
        return out

    def fresh_from_basis(self) -> "DistStateVector":
        """Output state of an evolve of this lazy basis state: its own shards
        (the input stays a lazy index -- statevector.py:71's copy without
        the second state)."""
        out = DistStateVector(self.n_qubits, self.comm, self.engine, None, self.perm,
                              basis=self._basis)
        out.shards  # noqa: B018  (materialise)
        return out

    # -- exchange ------------------------------------------------------------
    def _relayout(self, rl: Relayout) -> None:
        """Swap the top k local bits with global bits rl.S, pairwise in place."""
        import time

        k = rl.k
        if k == 0:
            return
        t0 = time.perf_counter()
        n_local = self.n_local
        chunk = 1 << (n_local - k)
        views = {}
        for r, s in self.shards.items():
            self.engine.synchronize(s)
            views[r] = self.engine.tensor(s)

        def s_value(r):
            return sum(((r >> rl.S[i]) & 1) << i for i in range(k))

        def partner(r, c):
            p = r
            for i in range(k):
                p = (p & ~(1 << rl.S[i])) | (((c >> i) & 1) << rl.S[i])
            return p

        remote = {}
        for r in self.comm.owned:
            rs = s_value(r)
            for c in range(1 << k):
                if c == rs:
                    continue
                p = partner(r, c)
                # (r, chunk c) <-> (p, chunk rs)
                if p in views:
                    if r < p:
                        self._swap_local(views[r], views[p], c * chunk, rs * chunk, chunk)
                else:
                    remote.setdefault(r, []).append((c, p))
        if remote and not (self._ipc_enabled() and self._ipc_exchange(remote, chunk, s_value)):
            self._p2p_exchange(views, remote, chunk)
        self._sync_after(views)
        self.stats["relayouts"] += 1
        self.stats["relayout_bytes_sent"] += 16 * (((1 << k) - 1) * chunk)  # per rank
        self.stats["relayout_seconds"] += time.perf_counter() - t0

    def _swap_local(self, ta, tb, oa: int, ob: int, chunk: int) -> None:
        """Swap ta[oa:oa+chunk] <-> tb[ob:ob+chunk] (both shards in this
        process) through one bounded staging piece, never a chunk-sized
        temporary (a chunk can be half of a 128 GiB shard)."""
        row_bytes = ta.element_size() * (ta.shape[1] if ta.dim() > 1 else 1)
        piece = max(1, min(chunk, self.comm_piece_bytes() // row_bytes))
        tmp = ta.new_empty((piece,) + tuple(ta.shape[1:]))
        for off in range(0, chunk, piece):
            w = min(piece, chunk - off)
            a = ta[oa + off:oa + off + w]
            b = tb[ob + off:ob + off + w]
            tmp[:w].copy_(a)
            a.copy_(b)
            b.copy_(tmp[:w])

    def comm_piece_bytes(self) -> int:
        return int(getattr(self.comm, "piece_bytes", 256 << 20))

    def _ipc_enabled(self) -> bool:
        """Device shards in several processes of one node: swap chunks in
        place over peer memory (CUDA IPC + swap kernel) instead of NCCL
        send/recv through staging.  QSV_DIST_IPC=0 keeps the NCCL path."""
        return (isinstance(self.engine, CudaEngine) and isinstance(self.comm, ProcessGroupComm)
                and os.environ.get("QSV_DIST_IPC", "1") != "0" and not _IPC_BROKEN)

    def _ipc_exchange(self, remote, chunk, s_value) -> bool:
        """Pairwise in-place chunk swap over peer memory: every rank exports
        its shard (qsv_ipc_get_handle), maps its partners' (qsv_ipc_open, for
        this exchange only) and swaps its half of each pair with the swap kernel
        (qsv_swap_peer: the lower rank the first half, the higher the second),
        so each byte is read and written once per side with no staging copy
        and both directions of every link busy.  Ordering: every rank drains
        its stream and meets the others at a barrier before any swap, and
        again after its own swaps -- no kernel ever waits on another rank.
        Every rank reports whether it could export and map; if any could not
        (no IPC in this environment), all return False before touching data
        and the caller takes the NCCL path."""
        from . import _lib

        global _IPC_BROKEN
        r = self.comm.rank
        shard = self.shards[r]
        L = _lib.lib()
        dev = self.engine.device
        h = (ctypes.c_char * 64)()
        ok = L.qsv_ipc_get_handle(shard.handle, h) == 0
        handles = self.comm.gather_arrays({r: bytes(h) if ok else None})
        if any(x is None for x in handles):
            _IPC_BROKEN = True
            return False
        mapped = {}
        try:
            # (test hook: QSV_DIST_IPC_FAIL=<rank> makes that rank's mapping fail)
            fail_here = os.environ.get("QSV_DIST_IPC_FAIL") == str(r)
            for c, p in remote[r]:
                ptr = ctypes.c_void_p()
                if fail_here or L.qsv_ipc_open(dev, handles[p], ctypes.byref(ptr)) != 0:
                    ok = False
                    break
                mapped[p] = ptr
            if not all(self.comm.gather_arrays({r: ok})):
                _IPC_BROKEN = True
                return False
            shard.synchronize()
            self.comm.barrier()  # every shard's earlier work is done
            rs = s_value(r)
            half = chunk // 2
            for c, p in remote[r]:
                off, ln = (0, half) if p > r else (half, chunk - half)
                _lib.check(L.qsv_swap_peer(shard.handle, c * chunk + off, mapped[p], rs * chunk + off, ln))
                self.stats["ipc_swaps"] = self.stats.get("ipc_swaps", 0) + 1
            shard.synchronize()
        finally:
            # a mapping pins the partner's allocation: unmap before the
            # partner may free its shard (128 GiB at config 5)
            for ptr in mapped.values():
                L.qsv_ipc_close(dev, ptr)
        self.comm.barrier()  # every half of every pair is swapped
        return True

    def _p2p_exchange(self, views, remote, chunk):
        """Pairwise chunk swap with the remote partners, one bounded piece at
        a time: send piece k of the outgoing chunk and receive the partner's
        piece k into a staging slot in the same group, then copy it into place
        (an in-place swap needs the slot: a receive into the piece being sent
        in the same round would race, and a receive posted a round later
        deadlocks the paired sends).  With NCCL, ``wait()`` only orders the
        CUDA stream -- the host does not block per piece."""
        import torch

        dist = self.comm.dist
        group = self.comm.group
        for r, lst in remote.items():
            t = views[r]
            row_bytes = t.element_size() * (t.shape[1] if t.dim() > 1 else 1)
            piece = max(1, min(chunk, self.comm.piece_bytes // row_bytes))
            staging = torch.empty((len(lst), piece) + tuple(t.shape[1:]), dtype=t.dtype,
                                  device=t.device)
            host = t.is_cuda and not self.comm.nccl
            if host:
                staging = staging.cpu()
            for off in range(0, chunk, piece):
                w = min(piece, chunk - off)
                ops = []
                for j, (c, p) in enumerate(lst):
                    src = t[c * chunk + off: c * chunk + off + w]
                    src = src.cpu() if host else src.contiguous()
                    ops.append(dist.P2POp(dist.isend, src, p, group))
                    ops.append(dist.P2POp(dist.irecv, staging[j, :w], p, group))
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
                for j, (c, p) in enumerate(lst):
                    t[c * chunk + off: c * chunk + off + w].copy_(staging[j, :w])

    def _sync_after(self, views):
        import torch

        for t in views.values():
            if t.is_cuda:
                torch.cuda.current_stream(t.device).synchronize()
                break

    # -- gates ---------------------------------------------------------------
    def apply_flat(self, kinds, qubits, values) -> None:
        """Apply a flattened bound gate list (logical qubits) in place."""
        key = (hashlib.blake2b(kinds.tobytes() + qubits.tobytes(), digest_size=16).digest(),
               self.n_qubits, self.n_local, tuple(self.perm))
        plan = _PLAN_CACHE.get(key)
        if plan is None:
            from . import _lib

            spans, masks = _lib.match_rotations(self.n_qubits, kinds, qubits)
            if len(spans):
                plan = ("units",) + plan_units(kinds, qubits, self.n_qubits, self.n_local, self.perm,
                                               spans, masks)
            else:
                plan = ("gates",) + plan_segments(kinds, qubits, self.n_qubits, self.n_local, self.perm)
            if len(_PLAN_CACHE) >= 16:
                _PLAN_CACHE.pop(next(iter(_PLAN_CACHE)))
            _PLAN_CACHE[key] = plan
        if plan[0] == "units":
            self._apply_units(kinds, qubits, values, plan[1], plan[2])
            return
        segs, perm = plan[1], plan[2]
        for seg in segs:
            L = len(seg.src)
            if L:
                sk = np.empty(L, dtype=np.int32)
                sv_ = np.zeros(3 * L, dtype=np.float64)
                for j, i in enumerate(seg.src):
                    if i < 0:
                        sk[j] = K_SWAP
                    else:
                        sk[j] = kinds[i]
                        sv_[3 * j:3 * j + 3] = values[3 * i:3 * i + 3]
                for r in self.comm.owned:
                    self.engine.apply_gates(self.shards[r], sk, seg.qubits, sv_)
            if seg.relayout is not None:
                self._relayout(seg.relayout)
        self.perm = perm

    def _apply_units(self, kinds, qubits, values, segs, perm) -> None:
        for seg in segs:
            k = 0
            E = seg.entries
            while k < len(E):
                j = k
                while j < len(E) and E[j][0] == E[k][0]:
                    j += 1
                run = E[k:j]
                if E[k][0] == "g":
                    L = len(run)
                    sk = np.empty(L, dtype=np.int32)
                    sq = np.empty(2 * L, dtype=np.int32)
                    sv_ = np.zeros(3 * L, dtype=np.float64)
                    for t, (_, gi, a, b) in enumerate(run):
                        sq[2 * t], sq[2 * t + 1] = a, b
                        if gi < 0:
                            sk[t] = K_SWAP
                        else:
                            sk[t] = kinds[gi]
                            sv_[3 * t:3 * t + 3] = values[3 * gi:3 * gi + 3]
                    for r in self.comm.owned:
                        self.engine.apply_gates(self.shards[r], sk, sq, sv_)
                else:
                    x = np.array([e[1] for e in run], dtype=np.uint64)
                    y = np.array([e[2] for e in run], dtype=np.uint64)
                    z = np.array([e[3] for e in run], dtype=np.uint64)
                    zg = [e[4] for e in run]
                    th = np.array([values[3 * e[5]] for e in run], dtype=np.float64)
                    for r in self.comm.owned:
                        sign = np.array([-1.0 if bin(m & r).count("1") & 1 else 1.0 for m in zg])
                        self.engine.apply_rotations(self.shards[r], x, y, z, th * sign)
                k = j
            if seg.relayout is not None:
                self._relayout(seg.relayout)
        self.perm = perm

    def _apply_swaps(self, swaps) -> None:
        if not swaps:
            return
        L = len(swaps)
        sk = np.full(L, K_SWAP, dtype=np.int32)
        sq = np.array([q for ab in swaps for q in ab], dtype=np.int32)
        sv_ = np.zeros(3 * L, dtype=np.float64)
        for r in self.comm.owned:
            self.engine.apply_gates(self.shards[r], sk, sq, sv_)

    # -- expectation ---------------------------------------------------------
    def _phys(self, mask: int) -> int:
        out = 0
        for q in range(self.n_qubits):
            if (mask >> q) & 1:
                out |= 1 << self.perm[q]
        return out

    def expectation_terms(self, x, y, z, cr, ci) -> tuple[float, float]:
        """(Re, Im) of sum_t c_t <P_t>, reduced over ranks in ascending order."""
        S = len(cr)
        lmask = (1 << self.n_local) - 1
        part = {r: np.zeros(2) for r in self.comm.owned}
        wide = [t for t in range(S) if bin(int(x[t]) | int(y[t])).count("1") > self.n_local]
        if wide:
            self._pairwise_terms(wide, x, y, z, cr, ci, part)
        wset = set(wide)
        remaining = [t for t in range(S) if t not in wset]
        while remaining:
            px = [self._phys(int(x[t])) for t in remaining]
            py = [self._phys(int(y[t])) for t in remaining]
            pz = [self._phys(int(z[t])) for t in remaining]
            loc = [j for j in range(len(remaining)) if ((px[j] | py[j]) >> self.n_local) == 0]
            if loc:
                lx = np.array([px[j] & lmask for j in loc], dtype=np.uint64)
                ly = np.array([py[j] & lmask for j in loc], dtype=np.uint64)
                lz = np.array([pz[j] & lmask for j in loc], dtype=np.uint64)
                gz = [pz[j] >> self.n_local for j in loc]
                c_re = np.array([cr[remaining[j]] for j in loc])
                c_im = np.array([ci[remaining[j]] for j in loc])
                for r in self.comm.owned:
                    per = self.engine.expectation_terms(self.shards[r], lx, ly, lz)
                    sign = np.array([-1.0 if bin(gzj & r).count("1") & 1 else 1.0 for gzj in gz])
                    v = per * sign
                    part[r][0] += float(np.dot(c_re, v))
                    part[r][1] += float(np.dot(c_im, v))
            keep = set(loc)
            remaining = [remaining[j] for j in range(len(remaining)) if j not in keep]
            if remaining:
                flips = [int(x[t]) | int(y[t]) for t in remaining]
                swaps, rl, perm = plan_localize(flips, self.n_qubits, self.n_local, self.perm)
                self._apply_swaps(swaps)
                self._relayout(rl)
                self.perm = perm
        parts = self.comm.gather_partials({r: part[r] for r in self.comm.owned})
        re = 0.0
        im = 0.0
        for p in parts:  # ascending rank order (engine.py:199)
            re += float(p[0])
            im += float(p[1])
        return re, im


    def _pairwise_terms(self, terms, x, y, z, cr, ci, part) -> None:
        """Strings wider than a shard's local qubits: for each global flip
        pattern fg, every rank r fetches the shard of r ^ fg and evaluates
        sum_j conj(psi_j) (P psi)_j over its own slice (one pairwise shard
        exchange per pattern)."""
        n_local = self.n_local
        lmask = (1 << n_local) - 1
        by_fg = {}
        for t in terms:
            px, py, pz = self._phys(int(x[t])), self._phys(int(y[t])), self._phys(int(z[t]))
            by_fg.setdefault((px | py) >> n_local, []).append((t, px, py, pz))
        for fg in sorted(by_fg):
            partners = self._fetch_partners(fg)
            scratch = {r: self.engine.zeros(n_local) for r in self.comm.owned}
            for t, px, py, pz in by_fg[fg]:
                yg = py >> n_local
                yzg = (py | pz) >> n_local
                ph = (1j) ** (bin(yg).count("1") & 3)
                c = complex(cr[t], ci[t])
                for r in self.comm.owned:
                    p = r ^ fg
                    sg = -1.0 if bin(p & yzg).count("1") & 1 else 1.0
                    self.engine.apply_pauli(partners[r], scratch[r], px & lmask, py & lmask,
                                            pz & lmask)
                    v = c * ph * sg * self.engine.vdot(self.shards[r], scratch[r])
                    part[r][0] += v.real
                    part[r][1] += v.imag

    def _fetch_partners(self, fg: int) -> dict:
        """{r: copy of rank (r ^ fg)'s shard} for every owned rank r."""
        out = {}
        remote = []
        for r in self.comm.owned:
            p = r ^ fg
            if p in self.shards:
                out[r] = self.shards[p]
            else:
                remote.append((r, p))
        if remote:
            import torch

            dist = self.comm.dist
            for r, p in remote:
                buf = self.engine.zeros(self.n_local)
                self.engine.synchronize(self.shards[r])
                mine = self.engine.tensor(self.shards[r])
                theirs = self.engine.tensor(buf)
                host = mine.is_cuda and not self.comm.nccl
                snd = mine.cpu() if host else mine
                rcv = torch.empty_like(snd) if host else theirs
                ops = [dist.P2POp(dist.isend, snd, p, self.comm.group),
                       dist.P2POp(dist.irecv, rcv, p, self.comm.group)]
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
                if host:
                    theirs.copy_(rcv)
                if theirs.is_cuda:
                    torch.cuda.current_stream(theirs.device).synchronize()
                out[r] = buf
        return out

    def align_to(self, target) -> None:
        """Re-layout this state (logically unchanged) to the physical qubit
        map `target`."""
        if list(target) == self.perm:
            return
        for kind, step in plan_align(self.perm, target, self.n_qubits, self.n_local):
            if kind == "swaps":
                self._apply_swaps(step)
            else:
                self._relayout(step)
        self.perm = list(target)

    def overlap(self, other: "DistStateVector") -> complex:
        """<self|other> = sum_j conj(self_j) other_j (engine.py:74-75): other
        is realigned to self's layout, then per-shard dot products are summed
        in ascending rank order."""
        if other.n_qubits != self.n_qubits:
            raise ValueError("state qubit counts differ")
        if self.basis_index is not None and other.basis_index is not None:
            return complex(1.0 if self.basis_index == other.basis_index else 0.0)
        other.align_to(self.perm)
        part = {}
        for r in self.comm.owned:
            v = self.engine.vdot(self.shards[r], other.shards[r])
            part[r] = np.array([v.real, v.imag])
        re = im = 0.0
        for p in self.comm.gather_partials(part):
            re += float(p[0])
            im += float(p[1])
        return complex(re, im)

    # -- host view -------------------------------------------------------------
    def amplitudes(self) -> np.ndarray:
        """Logical amplitude vector on the host (small states; test helper)."""
        arrays = self.comm.gather_arrays({r: self.engine.download(self.shards[r])
                                          for r in self.comm.owned})
        phys = np.concatenate([np.asarray(a) for a in arrays])
        n = self.n_qubits
        idx = np.arange(1 << n, dtype=np.int64)
        pidx = np.zeros_like(idx)
        for q in range(n):
            pidx |= ((idx >> q) & 1) << self.perm[q]
        return phys[pidx]


# ---------------------------------------------------------------------------
# reference-shaped API
# ---------------------------------------------------------------------------


def init_state(bitstring: str, comm, engine=None) -> DistStateVector:
    """init_state (statevector.py:42-54) on a sharded state."""
    n = len(bitstring)
    if n == 0 or any(c not in "01" for c in bitstring):
        raise ValueError(f"invalid bitstring {bitstring!r}")
    index = sum(1 << k for k, c in enumerate(bitstring) if c == "1")
    return DistStateVector.basis(n, index, comm, engine or CudaEngine())


def evolve(s: DistStateVector, c) -> DistStateVector:
    """evolve (statevector.py:65-74): new sharded state, input untouched."""
    from .circuit import flatten_bound

    if c.n_qubits != s.n_qubits:
        raise ValueError("circuit and state qubit counts differ")
    flat = flatten_bound(c)  # RuntimeError if unbound (statevector.py:69-70)
    out = s.fresh_from_basis() if s.basis_index is not None else s.copy()
    out.apply_flat(*flat)
    return out


def expectation(s: DistStateVector, h) -> float:
    """expectation (statevector.py:98-110) over the shards."""
    from .pauli import term_arrays

    if not h.is_hermitian():
        raise ValueError("expectation requires a Hermitian operator (real coefficients)")
    x, y, z, cr, ci = term_arrays(h, s.n_qubits)
    re, im = s.expectation_terms(x, y, z, cr, ci)
    if abs(im) > 1e-10:
        raise ArithmeticError(f"expectation has imaginary residue {im:.3e}")
    return re


class DistributedBackend:
    """Backend protocol (engine.py:59-75) over a sharded state."""

    name = "sv-b200-dist"
    supports_reverse_gradient = False

    def __init__(self, comm, engine=None):
        self.comm = comm
        self.engine = engine or CudaEngine()

    def prepare(self, bitstring: str) -> DistStateVector:
        return init_state(bitstring, self.comm, self.engine)

    def evolve(self, state: DistStateVector, bound) -> DistStateVector:
        return evolve(state, bound)

    def expectation(self, state: DistStateVector, h) -> float:
        return expectation(state, h)

    def overlap(self, a: DistStateVector, b: DistStateVector) -> complex:
        return a.overlap(b)
