"""Window-major piece layout of the segmented edge_softmax statistics
(kernels._softmax_segplan, gmp_segplan in include/gmp.h), built on the CPU
and checked structurally: perm is the heavy rows' in-edges ordered by
(window, heavy row, edge id); pieces are the runs of one (window, row),
cut every GMP_SEG_CHUNK positions; row_pieces lists each row's pieces in
window order; the start bits and chunk piece ids agree with the pieces. A
NumPy walk of the kernel's chunk / piece traversal then reproduces each heavy
row's sum of scores exactly as a direct per-row sum."""

import numpy as np
import torch

from paper_1909_01315_b200 import graph, kernels


class _Sched:
    def __init__(self, adj, heavy):
        deg = (adj.indptr[1:] - adj.indptr[:-1]).numpy()
        order = np.argsort(-deg, kind="stable").astype(np.int32)
        self.order = torch.as_tensor(order)
        self.n_heavy = int((deg > heavy).sum())


def _graph(n, m, seed):
    rng = np.random.default_rng(seed)
    # a few hubs plus uniform background; edge list grouped by source
    dst = np.where(rng.random(m) < 0.6, rng.integers(0, 5, m), rng.integers(0, n, m))
    src = rng.integers(0, n, m)
    o = np.argsort(src, kind="stable")
    return torch.as_tensor(src[o]), torch.as_tensor(dst[o]), n


def _check(adj, sched, win, group):
    plan = kernels._softmax_segplan(adj, sched, win, group)
    perm, starts, chunk_piece, row_ptr, row_pieces = (t.numpy() for t in plan.tensors)
    CS = kernels._SEG_CHUNK_SUB
    R = sched.n_heavy
    order = sched.order.numpy()[:R]
    ip = adj.indptr.numpy()
    eids = adj.edge_ids.numpy()
    keys = []
    for r, row in enumerate(order):
        for e in np.sort(eids[ip[row]:ip[row + 1]]):
            keys.append((e // win, r, e))
    keys.sort()
    # expected padded layout: each (window, row) run padded to `group`
    want_perm, want_new, want_row = [], [], []
    k = 0
    while k < len(keys):
        j = k
        while j < len(keys) and keys[j][:2] == keys[k][:2]:
            j += 1
        run = [x[2] for x in keys[k:j]]
        nsub = -(-len(run) // group)
        want_perm += run + [-1] * (nsub * group - len(run))
        want_new += [True] + [False] * (nsub - 1)
        want_row += [keys[k][1]] * nsub
        k = j
    while len(want_new) % CS:  # the last chunk is padded whole
        want_perm += [-1] * group
        want_new.append(False)
        want_row.append(want_row[-1])
    assert np.array_equal(perm, np.array(want_perm, dtype=np.int32))
    assert plan.struct.n_pos == len(want_perm) and plan.struct.group == group
    n_sub = len(want_new)
    new = np.array(want_new)
    new[::CS] = True
    bits = np.unpackbits(starts.view(np.uint32).view(np.uint8), bitorder="little")[:n_sub]
    assert np.array_equal(bits.astype(bool), new)
    pid = np.cumsum(new) - 1
    assert plan.struct.n_pieces == pid[-1] + 1
    assert np.array_equal(chunk_piece, pid[::CS])
    piece_row = np.array(want_row)[new]
    for r in range(R):
        q = row_pieces[row_ptr[r]:row_ptr[r + 1]]
        assert np.all(np.diff(q) > 0) and np.all(piece_row[q] == r)
    assert row_ptr[-1] == plan.struct.n_pieces
    # the kernel's walk: chunks of CS sub-steps of `group` positions; a piece
    # closes at each start bit and at every chunk end; rows fold their pieces
    score = np.random.default_rng(1).standard_normal(eids.size)
    part = np.zeros(plan.struct.n_pieces)
    for c in range(-(-n_sub // CS)):
        piece = chunk_piece[c] - 1
        for j in range(c * CS, min((c + 1) * CS, n_sub)):
            if bits[j]:
                piece += 1
            for e in perm[j * group:(j + 1) * group]:
                if e >= 0:
                    part[piece] += score[e]
    for r, row in enumerate(order):
        got = part[row_pieces[row_ptr[r]:row_ptr[r + 1]]].sum()
        want = score[eids[ip[row]:ip[row + 1]]].sum()
        assert abs(got - want) <= 1e-9 * (1 + abs(want))


def test_segplan_layout_and_walk():
    src, dst, n = _graph(400, 20000, 0)
    adj = graph._build_adjacency(dst, src, n)
    sched = _Sched(adj, heavy=40)
    for win, group in ((1500, 16), (700, 4), (5000, 32), (20000, 1)):
        _check(adj, sched, win, group)


def test_lane_groups_match_launch_layout():
    # fp32: float4 lanes when H % 4 == 0; fp64 at most 2 per lane
    assert kernels._softmax_lane_groups(8, 4) == 16
    assert kernels._softmax_lane_groups(1, 4) == 32
    assert kernels._softmax_lane_groups(16, 4) == 8
    assert kernels._softmax_lane_groups(8, 8) == 8
    assert kernels._softmax_lane_groups(6, 4) == 8
    assert kernels._softmax_lane_groups(128, 4) == 1
