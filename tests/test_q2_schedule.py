"""Host-side check of the Q2 wavefront schedule (reading R17) used by
`apply_q2wave_kernel` (q2w.cu): the step enumeration below mirrors the kernel's
(`dhi = min(G-1, t)`, `dlo` = first d with `t - d < J(G-1-d)`, block
`(G-1-d, t-d)`), and the checks are the conditions under which running the
blocks step by step equals the sequential order of reading R7 (groups last to
first, steps ascending): every block exactly once, the blocks of one step
pairwise disjoint, and every overlapping block that precedes a block in R7's
order scheduled at an earlier step.  No GPU: the GPU parity tests check the
kernel's numbers against the oracle."""
import pytest

NB, G = 64, 32
W = NB + G - 1


def groups(n):
    return (n - 1 + G - 1) // G   # sweeps 0 .. n-2 in groups of G


def steps(n, g):
    i0 = g * G
    return 0 if i0 > n - 2 else (n - 2 - i0) // NB + 1


def rows(n, g, j):
    r0 = g * G + 1 + j * NB
    return set(range(r0, min(n, r0 + W)))


def schedule(n):
    Gn = groups(n)
    T = 0
    for g in range(Gn):
        J = steps(n, g)
        if J > 0:
            T = max(T, J - 1 + (Gn - 1 - g) + 1)
    out = []
    for t in range(T):
        dhi = min(Gn - 1, t)
        dlo = 0
        while dlo <= dhi and t - dlo >= steps(n, Gn - 1 - dlo):
            dlo += 1
        out.append([(Gn - 1 - d, t - d) for d in range(dlo, dhi + 1)])
    return out


@pytest.mark.parametrize("n", [2, 3, 65, 66, 100, 257, 517, 1000, 2049])
def test_wavefront_schedule_matches_sequential_order(n):
    sched = schedule(n)
    Gn = groups(n)
    when = {}
    for t, blocks in enumerate(sched):
        for b in blocks:
            assert b not in when
            when[b] = t
    expect = {(g, j) for g in range(Gn) for j in range(steps(n, g))}
    assert set(when) == expect                      # every block exactly once
    for blocks in sched:                            # one step: pairwise disjoint windows
        for a in range(len(blocks)):
            for b in range(a + 1, len(blocks)):
                assert not (rows(n, *blocks[a]) & rows(n, *blocks[b]))
    seq = [(g, j) for g in range(Gn - 1, -1, -1) for j in range(steps(n, g))]
    pos = {b: k for k, b in enumerate(seq)}
    for b in seq:                                   # R7 predecessors that overlap run earlier
        rb = rows(n, *b)
        for a in seq[:pos[b]]:
            if rows(n, *a) & rb:
                assert when[a] < when[b], (a, b)


def test_wavefront_parallelism_n10000():
    """n = 10^4: ~J + G steps with up to ~J/2 disjoint blocks each (the
    per-fragment chain had 24.4K sequential blocks)."""
    sched = schedule(10000)
    nblocks = sum(len(s) for s in sched)
    assert nblocks == sum(steps(10000, g) for g in range(groups(10000)))
    assert len(sched) < 500 and max(len(s) for s in sched) > 100


def dataflow_deps(n, g, j):
    """Blocks apply_q2wave3_kernel waits for before block (g, j): (g, j-1),
    (g+1, j-1), (g+1, j), those that exist."""
    Gn = groups(n)
    out = []
    for gg, jj in ((g, j - 1), (g + 1, j - 1), (g + 1, j)):
        if 0 <= gg < Gn and 0 <= jj < steps(n, gg):
            out.append((gg, jj))
    return out


@pytest.mark.parametrize("n", [2, 3, 65, 66, 100, 257, 517, 1000, 2049])
def test_dataflow_waits_cover_every_overlapping_predecessor(n):
    """The 3M kernel replaces the grid barrier between steps by per-block
    completion counters and waits only for dataflow_deps: every block that
    precedes b in R7's order and overlaps it must be reachable from b through
    those waits (then it is complete when b starts), and every wait must point
    to an earlier step (no cycles)."""
    sched = schedule(n)
    when = {b: t for t, blocks in enumerate(sched) for b in blocks}
    Gn = groups(n)
    seq = [(g, j) for g in range(Gn - 1, -1, -1) for j in range(steps(n, g))]
    pos = {b: k for k, b in enumerate(seq)}
    reach = {}
    for b in sorted(seq, key=lambda x: when[x]):     # deps are at earlier steps: closure in step order
        r = set()
        for d in dataflow_deps(n, *b):
            assert when[d] < when[b], (d, b)
            r.add(d)
            r |= reach[d]
        reach[b] = r
    for b in seq:
        rb = rows(n, *b)
        for a in seq[:pos[b]]:
            if rows(n, *a) & rb:
                assert a in reach[b], (a, b)
