"""The weight ring of rollout_tc2.cu's producer, restated in Python: K-block pairs (hi, lo)
placed contiguously in a byte ring, a virtual byte counter that also counts the tail a wrap
skips, and in-order release.  Checked: no in-flight block is ever overwritten, for the block
sequences of the BASELINE configs and random ones (sizes, ring bytes, slot counts), and the
producer never waits on a block the consumer has not reached (no deadlock) when the ring holds
two blocks of the largest pair."""
import numpy as np
import pytest

K_SLOTS = 16


def simulate(blocks, ring, k_slots=K_SLOTS, lag=0):
    """blocks: list of (kblock id, bytes) in stream order, two entries (hi, lo) per K-block.
    The consumer releases K-block k after it has both blocks; the producer may run `lag`
    K-blocks ahead of the consumer at most by construction of the waits.  Returns the number
    of producer waits.  Raises on an overlap of in-flight blocks or a deadlock."""
    pos = vpos = 0
    inflight = []  # (kblock, phys_lo, phys_hi, vstart), oldest first
    released = -1  # highest K-block whose MMAs retired
    waits = 0
    i = 0
    while i < len(blocks):
        kb, b = blocks[i]
        assert blocks[i + 1][0] == kb and blocks[i + 1][1] == b
        if pos + 2 * b > ring:
            vpos += ring - pos
            pos = 0
        at0 = pos
        pos += 2 * b
        for part in range(2):
            at = at0 + part * b
            vs = vpos
            vpos += b
            while inflight:
                okb, lo, hi, ovs = inflight[0]
                if len(inflight) < k_slots and ovs - (vpos - ring) >= 0:
                    break
                # producer waits for the oldest block's K-block release: the consumer must be
                # able to get there without this block (its pair must be complete already)
                if okb == kb:
                    raise RuntimeError("deadlock: waiting for the pair being placed")
                released = max(released, okb)
                inflight = [e for e in inflight if e[0] > released]
                waits += 1
            for (okb, lo, hi, ovs) in inflight:
                assert hi <= at or lo >= at + b, ("overwrite of an in-flight block", okb, kb)
            inflight.append((kb, at, at + b, vs))
        i += 2
    return waits


def config_blocks(npads, kbs, steps=3):
    seq, k = [], 0
    for _ in range(steps):
        for npad, kb in zip(npads, kbs):
            for _ in range(kb):
                seq += [(k, npad * 128), (k, npad * 128)]
                k += 1
    return seq


@pytest.mark.parametrize("npads,kbs,ring", [
    ([256, 256, 256, 32], [2, 8, 8, 8], 170 * 1024),   # C3 (v2, one 256-wide tile)
    ([256, 256, 256, 32], [2, 8, 8, 8], 80 * 1024),    # C3 at the minimum ring
    ([128, 128, 64], [1, 4, 4], 48 * 1024),            # C4 with folded cost columns, minimum ring
    ([128, 128, 128, 16], [1, 4, 4, 4], 56 * 1024),    # C2 on v2 (two tiles)
    ([160, 160, 16], [1, 5, 5], 67 * 1024),            # 160-wide, ragged sizes
])
def test_ring_never_overwrites_in_flight_blocks(npads, kbs, ring):
    simulate(config_blocks(npads, kbs), ring)


def test_ring_random_sequences():
    rng = np.random.default_rng(0)
    for _ in range(300):
        sizes = rng.choice([16, 32, 48, 64, 96, 128, 160, 192, 256], size=rng.integers(1, 40))
        seq = []
        for k, npad in enumerate(sizes):
            seq += [(k, int(npad) * 128)] * 2
        biggest = 2 * max(b for _, b in seq)
        ring = int(rng.integers(biggest, biggest * 4)) & ~1023
        ring = max(ring, biggest)
        simulate(seq, ring, k_slots=int(rng.integers(2, 17)))
