"""Activation slot pool (include/janus/slots.hpp): the
executor's per-device slot counts, derived from the schedule's issue order,
on CPU — the fold is visible in the counts, the lane floor holds, and the
per-rank programs with the pool's release waits stay deadlock-free."""
import pytest


def sizes(janus, method, P, n_mb=32, k=1, local=True, lanes=1, unfolded=False):
    t = janus.schedule_text(method, P, n_mb, k)
    return janus.slot_pool(t, onef1b=(method == janus.METHOD_ONEF1B), local=local, unfolded=unfolded, lanes=lanes)


def test_symfold_keeps_2P_minus_d_live(janus):
    """Per rank, SymFold's device d holds 2P - d micro-batches (16..9 at P=8);
    one stage holds every micro-batch only in the unfolded layout."""
    for P in (2, 4, 8):
        got = sizes(janus, janus.METHOD_SYMFOLD, P, local=False)
        assert got == [2 * P - d for d in range(P)], (P, got)
        assert sizes(janus, janus.METHOD_SYMFOLD, P, unfolded=True) == [32] * P


@pytest.mark.parametrize("method", ["SYMFOLD", "WAVEK", "HANAYO", "ONEF1B"])
def test_pool_never_exceeds_micro_batches_and_honours_lanes(janus, method):
    m = getattr(janus, "METHOD_" + method)
    for P in (2, 4, 8):
        for lanes in (1, 8, 32):
            got = sizes(janus, m, P, k=P, lanes=lanes)
            assert all(min(lanes, 32) <= s <= 32 for s in got), (method, P, lanes, got)


def test_single_stage_lanes_floor(janus):
    """P=1: the list order keeps two micro-batches live; 32 lanes need 32 slots."""
    assert sizes(janus, janus.METHOD_SYMFOLD, 1) == [2]
    assert sizes(janus, janus.METHOD_SYMFOLD, 1, lanes=32) == [32]


def test_fold_beats_1f1b_per_device_objects(janus):
    """1F1B-2nd holds two blocks' stage objects per device; its largest
    per-object pool at P=8 (energy device 0) equals SymFold's, so its bytes
    per device are larger wherever a device carries both blocks."""
    s = sizes(janus, janus.METHOD_SYMFOLD, 8, local=False)
    o = sizes(janus, janus.METHOD_ONEF1B, 8, local=False)
    assert max(s) == max(o) == 16
