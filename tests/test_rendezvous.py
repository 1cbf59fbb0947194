"""Blocking-rendezvous replay of the multi-process issue program
(include/janus/rendezvous.hpp, VERDICT r01 item 2 / ADVICE high #1).

NCCL P2P blocks the stream until the peer's matching op runs, so an issue
program deadlocks unless every send can meet its receive.  The simulator runs
each rank's compute lanes and transfer streams with exactly those semantics.
Round 1 put all of a rank's sends on one stream and all receives on another:
SymFold P=2 deadlocks there (device 0 sends [SAE mb3, SGF mb0], device 1
receives [RGF mb0, RAE mb3]).  The executor now gives every channel (flow,
from, to) its own communicator and stream ends; every generated schedule must
then complete for every P, lane count and data-parallel degree.
"""
import pytest


def schedules(J):
    for P in (2, 3, 4, 6, 8):
        for n_mb in (1, 4, 12, 32):
            yield ("symfold", P, n_mb, J.schedule_text(J.METHOD_SYMFOLD, P, n_mb), False)
            yield ("hanayo", P, n_mb, J.schedule_text(J.METHOD_HANAYO, P, n_mb), False)
            for k in sorted({1, min(P, n_mb), min(2 * P, n_mb)}):
                yield (f"wavek{k}", P, n_mb, J.schedule_text(J.METHOD_WAVEK, P, n_mb, k), False)
            if P % 2 == 0:
                yield ("1f1b", P, n_mb, J.schedule_text(J.METHOD_ONEF1B, P, n_mb), True)


def test_round1_shared_streams_deadlock(janus):
    """The round-1 layout reproduces the advisor's circular wait."""
    t = janus.schedule_text(janus.METHOD_SYMFOLD, 2, 4)
    ok, done, tot, stuck = janus.check_rendezvous(t, shared_streams=True)
    assert not ok and done < tot
    assert "SAE mb3" in stuck or "RGF mb0" in stuck or "RAE mb3" in stuck


@pytest.mark.parametrize("lanes,dp", [(1, 1), (8, 1), (3, 2)])
def test_per_channel_streams_never_deadlock(janus, lanes, dp):
    n = 0
    for name, P, n_mb, text, onef1b in schedules(janus):
        ok, done, tot, stuck = janus.check_rendezvous(text, onef1b=onef1b, lanes=lanes, dp=dp)
        assert ok, f"{name} P={P} N_mb={n_mb} lanes={lanes} dp={dp}: {done}/{tot}\n{stuck}"
        n += 1
    assert n > 50


def test_shared_streams_fail_widely(janus):
    """Not a corner case: most multi-micro-batch SymFold / WaveK / 1F1B
    programs deadlock under the round-1 layout."""
    bad = sum(not janus.check_rendezvous(text, onef1b=o, shared_streams=True)[0]
              for name, P, n_mb, text, o in schedules(janus) if n_mb >= 12)
    assert bad >= 10
