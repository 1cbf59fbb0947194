"""Cost model + WaveK tuner (include/janus/tuner.hpp via janus_tune_wavek)
against the SPEC tuner / costmodel properties."""
import pytest

UMA = (26.25, 37.51, 43.59, 82.03)  # Table 4 UMA-1.2B
GB = 1e9


def test_divisor_candidates_and_argmax(janus):
    k, tuned, rows = janus.tune_wavek(4, 32, UMA, 1000 * GB, 0, 10 * GB, 1 * GB, 1 * GB)
    assert tuned and {r["k"] for r in rows} <= {4, 8, 16, 32}
    feas = [r for r in rows if r["feasible"]]
    best = min(feas, key=lambda r: (r["makespan"], r["k"]))
    assert k == best["k"]
    # k = 8 is at least as fast as k = P = 4 under generous memory (Appendix B.4
    # reports a 1.05x peak at k = 8; this WaveK picks its list policy and look-ahead window
    # per k by replay (schedule_gen.hpp wavek), which already closes most of that gap at k = P,
    # and that per-k window choice is also why peak memory is not monotone in k here)
    by = {r["k"]: r for r in rows}
    assert by[8]["makespan"] <= by[4]["makespan"]
    assert janus.tune_wavek(4, 32, UMA, 1000 * GB, 0, 10 * GB, 1 * GB, 1 * GB) == (k, tuned, rows)  # idempotent


def test_memory_budget_limits_k(janus):
    _, _, free = janus.tune_wavek(4, 32, UMA, 1000 * GB, 0, 10 * GB, 1 * GB, 1 * GB, divisors_only=False)
    lo = min(r["peak_max"] for r in free)
    hi = max(r["peak_max"] for r in free)
    assert hi > lo
    budget = (lo + hi) / 2
    k, tuned, rows = janus.tune_wavek(4, 32, UMA, budget, 0, 10 * GB, 1 * GB, 1 * GB, divisors_only=False)
    assert tuned
    chosen = next(r for r in rows if r["k"] == k)
    assert chosen["feasible"] and chosen["peak_max"] <= budget          # k* is memory-feasible
    assert all(r["feasible"] == (r["peak_max"] <= budget) for r in rows)
    assert all(chosen["makespan"] <= r["makespan"] for r in rows if r["feasible"])
    # no activation budget at all -> default k = P, untuned
    k, tuned, rows = janus.tune_wavek(4, 32, UMA, 10 * GB, 1 * GB, 10 * GB, 1 * GB, 1 * GB)
    assert (k, tuned, rows) == (4, False, [])


def test_non_divisor_candidates(janus):
    k, tuned, rows = janus.tune_wavek(4, 32, UMA, 1000 * GB, 0, 1 * GB, 1 * GB, 1 * GB, divisors_only=False)
    ks = [r["k"] for r in rows]
    assert ks == list(range(4, ks[-1] + 1)) and tuned
    with pytest.raises(janus.JanusError):  # partial order t_FE < t_FF < t_BE < t_BF
        janus.tune_wavek(4, 32, (2, 1, 3, 4), 1000 * GB, 0, GB, GB, GB)


def test_schedule_memory_lifetime_rule(janus):
    """zero activation bytes -> peak = static; SymFold peak <=
    1F1B-2nd peak (no replication, no recompute) under the SPEC uniform-static
    rule; the plan partition covers every unit once."""
    P, N = 4, 8
    sym = janus.schedule_text(janus.METHOD_SYMFOLD, P, N)
    one = janus.schedule_text(janus.METHOD_ONEF1B, P, N)
    assert (janus.schedule_memory(sym, UMA, 5.0, 0, 0) == 5.0).all()
    ps = janus.schedule_memory(sym, UMA, 10.0, 3.0, 2.0)
    po = janus.schedule_memory(one, UMA, 10.0, 3.0, 2.0)
    assert ps.max() <= po.max()
    m = janus.Model(L=32, H=256)
    plan = janus.plan_stages(m, 8)
    assert plan[0][0] == 0 and plan[-1][1] == m.n_units and all(plan[i][1] == plan[i + 1][0] for i in range(7))
