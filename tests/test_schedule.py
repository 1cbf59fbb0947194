"""Schedule layer: bit-exact parity with the reference's own code (frozen in
tests/golden/sched_golden.json by make_sched_golden.py from the compiled
reference headers), SPEC.md known-answer tests and property sweeps."""
import hashlib
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MINE = os.path.join(ROOT, "oracle", "_ref", "sched_mine")
REF = os.path.join(ROOT, "oracle", "_ref", "sched_ref")
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "sched_golden.json")))


def cli(*args, binary=MINE, ok=True):
    r = subprocess.run([binary, *map(str, args)], capture_output=True, text=True)
    if ok:
        assert r.returncode == 0, r.stdout + r.stderr
    return r


@pytest.fixture(scope="module")
def tmpfile(tmp_path_factory, built):
    d = tmp_path_factory.mktemp("sched")

    def write(name, text):
        p = d / name
        p.write_text(text)
        return str(p)
    return write


def test_passes_match_reference_golden(tmpfile):
    """Pass 0 (ours) -> Passes 1-3 by OUR headers == reference output (sha)."""
    for key, rec in GOLD["grid"].items():
        P, N = map(int, key.split("_"))
        first = cli("first", P, N).stdout
        assert hashlib.sha256(first.encode()).hexdigest() == rec["first_sha"]
        fp = tmpfile("first.txt", first)
        for m in ("fold", "lin"):
            head, body = cli("passes", fp, m).stdout.split("\n", 1)
            assert int(head.split()[-1]) == rec[f"{m}_pruned"], (P, N, m)
            assert hashlib.sha256(body.encode()).hexdigest() == rec[f"{m}_sha"], (P, N, m)
            sp = tmpfile(f"{m}.txt", body)
            for tn, t in (("uma-1.2b", ["26.25", "37.51", "43.59", "82.03"]), ("uniform", ["1", "2", "3", "4"])):
                line = cli("replay", sp, *t).stdout.split("\n", 1)[0].split()
                assert line[3] == rec[f"{m}_{tn}_makespan"] and line[5] == rec[f"{m}_{tn}_oracle"], (P, N, m, tn)


def test_symfold_generator_equals_reference_text():
    for name, text in GOLD["text"].items():
        m, P, N = name.split("_")
        if m != "fold":
            continue
        assert cli("symfold", P[1:], N[1:]).stdout == text


def test_prune_count_is_4nmb():
    """Pass 3 removes exactly 4 N_mb comm instructions."""
    for rec_key, rec in GOLD["grid"].items():
        N = int(rec_key.split("_")[1])
        assert rec["fold_pruned"] == 4 * N


@pytest.mark.skipif(not os.path.exists(REF), reason="reference checker needs /root/reference (dev container only)")
def test_live_reference_diff(tmpfile):
    """When the reference is present, diff every API mode live (not just hashes)."""
    for P, N in [(1, 1), (2, 3), (3, 4), (4, 8), (8, 12)]:
        for gen in ("symfold", "first") + (("onef1b",) if P % 2 == 0 else ()):
            f = tmpfile("s.txt", cli(gen, P, N).stdout)
            for mode in (["roundtrip"], ["deps"], ["topo", "slot"], ["topo", "mbmajor"],
                         ["replay", "0.1", "0.2", "0.3", "0.7"]):
                a = cli(mode[0], f, *mode[1:]).stdout
                b = cli(mode[0], f, *mode[1:], binary=REF).stdout
                assert a == b, (gen, P, N, mode)


@pytest.mark.parametrize("text,line", [
    ("", 1),
    ("SCHEDULE P=1 NMB=1 ORDER=second\nD0 0 XX mb=0 vs=0 peer=-\n", 2),
    ("SCHEDULE P=1 NMB=1 ORDER=second\nD3 0 FE mb=0 vs=0 peer=-\n", 2),
    ("SCHEDULE P=1 NMB=1 ORDER=second\nD0 0 FE mb=0 vs=0\n", 2),
    ("SCHEDULE P=0 NMB=1 ORDER=second\n", 1),
    ("SCHEDULE P=1 NMB=1 ORDER=third\n", 1),
    ("SCHEDULE P=1 NMB=1 ORDER=second\nD0 0 FE mb=0 vs=0 peer=- flags=foo\n", 2),
])
def test_parse_errors_carry_line(tmpfile, text, line):
    """errors.hpp:19-24 / SPEC.md:90: malformed text -> parse_error with line."""
    r = cli("roundtrip", tmpfile("bad.txt", text), ok=False)
    assert r.returncode == 3 and r.stdout.startswith(f"parse_error line {line}")


def test_validator_accepts_generators_sweep(tmpfile):
    """SPEC.md:95/137/147 — every generator output validates (P 1..8, N 1..16)."""
    for P in range(1, 9):
        for N in (1, 2, 3, 5, 8, 16):
            for gen, extra in (("symfold", []), ("first", []), ("wavek", [max(1, N // 2)])):
                if gen == "wavek" and P > 4 and N > 8:
                    continue  # covered by the bench-size test below; keep the sweep < 60 s
                f = tmpfile("v.txt", cli(gen, P, N, *extra).stdout)
                assert cli("validate", f).stdout.startswith("ok 1"), (gen, P, N)
            if P % 2 == 0:
                f = tmpfile("v.txt", cli("onef1b", P, N).stdout)
                assert cli("validate", f).stdout.startswith("ok 1"), ("onef1b", P, N)


def _lines(text):
    return text.rstrip("\n").split("\n")


def test_validator_rejects_mutations(tmpfile):
    """deleting/duplicating a compute or deleting a receive is caught."""
    base = _lines(cli("symfold", 3, 2).stdout)
    computes = [i for i, l in enumerate(base) if l.split()[2:3] and l.split()[2] in ("FE", "FF", "BE", "BF")]
    recvs = [i for i, l in enumerate(base) if l.split()[2:3] and l.split()[2] in ("RAF", "RAE", "RGF", "RGE")]
    for i in computes[:6] + recvs[:4]:
        mutated = base[:i] + base[i + 1:]
        f = tmpfile("m.txt", "\n".join(mutated) + "\n")
        assert not cli("validate", f, ok=False).stdout.startswith("ok 1"), base[i]
    for i in computes[:4]:
        mutated = base[:i + 1] + [base[i]] + base[i + 1:]
        f = tmpfile("m.txt", "\n".join(mutated) + "\n")
        assert not cli("validate", f, ok=False).stdout.startswith("ok 1"), base[i]


def test_validator_rejects_dependency_transposition(tmpfile):
    """Swap FF(mb0) and BF(mb0) on D0 -> BF before its FF: dependency error."""
    text = cli("symfold", 1, 2).stdout
    lines = _lines(text)
    ff = next(i for i, l in enumerate(lines) if " FF mb=0 " in l)
    bf = next(i for i, l in enumerate(lines) if " BF mb=0 " in l)
    a, b = lines[ff].split(" ", 2), lines[bf].split(" ", 2)
    lines[ff], lines[bf] = " ".join([a[0], a[1], b[2]]), " ".join([b[0], b[1], a[2]])
    out = cli("validate", tmpfile("t.txt", "\n".join(lines) + "\n"), ok=False).stdout
    assert out.startswith("ok 0") and "dependency 1" in out


def test_wavek_beats_symfold_and_1f1b_in_replay():
    """Directional SPEC.md:726 (a): best-k WaveK <= SymFold < 1F1B-2nd makespan."""
    out = cli("compare", 4, 32, "uma-1.2b").stdout
    ms = {l.split("makespan")[0].strip(): float(l.split()[-5]) for l in _lines(out)}
    best = min(v for k, v in ms.items() if k.startswith("wavek"))
    assert best <= ms["symfold"] < ms["onef1b_2nd"]
    assert all(l.endswith("valid 1") for l in _lines(out))


def test_hanayo_2nd_baseline(janus):
    """Hanayo-2nd: V-shape = fold_map placement,
    valid for P 1..8 x N 4..12, FF carries the recompute flag, hanayo_2nd(1,1)
    keeps both virtual stages on D0; under Table 4 times it is slower than
    SymFold (it recomputes FE inside FF)."""
    for P in (1, 2, 3, 4, 8):
        for N in (1, 4, 8, 12):
            text = janus.schedule_text(janus.METHOD_HANAYO, P, N)
            assert janus.validate_schedule(text) == 0, (P, N)
            sym = janus.schedule_text(janus.METHOD_SYMFOLD, P, N)
            # same instructions per device as SymFold (V placement), wave order, FF recompute
            body = lambda t: sorted(" ".join(l.replace(" flags=recompute", "").split()[:1] +  # noqa: E731
                                             l.replace(" flags=recompute", "").split()[2:])
                                    for l in t.splitlines()[1:])
            assert body(text) == body(sym), (P, N)
            ff = [l for l in text.splitlines()[1:] if l.split()[2] == "FF"]
            assert ff and all(l.endswith("flags=recompute") for l in ff), ff[:2]
    t1 = janus.schedule_text(janus.METHOD_HANAYO, 1, 1)
    assert {l.split()[0] for l in t1.splitlines()[1:]} == {"D0"}
    uma = (26.25, 37.51, 43.59, 82.03)
    for P in (4, 8):
        mh, _ = janus.schedule_replay(janus.schedule_text(janus.METHOD_HANAYO, P, 2 * P), *uma)
        ms, _ = janus.schedule_replay(janus.schedule_text(janus.METHOD_SYMFOLD, P, 2 * P), *uma)
        assert ms < mh


def test_render_timeline(janus):
    """render: symfold(1,1) lane reads FE FF BF BE; byte-identical reruns; SVG well-formed."""
    txt = janus.schedule_text(janus.METHOD_SYMFOLD, 1, 1)
    a = janus.render_timeline(text=txt, t=(1, 2, 3, 4), quantum=0)
    lane = a.splitlines()[0]
    assert [lane.index(x) for x in ("FE", "FF", "BF", "BE")] == sorted(lane.index(x) for x in ("FE", "FF", "BF", "BE"))
    assert a == janus.render_timeline(text=txt, t=(1, 2, 3, 4), quantum=0)
    w = janus.schedule_text(janus.METHOD_WAVEK, 4, 12, 4)
    r4 = janus.render_timeline(text=w, t=(26.25, 37.51, 43.59, 82.03), quantum=10)
    assert len(r4.splitlines()) == 4 and r4 == janus.render_timeline(text=w, t=(26.25, 37.51, 43.59, 82.03), quantum=10)
    svg = janus.render_timeline(text=w, t=(26.25, 37.51, 43.59, 82.03), svg=True, quantum=0.5)
    assert svg.startswith("<svg") and svg.rstrip().endswith("</svg>") and svg.count("<rect") == 4 * 4 * 12
    recs = [[0, 0, 0, 0.0, 1.0], [0, 1, 0, 1.0, 3.0], [1, 3, 0, 3.0, 7.0]]
    out = janus.render_timeline(recs=recs, quantum=0.5)
    assert out.splitlines()[0].startswith("D0 |FEFF==") and out.splitlines()[1].startswith("D1 |......BF")
