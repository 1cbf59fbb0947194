"""Freeze the reference's own schedule outputs as golden data.

Runs in the dev container only (needs /root/reference): builds
oracle/_ref/sched_ref (oracle/sched_cli.cpp compiled against the reference
headers, read-only in place) and records, for a grid of (P, N_mb):
  * sha256 of Passes 1+2+3 applied by the REFERENCE to our Pass-0 text, for
    the SymFold map (fold_map, ir.hpp:161) and the linear 1F1B-2nd map;
  * the reference replay makespan + longest-path oracle under Table-4 times;
  * the reference Pass-3 prune count;
  * full text for a few small schedules.
tests/test_schedule_golden.py compares the repo's generators against this.
Usage: python tests/golden/make_sched_golden.py
"""
import hashlib
import json
import os
import subprocess
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.path.join(ROOT, "oracle", "_ref", "sched_ref")
MINE = os.path.join(ROOT, "oracle", "_ref", "sched_mine")
PS = list(range(1, 9))
NS = [1, 2, 3, 4, 5, 8, 12, 16, 32]
TIMES = {"uma-1.2b": ["26.25", "37.51", "43.59", "82.03"], "uniform": ["1", "2", "3", "4"]}


def run(*args):
    return subprocess.run(list(args), check=True, capture_output=True, text=True).stdout


def main():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    assert os.path.exists(REF), "reference checker not built (is /root/reference present?)"
    out = {"grid": {}, "text": {}}
    with tempfile.TemporaryDirectory() as td:
        for P in PS:
            for N in NS:
                first = run(MINE, "first", str(P), str(N))
                fp = os.path.join(td, "first.txt")
                open(fp, "w").write(first)
                rec = {"first_sha": hashlib.sha256(first.encode()).hexdigest()}
                for m in ("fold", "lin"):
                    txt = run(REF, "passes", fp, m)
                    head, body = txt.split("\n", 1)
                    rec[f"{m}_pruned"] = int(head.split()[-1])
                    rec[f"{m}_sha"] = hashlib.sha256(body.encode()).hexdigest()
                    sp = os.path.join(td, f"{m}.txt")
                    open(sp, "w").write(body)
                    for tn, t in TIMES.items():
                        line = run(REF, "replay", sp, *t).split("\n", 1)[0].split()
                        rec[f"{m}_{tn}_makespan"] = line[3]
                        rec[f"{m}_{tn}_oracle"] = line[5]
                    if P <= 3 and N <= 2:
                        out["text"][f"{m}_P{P}_N{N}"] = body
                out["grid"][f"{P}_{N}"] = rec
    path = os.path.join(ROOT, "tests", "golden", "sched_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
