"""Programmatic dependent launch invariant (csrc/common.cuh).

stage.cu launches its kernels with programmatic stream serialization, so a
kernel may start before its predecessor on the lane stream has completed.
That is safe only because every such kernel executes griddepcontrol.wait
(JANUS_GDC_WAIT) as its FIRST statement: nothing it reads or writes precedes
the predecessor's completion, and completion stays transitive along the
stream.  This CPU test checks the invariant on the sources and that every
janus::pdl launch names a kernel that carries the wait.
"""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2605_18404_b200", "csrc")
KERNEL_FILES = ["edge_kernels.cuh", "edge_tc.cuh", "pair_tc.cuh", "upd_tc.cuh", "wgrad_tc.cuh", "node_kernels.cuh",
                "wide.cuh", "stage.cu", "nbrlist.cu", "gemm_tc.cuh"]
LAUNCH_FILES = ["stage.cu", "stage_wide.inc", "nbrlist.cu", "gemm_tc_host.hpp", "edge_kernels.cuh"]


def kernels(text):
    """(name, first statement of the body) of every __global__ definition."""
    out = []
    for m in re.finditer(r"__global__", text):
        i, depth = m.end(), 0
        while True:
            ch = text[i]
            if ch == "(":
                depth += 1
            elif ch == ")":
                depth -= 1
            elif depth == 0 and ch == ";":
                i = None
                break
            elif depth == 0 and ch == "{":
                break
            i += 1
        if i is None:
            continue
        head = text[m.end():i]
        names = [n for n in re.findall(r"(\w+)\s*\(", head) if n not in ("__launch_bounds__", "__maxnreg__")]
        body = text[i + 1:].lstrip()
        out.append((names[0], body.split(";", 1)[0].strip()))
    return out


def test_every_kernel_waits_first():
    seen = {}
    for f in KERNEL_FILES:
        for name, first in kernels(open(os.path.join(CSRC, f)).read()):
            assert first == "JANUS_GDC_WAIT()", f"{f}: kernel {name} starts with {first!r}"
            seen[name] = f
    assert len(seen) > 60


def test_pdl_launches_name_waiting_kernels():
    waiting = set()
    for f in KERNEL_FILES:
        waiting |= {n for n, _ in kernels(open(os.path.join(CSRC, f)).read())}
    n = 0
    for f in LAUNCH_FILES:
        text = open(os.path.join(CSRC, f)).read()
        assert "<<<" not in text, f"{f}: plain <<<>>> launch in a PDL launch file"
        for m in re.finditer(r"janus::pdl\(([\w:]+)", text):
            name = m.group(1).split("::")[-1]
            assert name == "KERN" or name in waiting, f"{f}: janus::pdl launches {name}, which has no JANUS_GDC_WAIT"
            n += 1
    assert n > 80
