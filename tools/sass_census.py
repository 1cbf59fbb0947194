"""Per-kernel SASS census of the built library: tcgen05 / TMEM / TMA
instruction counts (the evidence of which kernels run on the Blackwell tensor
pipe).  UTCHMMA/UTCQMMA = tcgen05.mma, LDTM/STTM = tcgen05.ld/st, UTCBAR =
tcgen05.commit, UBLKCP = cp.async.bulk (1-D TMA), UTMALDG = tensor-map TMA,
HMMA = legacy mma.sync, FFMA = SIMT fp32 FMA.

    python tools/sass_census.py paper_2605_18404_b200/libjanus_b200.so > profiles/r02_sass_census.txt
"""
import re
import subprocess
import sys

OPS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UTMALDG", "HMMA", "FFMA"]


def main(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout
    kern, counts, order = None, {}, []
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            kern = m.group(1)
            counts[kern] = dict.fromkeys(OPS, 0)
            order.append(kern)
            continue
        if kern is None:
            continue
        ins = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if ins:
            op = ins.group(1)
            for o in OPS:
                if op == o:
                    counts[kern][o] += 1
    dem = subprocess.run(["c++filt"], input="\n".join(order), capture_output=True, text=True).stdout.splitlines()
    print("kernel".ljust(70) + "".join(o.rjust(9) for o in OPS))
    for k, d in zip(order, dem):
        c = counts[k]
        if not any(c[o] for o in OPS):
            continue
        print(d[:69].ljust(70) + "".join(str(c[o]).rjust(9) for o in OPS))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "paper_2605_18404_b200/libjanus_b200.so")
