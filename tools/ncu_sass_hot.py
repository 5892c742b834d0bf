"""Hot SASS regions of one kernel in an ncu report (instructions executed and stall samples).
Usage: python tools/ncu_sass_hot.py report.ncu-rep kernel_regex [region_bytes] [top]"""
import collections
import csv
import io
import subprocess
import sys


def main(path, kern, region=0x200, top=12):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ie, src, ad = h.index("Instructions Executed"), h.index("Source"), h.index("Address")
    smp = h.index("Warp Stall Sampling (All Samples)")
    data = [(int(r[ad], 16), float(r[ie] or 0), float(r[smp] or 0), r[src].strip()) for r in rows[2:]
            if r[ad].startswith("0x")]
    base = data[0][0]
    ti = sum(d[1] for d in data) or 1
    ts = sum(d[2] for d in data) or 1
    reg_i, reg_s, ops = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
    for a, i, s, t in data:
        k = (a - base) // region
        reg_i[k] += i
        reg_s[k] += s
        op = t.split()[1] if t.startswith("@") else t.split()[0]
        ops[k][op] += i
    print(f"total warp instructions {ti:.0f}, samples {ts:.0f}")
    for k in sorted(reg_i, key=lambda k: -reg_i[k])[:top]:
        print(f"{hex(k * region):>8} instr {reg_i[k] / ti * 100:5.1f}%  stall {reg_s[k] / ts * 100:5.1f}%  "
              + " ".join(f"{o}:{c / reg_i[k] * 100:.0f}" for o, c in ops[k].most_common(6)))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3], 0) if len(sys.argv) > 3 else 0x200,
         int(sys.argv[4]) if len(sys.argv) > 4 else 12)
