"""Attribute ncu per-SASS samples / instruction counts to CUDA source lines.

usage: python tools/ncu_lines.py REPORT.ncu-rep OBJECT.o KERNEL_SUBSTR [top]

Joins `ncu --page source --print-source sass --csv` (per-address warp-stall
samples and executed instructions) with `nvdisasm -g` line info of the kernel's
cubin (objects are built with -lineinfo).  Development aid for profiles/."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_lines(obj, kernel_sub):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True,
                   capture_output=True)
    cubin = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cubin)], capture_output=True,
                         text=True).stdout
    out, cur, on, where = {}, None, False, None
    for line in txt.splitlines():
        m = re.match(r"^\.text\.(\S+):", line)
        if m:
            on = kernel_sub in m.group(1)
            continue
        if not on:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            where = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", line)
        if m and where:
            out[int(m.group(1), 16)] = (where, m.group(2).strip().rstrip(";"))
    return out


def main():
    rep, obj, ksub = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    # one kernel of a multi-kernel report: filter on import, first matching launch
    kfilt = ksub.split("ILi")[0]  # a mangled template suffix selects SASS, not the ncu filter
    raw = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kfilt}", "-c", "1", "--page", "source",
                          "--print-source", "sass", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr_i]
    ia, isamp, iinst = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    lines = sass_lines(obj, ksub)
    agg = collections.defaultdict(lambda: [0.0, 0.0, collections.Counter()])
    tot_s = tot_i = 0.0
    base = None
    for r in rows[hdr_i + 1:]:
        if len(r) <= iinst or not r[ia].startswith("0x") and not r[ia].isdigit():
            continue
        addr = int(r[ia], 16) if r[ia].startswith("0x") else int(r[ia])
        base = addr if base is None else base
        addr -= base  # the report holds load addresses; the listing starts at 0
        s = float(r[isamp] or 0)
        n = float((r[iinst] or "0").replace(",", ""))
        where = lines.get(addr, ("?", ""))[0]
        a = agg[where]
        a[0] += s
        a[1] += n
        for c in stall_cols:
            v = float(r[c] or 0)
            if v:
                a[2][h[c]] += v
        tot_s += s
        tot_i += n
    print(f"{'line':28s} {'samples%':>9s} {'inst%':>7s}  top stalls")
    for where, (s, n, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        ss = ", ".join(f"{k[6:]}={v / max(s, 1) * 100:.0f}%" for k, v in st.most_common(3))
        print(f"{where:28s} {100 * s / tot_s:9.2f} {100 * n / tot_i:7.2f}  {ss}")


if __name__ == "__main__":
    main()
