"""Render ncu --set full reports into a committed text summary (key metrics, stall
reasons, top source lines, opcode mix) and record each kernel's DRAM bytes per launch
in profiles/ncu_traffic.json (bench.py reports it as roofline.traffic).
usage: python tools/ncu_summary.py OUT.txt HEADER rep1.ncu-rep [rep2 ...]"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct", "lts__t_bytes.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    out, header, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    lines = [f"# {header}"]
    tpath = "profiles/ncu_traffic.json"
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for rep in reps:
        rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
        h, units = rows[0], rows[1]
        for d in rows[2:]:
            name = d[h.index("Kernel Name")]
            short = re.sub(r"\(.*", "", name).strip()
            lines.append(f"\n## {short}   ({os.path.basename(rep)})")
            for k in KEYS:
                if k in h:
                    lines.append(f"   {k:62s} {d[h.index(k)]} {units[h.index(k)]}")
            rd = float(d[h.index("dram__bytes_read.sum")]) * SCALE.get(units[h.index("dram__bytes_read.sum")], 1)
            wr = float(d[h.index("dram__bytes_write.sum")]) * SCALE.get(units[h.index("dram__bytes_write.sum")], 1)
            key = re.sub(r"^void\s+", "", short)
            traffic[key.split("<")[0].split("::")[-1]] = {"kernel": key, "dram_bytes_per_launch": rd + wr,
                                                           "read": rd, "write": wr, "report": os.path.basename(rep)}
        # stall reasons and opcode mix from the SASS source page
        sass = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
        hs = next((r for r in sass if r and r[0] == "Address"), None)
        if hs:
            ie, src = hs.index("Instructions Executed"), hs.index("Source")
            stall = [c for c in hs if c.startswith("stall_")] if any(c.startswith("stall_") for c in hs) else []
            ops, tot = collections.Counter(), 0
            st = collections.Counter()
            for r in sass[sass.index(hs) + 1:]:
                if len(r) < len(hs) or not r[ie].strip().isdigit():
                    continue
                n = int(r[ie])
                tok = r[src].strip().split()
                if not tok:
                    continue
                o = tok[1] if tok[0].startswith("@") else tok[0]
                ops[o.split(".")[0]] += n
                tot += n
                for c in stall:
                    v = r[hs.index(c)].strip()
                    if v.replace(".", "").isdigit():
                        st[c] += float(v)
            lines.append("   opcode mix (executed warp instructions): " +
                         ", ".join(f"{o} {100 * n / max(tot, 1):.1f}%" for o, n in ops.most_common(12)))
            if st:
                lines.append("   stall samples: " + ", ".join(f"{k[6:]} {int(v)}" for k, v in st.most_common(8)))
        # top source lines
        src_rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass"))))
        hc = next((r for r in src_rows if r and r[0] == "Line No"), None)
        if hc:
            si = hc.index("Warp Stall Sampling (All Samples)")
            data = []
            fname = ""
            for r in src_rows:
                if r and r[0] in ("File Path", "File Name") and len(r) > 1:
                    fname = os.path.basename(r[1])
                # source-line rows only (the interleaved SASS rows have no line number)
                if len(r) == len(hc) and r[0].strip().isdigit() and r[si].strip().isdigit() and int(r[si]) > 0:
                    data.append((int(r[si]), f"{fname}:{r[0]}", r[1].strip()[:80]))
            tot = sum(x[0] for x in data)
            lines.append("   top source lines by stall samples:")
            for n, ln, s in sorted(data, reverse=True)[:10]:
                lines.append(f"     {100 * n / max(tot, 1):5.1f}%  {ln:>16s}  {s}")
    open(out, "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(tpath, "w"), indent=1)
    print(open(out).read())


if __name__ == "__main__":
    main()
