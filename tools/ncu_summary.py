"""Summarise an `ncu --set full` report (.ncu-rep) into the text committed under
profiles/: per kernel the headline counters, the top stall reasons and (optionally)
the DRAM bytes per launch merged into profiles/<traffic json> (bench.py's
roofline.traffic).

    python tools/ncu_summary.py gpurun_out/fused2.ncu-rep profiles/r1_ncu_fused.txt \
        [--traffic profiles/r1_ncu_traffic.json] [--header "command line ..."]
"""
import argparse
import csv
import io
import json
import re
import subprocess

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__grid_size",
    "launch__block_size",
    "launch__cluster_dim_x",
    "launch__shared_mem_per_block_dynamic",
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--traffic", default=None)
    ap.add_argument("--header", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = []
    if a.header:
        lines.append("# " + a.header)
    lines.append("# ncu --set full, cold-cache serialised replay: use shares / counters, not absolute times")
    traffic = {}
    for r in data:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?")
        lines.append("")
        lines.append("kernel: " + name)
        for k in KEYS:
            if k in d:
                lines.append(f"  {k:70s} {d[k]} {u.get(k, '')}")
        st = []
        for k in hdr:
            m = re.match(r"smsp__average_warps_issue_stalled_(.+)_per_issue_active\.ratio$", k)
            if m and d.get(k):
                st.append((m.group(1), float(d[k])))
        st.sort(key=lambda x: -x[1])
        lines.append("  top stall reasons (warps per issue): " +
                     ", ".join(f"{n}={v:.2f}" for n, v in st[:8]))
        short = re.sub(r"^.*?(k_[A-Za-z0-9_]+).*$", r"\1", name)

        def mb(k):
            v = float(d[k])
            unit = u.get(k, "")
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)

        if "dram__bytes_read.sum" in d:
            traffic[short] = {"dram_bytes_per_launch": mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"),
                              "dram_read": mb("dram__bytes_read.sum"), "dram_write": mb("dram__bytes_write.sum"),
                              "capture": a.out}
    with open(a.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if a.traffic:
        try:
            with open(a.traffic) as f:
                old = json.load(f)
        except Exception:
            old = {}
        old.update(traffic)
        with open(a.traffic, "w") as f:
            json.dump(old, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
