"""Copy the judged profile summaries from gpurun_out/ into profiles/ (tracked).
usage: make_profiles.py TAG  (reads gpurun_out/TAG.* of scripts/gpu_round.sh, tr1.* of
scripts/gpu_traffic.sh and k_trace_b2 of the bounce-2 capture when present)."""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def ncu_details(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    open(out, "w").write(txt)


def ncu_raw(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    open(out, "w").write(txt)


def ncu_lines(rep, out):
    txt = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_lines.py"), rep, "40"],
                         capture_output=True, text=True).stdout
    open(out, "w").write(txt)


def traffic(csv_path):
    """DRAM bytes per k_trace launch from an ncu --metrics dram__bytes_* list."""
    rows = list(csv.reader(open(csv_path)))
    hdr, L = None, {}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            L.setdefault(int(d["ID"]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return [L[k] for k in sorted(L)]


def main():
    tag = sys.argv[1]
    os.makedirs(P, exist_ok=True)
    b = os.path.join(G, f"{tag}.bench.json")
    if os.path.exists(b):
        shutil.copy(b, os.path.join(P, "r01_bench_C2.json"))
    lc = os.path.join(G, f"{tag}.launches.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join(P, "r01_launches_C2.csv"))
        s = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "summarize_launches.py"), lc],
                           capture_output=True, text=True).stdout
        open(os.path.join(P, "r01_launches_C2_summary.txt"), "w").write(s)
    for rep, name in ((os.path.join(G, f"{tag}.k_trace.ncu-rep"), "k_trace_b0"),
                      (os.path.join(G, "k_trace_b2.ncu-rep"), "k_trace_b2"),
                      (os.path.join(G, "tr1.k_refine.ncu-rep"), "k_refine")):
        if os.path.exists(rep):
            ncu_details(rep, os.path.join(P, f"r01_ncu_{name}_details.csv"))
            ncu_raw(rep, os.path.join(P, f"r01_ncu_{name}_raw.csv"))
            ncu_lines(rep, os.path.join(P, f"r01_ncu_{name}_lines.txt"))
    t = os.path.join(G, "tr1.trace_dram.csv")
    if os.path.exists(t):
        shutil.copy(t, os.path.join(P, "r01_k_trace_dram_per_launch.csv"))
        L = traffic(t)
        # prof_step C2 2: rep 0 = launches 0-7 (4 primary + 4 fan bounces), rep 1 = 8-15
        prim = L[8:12]
        rd = sum(x["dram__bytes_read.sum"] for x in prim)
        wr = sum(x["dram__bytes_write.sum"] for x in prim)
        json.dump({"C2": {"kernel": "k_trace, the 4 primary bounces of one launch",
                          "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                          "per_bounce_dram_bytes": [x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in prim],
                          "per_bounce_l2_hit_pct": [x["lts__t_sector_hit_rate.pct"] for x in prim],
                          "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
                                    "--clock-control none -k regex:k_trace python scripts/prof_step.py C2 2 "
                                    "(scripts/gpu_traffic.sh), second repetition"}},
                  open(os.path.join(P, "r01_traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
