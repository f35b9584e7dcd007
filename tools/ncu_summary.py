"""Key metrics of ncu --set full reports -> JSON (the summaries committed under profiles/)."""
import csv, json, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct"]


def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                d[k] = f"{v[i]} {units[i]}".strip()
        stalls = {}
        for i, x in enumerate(h):
            if x.startswith("smsp__average_warps_issue_stalled") and x.endswith("per_issue_active.ratio"):
                try:
                    if float(v[i]) >= 0.2:
                        stalls[x[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v[i])
                except ValueError:
                    pass
        d["stalls_per_issue"] = stalls
        res.append(d)
    return res


def build_hash():
    """md5 of the in-tree library the captures ran."""
    import hashlib, os
    lib = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_2311_01135_b200", "libqm1b_b200.so")
    return hashlib.md5(open(lib, "rb").read()).hexdigest()


def source_hash(root=None):
    """md5 over the kernel sources the library is built from (csrc/*.cu, *.cuh, Makefile and the C
    header, names and contents in sorted order).  nvcc's output is not bit-reproducible between
    builds of the same sources, so bench.py matches a capture to the running code by this hash
    (the library md5 is kept as well)."""
    import glob, hashlib, os
    root = root or os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    c = os.path.join(root, "paper_2311_01135_b200", "csrc")
    files = sorted(glob.glob(os.path.join(c, "*.cu")) + glob.glob(os.path.join(c, "*.cuh")) +
                   [os.path.join(c, "Makefile"), os.path.join(root, "include", "qm1b_b200.h")])
    h = hashlib.md5()
    for f in files:
        h.update(os.path.relpath(f, root).encode())
        h.update(open(f, "rb").read())
    return h.hexdigest()


if __name__ == "__main__":
    out = {"_build": build_hash(), "_src": source_hash()}
    for arg in sys.argv[2:]:
        name, rep = arg.split("=", 1)
        out[name] = summarize(rep)
    json.dump(out, open(sys.argv[1], "w"), indent=1)
