"""Stamp the DRAM traffic of one PageRank launch from an ncu capture into
profiles/pagerank_traffic.json (read by bench.py as roofline.traffic).

    python scripts/capture_traffic.py gpurun_out/<tag>/prof_pr.ncu-rep <tag> [workload kind iterations]

The capture must come from the tree it is stamped on: the file records the
kernel-source sha (csrc/tk_staged.cu + tk_internal.cuh) and bench.py ignores
it once the kernel source changes.  The capture command is the `ncu` pass of
scripts/gpu_session.sh (dram__bytes_read.sum + dram__bytes_write.sum on the
PageRank kernel of one C5 bench step).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rep, tag = sys.argv[1], sys.argv[2]
    workload, kind, iters = (sys.argv[3:6] + ["c5", "adjacent", "29"][len(sys.argv[3:6]):])
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    for r in rows[2:]:
        d = dict(zip(head, r))
        if "pagerank" not in d["Kernel Name"]:
            continue
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(d[m].replace(",", "")) * scale[units[head.index(m)]]
        import bench

        t = {"workload": workload, "kind": kind, "iterations": int(iters),
             "kernel": d["Kernel Name"], "dram_bytes_per_launch": int(b),
             "dram_read_bytes": float(d["dram__bytes_read.sum"]) * scale[units[head.index("dram__bytes_read.sum")]],
             "dram_write_bytes": float(d["dram__bytes_write.sum"]) * scale[units[head.index("dram__bytes_write.sum")]],
             "l2_hit_pct": float(d.get("lts__t_sector_hit_rate.pct", "nan")),
             "kernel_source_sha": bench.kernel_source_sha(),
             "source": f"ncu capture gpurun_out/{tag}/prof_pr.ncu-rep (scripts/gpu_session.sh ncu pass)"}
        with open(os.path.join(ROOT, "profiles", "pagerank_traffic.json"), "w") as f:
            json.dump(t, f, indent=1)
        print(json.dumps(t))
        return
    sys.exit("no pagerank kernel in " + rep)


if __name__ == "__main__":
    main()
