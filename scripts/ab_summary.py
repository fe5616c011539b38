"""Print the phases of the A/B bench lines of gpurun_out/<tag>."""
import glob, json, os, sys
for f in sorted(glob.glob(f"gpurun_out/{sys.argv[1]}/bench_*.json")):
    env = open(f.replace(".json", ".env")).read().strip() if os.path.exists(f.replace(".json", ".env")) else ""
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, env, "FAILED", open(f.replace(".json", ".err")).read()[-300:]); continue
    ham = d.get("hamming") or {}
    print(os.path.basename(f), f"[{env}]", d["config"].get("kind"), d["ms_per_step"], d.get("phases_ms"),
          "ham:", ham.get("phases_ms"), "clk", (d.get("clocks") or {}).get("sm_mhz"))
