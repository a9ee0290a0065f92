"""Per-launch numbers bench.py folds into `roofline` (profiles/ncu_config<c>.json) from an ncu --set full report.
Usage: python tools/ncu_to_json.py report.ncu-rep <key>=<kernel-regex> [...] --source "<text>" > out.json
Each key gets <key>_dram_bytes_per_launch, <key>_issue_slot_util, <key>_active_lanes_per_instr, <key>_ms_ncu from the
first kernel whose name matches its regex."""
import csv
import io
import json
import re
import subprocess
import sys


def main():
    rep = sys.argv[1]
    pairs = [a.split("=", 1) for a in sys.argv[2:] if "=" in a and not a.startswith("--")]
    src = sys.argv[sys.argv.index("--source") + 1] if "--source" in sys.argv else rep
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1,
             "%": 0.01, "": 1}
    res = {}
    for key, rx in pairs:
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            if not re.search(rx, d.get("Kernel Name", "")):
                continue
            u = dict(zip(hdr, units))

            def val(m):
                return float(d[m].replace(",", "")) * scale.get(u[m], 1)

            res[f"{key}_dram_bytes_per_launch"] = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
            res[f"{key}_issue_slot_util"] = round(val("sm__inst_issued.avg.pct_of_peak_sustained_active"), 4)
            res[f"{key}_active_lanes_per_instr"] = round(val("smsp__thread_inst_executed_per_inst_executed.ratio"), 2)
            res[f"{key}_ms_ncu"] = val("gpu__time_duration.sum")
            break
    res["source"] = src
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
