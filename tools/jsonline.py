"""Print the key numbers of bench.py JSON lines read from stdin (one per line)."""
import json
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else ""
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    rf = d.get("roofline") or {}
    e2e = d.get("e2e") or {}
    print(tag, d.get("config", {}).get("workload", "")[:40], "value", round(d.get("value") or 0),
          "ms/step", round(d.get("ms_per_step") or 0), "frac", rf.get("frac"),
          "kernel", (rf.get("kernel") or "")[:60], "e2e", round(e2e.get("value") or 0),
          "clk", (d.get("clocks") or {}).get("sm_mhz"))
