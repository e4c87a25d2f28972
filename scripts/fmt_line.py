"""One-line summary of a bench.py JSON line (stdin)."""
import json
import sys

d = json.loads(sys.stdin.read())
r = d.get("roofline") or {}
lp = d.get("latency_pct_ms") or {}
u = d.get("updates") or {}
print(d["config"]["workload"], "| ms", round(d["ms_per_step"], 4), "| qps", round(d.get("qps", 0), 1),
      "| value %.3g" % d["value"], "| frac", r.get("frac"), r.get("bound"), "| scan_ms", r.get("scan_ms_per_launch"),
      "| p50/p95", round(lp.get("p50", 0), 4), round(lp.get("p95", 0), 4),
      "| upd", (u.get("calls_in_timed_region"), round(u.get("update_call_ms", 0), 4)) if u else "-",
      "| e2e %.3g" % d["e2e"]["value"], "| clk", d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
