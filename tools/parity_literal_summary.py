"""Summarise the literal residual-history rule (|rho'_k - rho_k| <= 1e-8 rho_k,
BASELINE.json north_star) logged by the GPU parity tests (MG_PARITY_LOG):
per test, how many cycles pass it, and the rounding-floor ratio tau_k / rho_k
of the cycles that do not (reading A20).
    python tools/parity_literal_summary.py profiles/r02/<tag>/parity_literal.jsonl"""
import collections
import json
import sys

per = collections.OrderedDict()
for line in open(sys.argv[1]):
    d = json.loads(line)
    t = d["tag"].split("::")[-1]
    r = per.setdefault(t, {"runs": 0, "cycles": 0, "literal": 0, "a20": 0, "min_fail_ratio": None,
                           "max_pass_diff": 0.0})
    r["runs"] += 1
    r["a20"] += bool(d["a20_pass"])
    for ok, diff, tr in zip(d["literal_per_cycle"], d["rel_diff_per_cycle"], d["tau_over_rho"]):
        r["cycles"] += 1
        if ok:
            r["literal"] += 1
            r["max_pass_diff"] = max(r["max_pass_diff"], diff)
        else:
            r["min_fail_ratio"] = tr if r["min_fail_ratio"] is None else min(r["min_fail_ratio"], tr)
print("| test | runs | A20 rule passed | cycles | literal rule passed | smallest tau_k/rho_k of a failing cycle |")
print("|---|---|---|---|---|---|")
for t, r in per.items():
    mf = "-" if r["min_fail_ratio"] is None else f"{r['min_fail_ratio']:.1e}"
    print(f"| {t} | {r['runs']} | {r['a20']}/{r['runs']} | {r['cycles']} | {r['literal']} | {mf} |")
