#!/usr/bin/env python
"""Markdown summary of one evidence refresh (tools/refresh_profiles.sh with TAG=<tag>) for profiles/:
the bench line of every config (value, e2e, step time, the dominant class and its roofline, the
whole-step fraction, executed work, conformance flips, clocks), the oracle reference arm, the C4
launch list and the key metrics of the steady-state --set full captures.

    python tools/round_summary.py <tag> > profiles/r02/ncu_<tag>.md
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary  # noqa: E402

O = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "gpurun_out")


def last_json(path):
    if not os.path.exists(path):
        return None
    for line in reversed(open(path).read().strip().splitlines()):
        line = line.strip()
        if line.startswith("{"):
            return json.loads(line)
    return None


def main(tag):
    out = ["# Evidence refresh `%s`" % tag, "",
           "Captured on one B200 with `TAG=%s tools/refresh_profiles.sh` and `tools/ncu_steady.sh`. ncu numbers are "
           "serialised replays with `--clock-control none`: compare shares, utilisations and DRAM bytes with the "
           "bench line, not absolute times." % tag, "",
           "| config | EM it/s | e2e | ms/step | dominant class | bound | frac | step frac (HBM) | work | "
           "executed RHS applies/s | conformance flips | SM MHz | throttle |",
           "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    lines = []
    for wl in ("C4", "C1", "C2", "C3", "C5"):
        d = last_json(os.path.join(O, "%s_bench_%s.json" % (tag, wl)))
        if not d:
            out.append("| %s | (missing) |||||||||||" % wl)
            continue
        lines.append(d)
        r = d["roofline"]
        conf = d.get("conformance") or {}
        out.append("| %s | %.2f | %.2f | %.2f | %s | %s | %.3f | %.3f | %.2f | %.0f | %s | %s | %s |" % (
            d["config"]["workload"], d["value"], d["e2e"]["value"], d["ms_per_step"], r.get("kernel"), r["bound"],
            r["frac"], r["step"]["frac"], r.get("work_fraction", 1.0), d.get("rhs_applies_per_s", 0),
            conf.get("support_flips"), d["clocks"].get("sm_mhz"), ",".join(d["clocks"].get("reasons", [])) or "-"))
    ref = last_json(os.path.join(O, "%s_ref_C4.json" % tag))
    if ref:
        lines.append(ref)
        out.append("| reference arm (fp64 oracle, C4 sample, %s cores) | %.5f | | | | | | | | | | | |" % (
            ref.get("cpu_baseline", {}).get("cores"), ref["value"]))
    out += ["", "Pipe utilisation of each dominant kernel (`roofline.ncu_pipes`, % of peak while active):", ""]
    for d in lines:
        p = d.get("roofline", {}).get("ncu_pipes")
        if p:
            out.append("- %s `%s`: %s" % (d["config"]["workload"], d["roofline"]["kernel"],
                                           ", ".join("%s %s" % (k, v) for k, v in p.items() if k != "source")))
    lc = os.path.join(O, "%s_launches_C4.csv" % tag)
    if os.path.exists(lc):
        out += ["", "## C4 launch list (one timed E-step, serialised)", "", ncu_summary.launches(lc)]
    for wl in ("C4", "C3", "C5"):
        rep = os.path.join(O, "%s_%s_full.ncu-rep" % (tag, wl))
        if os.path.exists(rep):
            out += ["", "## --set full key metrics, %s (steady state)" % wl, "", ncu_summary.full(rep)]
    print("\n".join(out))
    with open(os.path.join(O, "%s_bench_lines.jsonl" % tag), "w") as f:
        for d in lines:
            f.write(json.dumps(d) + "\n")


if __name__ == "__main__":
    main(sys.argv[1])
