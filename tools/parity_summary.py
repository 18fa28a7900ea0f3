"""Summarise gpurun_out/parity_errors.jsonl (written by tests/conftest.py record_parity): per test
family the number of checks, the largest error and the share of its bound used.  Injected-fault
checks (expect = fail) must exceed their bound.  Usage: python tools/parity_summary.py FILE..."""
import collections
import json
import sys


def main(paths):
    seen = {}
    for p in paths:
        for line in open(p):
            r = json.loads(line)
            seen[r["test"]] = r
    fam = collections.defaultdict(list)
    for r in seen.values():
        name = r["test"]
        key = name.split("/")[0] if "/" in name else name.rsplit("_N", 1)[0].rsplit("_head", 1)[0]
        fam[key].append(r)
    print("%-44s %6s %11s %8s %7s" % ("family", "checks", "max err", "bound", "used"))
    for key in sorted(fam):
        rs = fam[key]
        worst = max(rs, key=lambda r: r["used"])
        tag = "  (fault injected: must exceed)" if worst.get("expect") == "fail" else ""
        print("%-44s %6d %11.3e %8.0e %6.1f%%%s" % (key, len(rs), worst["err"], worst["tol"], 100 * worst["used"], tag))
    clean = [r for r in seen.values() if r.get("expect") != "fail"]
    print("\n%d checks; largest share of a bound used by a clean check: %.1f%% (%s)" %
          (len(clean), 100 * max(r["used"] for r in clean), max(clean, key=lambda r: r["used"])["test"]))


if __name__ == "__main__":
    main(sys.argv[1:])
