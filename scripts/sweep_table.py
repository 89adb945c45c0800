"""Markdown table of a sweep.py jsonl (tokens/s, MFU, measured / replayed / Eq. 7 bubble, vs 1F1B)."""
import json
import sys


def main(path):
    rows = [json.loads(l) for l in open(path) if l.strip()]
    ref = {r["sweep_beta"]: r["value"] for r in rows if r.get("sweep_schedule") == "1f1b" and r.get("value")}
    print("| beta (seq/GPU) | schedule | tokens/s | MFU spec | MFU measured-peak | bubble measured | "
          "bubble replayed | bubble Eq.7 | vs 1F1B |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r in sorted(rows, key=lambda r: (r["sweep_beta"], r["sweep_schedule"])):
        if not r.get("value"):
            print(f"| {r['sweep_beta']} | {r['sweep_schedule']} | error: {r.get('error', '?')[:60]} |")
            continue
        b, m = r["bubble_fraction"], r["mfu"]
        vs = r["value"] / ref[r["sweep_beta"]] if r["sweep_beta"] in ref else float("nan")
        print(f"| {r['sweep_beta']} | {r['sweep_schedule']} | {r['value']:,.0f} | {m['vs_spec_2250TF']:.3f} | "
              f"{m['vs_measured_burst']:.3f} | {b['measured']:.3f} | {b['simulated_with_measured_timing']:.3f} | "
              f"{b['eq7']:.3f} | {vs:.2f} |")


if __name__ == "__main__":
    main(sys.argv[1])
