"""Markdown results table from a sweep JSONL (tools/sweep_r02.sh): python tools/results_table.py FILE"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
print("| workload | B | frames/s (enc+dec) | enc / dec | e2e | bpp | B=1 enc / dec ms | dominant (frac) |")
print("|---|---|---|---|---|---|---|---|")
for d in rows:
    if "workload_failed" in d:
        print(f"| {d['workload_failed']} | failed | | | | | | |")
        continue
    w = d["config"]["workload"].split(":")[0]
    lat = d.get("latency_b1") or {}
    r = d.get("roofline") or {}
    enc, dec = d.get("enc_fps"), d.get("dec_fps")
    ed = f"{enc:,.0f} / {dec:,.0f}" if enc else "—"
    b1 = f"{lat['enc_ms']:.2f} / {lat['dec_ms']:.2f}" if lat else "—"
    print(f"| {w} | {d['config']['frames_per_gpu_per_step']} | {d['value']:,.0f} | {ed} | {d['e2e']['value']:,.0f} | "
          f"{d['bpp']:.2f} | {b1} | {r.get('kernel')} ({r.get('frac', 0):.2f}) |")
