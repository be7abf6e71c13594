"""Table of the bench lines written by tools/run_configs.sh: python tools/configs_summary.py gpurun_out/r2_cfg_*.json"""
import json, sys, os
print("| point | q_nom | q_true | nnz | ms/step | select | adapt | expmv | Taylor frac (SURVEY bytes) | Taylor frac (bytes moved) | step frac (SURVEY 8d bytes) | e2e | parity vs reference | reference CPU |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for p in sys.argv[1:]:
    try:
        d = json.loads([l for l in open(p) if l.startswith("{")][-1])
    except Exception as e:
        print("|", os.path.basename(p), "| failed:", e, "|")
        continue
    name = os.path.basename(p).replace("r2_cfg_", "").replace(".json", "")
    ph, r, st = d["phase_ms_per_step"], d["roofline"], d["state"]
    cpu = d.get("cpu_baseline")
    par = "not run"
    ref = "not run"
    if cpu:
        pp = cpu["parity_on_sample"]
        par = "table + coefficients bit-exact" if pp["table_bit_exact"] and pp["coeff_bit_exact"] else "MISMATCH"
        ref = f"{cpu['value']:.4f} timesteps/s ({cpu['cores']} cores)"
    e2e = f"{d['e2e']['value']:.1f}/s" if d.get("e2e") else "-"
    print(f"| {name} | {d['config']['q_nom']:.0e} | {int(st['q_true_mean_over_timed_steps'])} | {int(st['nnz_mean_over_timed_steps'])} | "
          f"{d['ms_per_step']:.3f} | {ph['select_ms']:.3f} | {ph['grow_ms']:.3f} | {ph['expmv_ms']:.3f} | {r['frac']:.3f} | "
          f"{r['as_implemented']['frac']:.3f} | {d['roofline_step']['frac']:.3f} | {e2e} | {par} | {ref} |")
