import json, sys
for f in sys.argv[1:]:
    for line in open(f):
        line = line.strip()
        if not line.startswith('{'):
            if line: print('  |', line[:200])
            continue
        d = json.loads(line); r = d.get('roofline') or {}
        print(f"{f}: {d['config']['workload']} value={d['value']:.3e} ms/step={d.get('ms_per_step', 0):.3f} "
              f"frac={r.get('frac', 0):.4f} achieved={r.get('achieved', 0):.2f}TF hbm_frac={r.get('hbm_frac', 0):.3f} "
              f"p1/sweep={r.get('pass1_ms_per_sweep', 0):.3f}ms p2/sweep={r.get('pass2_ms_per_sweep', 0):.3f}ms "
              f"share={r.get('share_of_step')} launches={d.get('gpu_launches')}")
        print('   e2e', d.get('e2e'), ' clocks', d.get('clocks'))
        if d.get('cpu_baseline'): print('   cpu', d['cpu_baseline']['value'], d['cpu_baseline']['cores'])
