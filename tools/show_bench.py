import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
sw = d.pop("sweep", []); rf = d.pop("roofline", {}); cfg = d.pop("config", {})
print(json.dumps({k: v for k, v in d.items()}, indent=None)[:1500])
print("roofline:", json.dumps(rf))
for s in sw:
    print(f"p={s['p']:.1f} keep={s['keep']:.3f} ms={s['ms_per_step']:.4f} dense-eq={s['dense_equiv_tflops']:.0f} exec={s['executed_tflops']:.0f} speedup={s['speedup_vs_dense']:.3f} vs1cta={s.get('speedup_vs_dense_1cta', 0):.3f} t/dense/keep={s['time_vs_dense_over_keep']:.3f}")
