import json,sys
for f in sys.argv[1:]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    print(f, round(d['value'],1), round(d['e2e']['value'],1), round(d['ms_per_step'],1), d['gpu_launches'], round(d['per_clip_latency']['p50_ms'],2))
    if '-v' in sys.argv: 
        for k,v in d['step_roofline']['families'].items(): print('   ',k, v['launches'], round(v['share'],3), round(v['ms'],1), round(v['hbm_frac'],2), round(v['fp64_frac'],2))
