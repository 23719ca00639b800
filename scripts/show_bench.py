import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'no json', e); continue
    print('==', f, {k: d.get(k) for k in ['value', 'ms_per_step', 'iters_per_s', 'gpu_launches', 'graph_build_s']})
    r = d['roofline']; print('  roof', r['kernel'], round(r['achieved'], 1), r['unit'], 'frac', round(r['frac'], 3))
    print('  clk', d['clocks'], 'e2e', round(d['e2e']['value'], 5), round(d['e2e']['ms_per_step'], 3))
    for k, v in d['kernels'].items():
        print('   %-12s %7.3f ms  %8s GB/s  %8s TF/s  x%.0f' % (k, v['ms_per_step'], None if v['GB_per_s'] is None else round(v['GB_per_s']), None if not v['TFLOP_per_s'] else round(v['TFLOP_per_s'], 1), v['launches_per_step']))
    if d.get('cpu_baseline'): print('  cpu', d['cpu_baseline']['value'], d['cpu_baseline']['cores'])
