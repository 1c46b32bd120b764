python -c "
import json,sys
for line in open('gpurun_out/b.log'):
    if line.startswith('{'):
        d=json.loads(line)
        print('value', round(d['value']), 'ms/step', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value']), 'launches', d.get('gpu_launches'))
        r=d['roofline']; print('roofline', r['kernel'], round(r['achieved']), 'GB/s frac', round(r['frac'],3), 'share', round(r['share_of_step'],3))
        print('clocks', d['clocks'], 'cpu', d.get('cpu_baseline',{}).get('value'))
"
