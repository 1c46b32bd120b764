#!/bin/bash
# one-line summary of each bench JSON line in the given logs (default gpurun_out/b.log)
for f in "${@:-gpurun_out/b.log}"; do python - "$f" <<'PY'
import json, sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d = json.loads(line)
        if 'unavailable' in d or d.get('impl') == 'reference':
            print(sys.argv[1], 'reference', d.get('value'), d.get('unavailable', '')); continue
        print(sys.argv[1], 'value', round(d['value']), 'ms/step', round(d['ms_per_step'], 3), 'e2e', round(d['e2e']['value']),
              'launches', d.get('gpu_launches'), 'clocks', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'),
              'cpu', (d.get('cpu_baseline') or {}).get('value'))
        for k in ('roofline', 'roofline_other'):
            r = d.get(k)
            if r:
                print('   ', k, r['kernel'][:40], round(r['achieved']), r['unit'], 'frac', round(r['frac'], 3),
                      'share', round(r['share_of_step'] or 0, 3))
PY
done
