python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for w in ${WL:-A1 V1 V2}; do python bench.py --workload $w --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.rstrip()); continue
  print(d['config']['workload'], round(d['value']), 'ms/step', round(d['ms_per_step']*1e3,1), 'roof', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['roofline']['launch'], round(d['roofline']['avg_launch_us'],1), 'e2e', round(d['e2e']['value']), d['config']['launches'][0]['kernel'], d['clocks']['sm_mhz'])
"; done
