import sys, json
for line in sys.stdin:
    try: d = json.loads(line)
    except Exception: print(line.strip()[:300]); continue
    r = d.get('roofline') or {}
    print(d['config'].get('batch'), d['config'].get('preset'), 'qps', round(d['qps']), 'ms/step', round(d['ms_per_step'], 4),
          'lat', round(d.get('latency_ms', 0), 4), 'items/s %.3g' % d['value'],
          {k: r.get(k) for k in ('bound', 'achieved', 'frac', 'scan_ms_per_launch', 'merge_ms_per_launch')},
          'e2e %.3g' % d['e2e']['value'] if d.get('e2e') else '')
