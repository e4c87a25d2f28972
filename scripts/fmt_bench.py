import sys, json
for line in sys.stdin:
    try: d = json.loads(line)
    except Exception: print(line.strip()[:300]); continue
    print(d['config']['batch'], 'qps', round(d['qps']), 'ms/step', round(d['ms_per_step'],3), 'items/s %.3g' % d['value'], {k: d['roofline'][k] for k in ('bound','achieved','frac','hbm_frac','tensor_frac','scan_ms_per_launch','merge_ms_per_launch')} if d['roofline'] else None)
