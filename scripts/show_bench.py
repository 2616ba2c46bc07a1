"""Print value / e2e / per-layer ms of bench JSON lines in the given log files."""
import json, sys
for f in sys.argv[1:]:
    ls = [x for x in open(f) if x.startswith('{')]
    if not ls:
        print(f, 'no JSON line'); continue
    d = json.loads(ls[-1])
    lay = ' '.join(f"{k}={v['ms_per_launch']:.3f}" for k, v in d.get('layers', {}).items())
    print(f"{f}: {d['value']:.1f} fps, e2e {d['e2e']['value']:.1f}, {d.get('clocks', {}).get('sm_mhz')} MHz | {lay}")
