"""Print the value and per-kernel launch times of bench.py JSON lines.  python tools/bench_show.py f1.json f2.json ..."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'unreadable', e)
        continue
    print('%-34s %9.1f %s  %.4f ms/step' % (f.split('/')[-1], d['value'], d['unit'], d['ms_per_step']))
    for k, v in d.get('kernels', {}).items():
        print('    %-22s %7.1f us x%.0f  share %.3f  hbm %.3f' % (k, v['avg_launch_us'], v['launches_per_step'], v['share'], v['hbm_frac']))
