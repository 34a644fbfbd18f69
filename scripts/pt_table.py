"""Per-pass table from the ncu launch lists written by scripts/pass_times.sh (timed step only)."""
import csv, collections, sys
for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]; ix = {k: i for i, k in enumerate(h)}
    d = collections.OrderedDict()
    for r in rows[1:]:
        if 'qsv_pass' not in r[ix['Kernel Name']]: continue
        d.setdefault(r[ix['ID']], {})[r[ix['Metric Name']]] = float(r[ix['Metric Value']].replace(',', ''))
    v = list(d.values()); v = v[len(v) // 2:]
    ms = [x['gpu__time_duration.sum'] / 1e6 for x in v]
    print(path, 'total %.2f' % sum(ms), ' '.join('%.2f' % t for t in ms))
    print('   fp64%', ' '.join('%.0f' % x['sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'] for x in v))
