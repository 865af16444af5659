"""Summaries of a bench JSON line and an ncu launch list (development)."""
import collections
import csv
import json
import sys


def bench(path):
    d = json.loads(open(path).read().strip().splitlines()[-1])
    print('value %.4e ms %.2f' % (d['value'], d['ms_per_step']), d.get('step_ms'))
    print('build', {k: round(v, 3) for k, v in d['build'].items()})
    print('query', {k: (round(v, 3) if isinstance(v, float) else v) for k, v in d['query'].items()})
    print('roof', {k: d['roofline'][k] for k in ('achieved', 'frac', 'kernel_ms')},
          'roofq', {k: d['roofline_query'][k] for k in ('achieved', 'frac')})
    print('clocks', d['clocks'], 'e2e', d.get('e2e', {}).get('ms_per_step'))
    if 'parity' in d:
        print('parity', {k: d['parity'][k] for k in ('users_sampled', 'disagreements', 'in_band_pairs')})
    for k, v in d.get('configs', {}).items():
        print(k, 'ms %.3f build %.3f contr %.3f q %.3f qf %.3f parity %s roof %.3f' % (
            v['ms_per_step'], v['build']['ms'], v['build']['contraction_ms'], v['query']['ms'],
            v['query']['filter_ms'], v['parity']['disagreements'], v['roofline']['frac']), v.get('step_ms'))


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
    agg = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ki].split('(')[0][:60]
        v = float(r[vi].replace(',', ''))
        v *= {'ms': 1e3, 'ns': 1e-3, 'us': 1.0, 'usecond': 1.0, 'msecond': 1e3, 'nsecond': 1e-3}.get(r[ui], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print('%-60s n=%4d total %9.1f us  avg %8.2f us  %.1f%%' % (k, c, v, v / c, 100 * v / tot))


if __name__ == '__main__':
    for p in sys.argv[1:]:
        (launches if p.endswith('.csv') else bench)(p)
