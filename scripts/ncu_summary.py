"""Summaries of ncu outputs: launch-list shares and per-kernel raw metrics."""
import collections, csv, subprocess, sys


def launches(path, steps):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]; data = rows[hi + 1:]
    ki, vi = h.index('Kernel Name'), h.index('Metric Value')
    agg = collections.OrderedDict(); tot = 0.0
    for r in data:
        if len(r) <= vi: continue
        v = float(r[vi].replace(',', ''))
        short = r[ki].split('(')[0].replace('void ', '').replace('(anonymous namespace)::', '').replace('unnamed>::', '')[:48]
        a = agg.setdefault(short, [0, 0.0]); a[0] += 1; a[1] += v; tot += v
    out = []
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append((k, c, t / 1e6, t / c / 1e3, t / tot * 100))
    return out, tot / 1e6 / steps


def raw(rep):
    txt = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units, data = rows[0], rows[1], rows[2:]
    want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
            'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
            'launch__registers_per_thread', 'sm__warps_active.avg.pct_of_peak_sustained_active',
            'lts__t_sector_hit_rate.pct', 'sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active',
            'sm__inst_executed_pipe_tensor_op_hmma.avg.pct_of_peak_sustained_active']
    idx = {w: h.index(w) for w in want if w in h}
    res = []
    for r in data:
        d = {w.split('__')[-1] if '__' in w else w: r[i] for w, i in idx.items()}
        d['units'] = {w: units[i] for w, i in idx.items()}
        res.append(d)
    return res


if __name__ == '__main__':
    if sys.argv[1] == 'list':
        out, per_step = launches(sys.argv[2], int(sys.argv[3]))
        for k, c, t, a, s in out[:25]:
            print(f"{k:48s} n={c:4d} total={t:8.3f} ms avg={a:8.1f} us share={s:5.1f}%")
        print('serialized ms/step', per_step)
    else:
        for d in raw(sys.argv[2]):
            print(d['Kernel Name'][:40].replace('(anonymous namespace)::', ''), '| t=%s ms | rd=%s wr=%s GB | dram%%=%s sm%%=%s | regs=%s warps%%=%s L2hit=%s' % (
                d.get('time_duration.sum'), d.get('bytes_read.sum'), d.get('bytes_write.sum'),
                d.get('dram_throughput.avg.pct_of_peak_sustained_elapsed', '')[:5], d.get('throughput.avg.pct_of_peak_sustained_elapsed', '')[:5],
                d.get('registers_per_thread'), d.get('warps_active.avg.pct_of_peak_sustained_active', '')[:5], d.get('t_sector_hit_rate.pct', '')[:5]))
