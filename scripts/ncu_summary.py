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


_SCALE = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'Tbyte': 1e12,
          'ns': 1e-3, 'us': 1, 'ms': 1e3, 'usecond': 1, 'nsecond': 1e-3, 'msecond': 1e3}


def norm(d, key):
    """Value of metric `key` in bytes (byte metrics) or microseconds (time)."""
    full = [k for k in d['units'] if k.endswith(key)]
    if not full or not d.get(key):
        return None
    return float(d[key].replace(',', '')) * _SCALE.get(d['units'][full[0]], 1)


def summary(d):
    t = norm(d, 'time_duration.sum')
    rd, wr = norm(d, 'bytes_read.sum'), norm(d, 'bytes_write.sum')
    return {'kernel': d['Kernel Name'].split('(')[0].replace('void ', '').replace('(anonymous namespace)::', '')
            .replace('unnamed>::', ''), 'us': t, 'dram_read_GB': rd / 1e9, 'dram_write_GB': wr / 1e9,
            'dram_TBps': (rd + wr) / t / 1e6, 'dram_pct': d.get('dram_throughput.avg.pct_of_peak_sustained_elapsed'),
            'sm_pct': d.get('throughput.avg.pct_of_peak_sustained_elapsed'), 'regs': d.get('registers_per_thread'),
            'warps_active_pct': d.get('warps_active.avg.pct_of_peak_sustained_active'),
            'l2_hit_pct': d.get('t_sector_hit_rate.pct')}


if __name__ == '__main__':
    if sys.argv[1] == 'list':
        out, per_step = launches(sys.argv[2], int(sys.argv[3]))
        for k, c, t, a, s in out[:25]:
            print(f"{k:48s} n={c:4d} total={t:8.3f} ms avg={a:8.1f} us share={s:5.1f}%")
        print('serialized ms/step', per_step)
    elif sys.argv[1] == 'traffic':
        # traffic <out.json> class=rep ... : dram bytes per launch per kernel class
        import json
        res = {}
        for arg in sys.argv[3:]:
            cls, rep = arg.split('=', 1)
            for d in raw(rep):
                sm = summary(d)
                res[cls] = {'bytes': (sm['dram_read_GB'] + sm['dram_write_GB']) * 1e9, **sm,
                            'source': rep.split('/')[-1]}
        json.dump(res, open(sys.argv[2], 'w'), indent=1)
        for k, v in res.items():
            print(f"{k:10s} {v['kernel'][:34]:34s} {v['us']:8.1f} us  rd {v['dram_read_GB']:.3f} GB  wr "
                  f"{v['dram_write_GB']:.3f} GB  {v['dram_TBps']:.2f} TB/s  dram% {v['dram_pct'][:5]}  "
                  f"sm% {v['sm_pct'][:5]}  regs {v['regs']}  warps% {v['warps_active_pct'][:5]}  L2hit {v['l2_hit_pct'][:5]}")
    else:
        for d in raw(sys.argv[2]):
            print(summary(d))
