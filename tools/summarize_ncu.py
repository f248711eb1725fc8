"""Turn ncu outputs (gpurun_out/) into committed summaries under profiles/ (run on the CPU side)."""
import csv, collections, json, subprocess, sys, io


def launches(csv_path, out_md, title):
    rows = list(csv.reader(open(csv_path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]; data = rows[hi + 1:]
    ki = h.index('Kernel Name'); mi = h.index('Metric Value')
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= mi: continue
        agg[r[ki].split('(')[0]][0] += 1
        agg[r[ki].split('(')[0]][1] += float(r[mi].replace(',', ''))
    tot = sum(v[1] for v in agg.values())
    with open(out_md, 'w') as f:
        f.write(f"# {title}\n\nncu `--metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised "
                "launches: compare SHARES, not absolute times). Source: `{}`.\n\n".format(csv_path))
        f.write("| kernel | launches | total ms | avg us | share |\n|---|---:|---:|---:|---:|\n")
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"| `{k}` | {v[0]} | {v[1]/1e6:.2f} | {v[1]/v[0]/1e3:.2f} | {v[1]/tot:.3f} |\n")
    return agg, tot


def full(rep, out_md, title, algo_bytes=None):
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw))); h, u, v = r[0], r[1], r[2]
    get = lambda k: (float(v[h.index(k)].replace(',', '')), u[h.index(k)]) if k in h else (None, None)
    det = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    d = list(csv.reader(io.StringIO(det))); dh = d[0]
    si, mi, vi, ui = (dh.index(x) for x in ('Section Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
    keep = ('GPU Speed Of Light Throughput', 'Memory Workload Analysis', 'Compute Workload Analysis', 'Occupancy',
            'Scheduler Statistics', 'Warp State Statistics', 'Launch Statistics')
    t, tu = get('gpu__time_duration.sum')
    rd, rdu = get('dram__bytes_read.sum')
    wr, wru = get('dram__bytes_write.sum')
    scale = {'Gbyte': 1e9, 'Mbyte': 1e6, 'Kbyte': 1e3, 'byte': 1.0}
    traffic = rd * scale[rdu] + wr * scale[wru]
    with open(out_md, 'w') as f:
        f.write(f"# {title}\n\n`ncu --set full --clock-control none --import-source on`, report `{rep}`.\n\n")
        f.write(f"* duration: {t} {tu}\n* dram read: {rd} {rdu}, write: {wr} {wru} -> traffic {traffic/1e9:.3f} GB/launch\n")
        if algo_bytes:
            f.write(f"* algorithmic bytes per launch (DESIGN.md model): {algo_bytes/1e9:.3f} GB "
                    f"-> traffic / algorithmic = {traffic/algo_bytes:.2f}\n")
        f.write("\n| section | metric | value | unit |\n|---|---|---:|---|\n")
        for row in d[1:]:
            if row[si] in keep:
                f.write(f"| {row[si]} | {row[mi]} | {row[vi]} | {row[ui]} |\n")
    return traffic


if __name__ == '__main__':
    import os
    rnd = sys.argv[1] if len(sys.argv) > 1 else 'round2'
    go = 'gpurun_out'
    bench = json.loads(open(f'{go}/bench_c5.json').read().strip().splitlines()[-1])
    algo = {bench['roofline']['kernel'].split()[0]: bench['roofline']['algorithmic_bytes_per_launch'],
            bench['roofline_secondary']['kernel'].split()[0]: bench['roofline_secondary']['algorithmic_bytes_per_launch']}
    launches(f'{go}/launches_bench_c5.csv', f'profiles/{rnd}_launches_bench_c5.md',
             f'{rnd} launch list: `bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline` (config c5)')
    if os.path.exists(f'{go}/launches_bench_c4.csv') and os.path.getsize(f'{go}/launches_bench_c4.csv') > 1000:
        launches(f'{go}/launches_bench_c4.csv', f'profiles/{rnd}_launches_bench_c4.md',
                 f'{rnd} launch list: `bench.py --config c4 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline` (config c4)')
    tr = {}
    try:   # keep the figures of kernels that were not captured again
        tr = json.load(open('profiles/traffic.json'))['dram_bytes_per_launch']
    except Exception:
        pass
    tr['k_prec_coop'] = full(f'{go}/r2_k_prec_coop.ncu-rep', f'profiles/{rnd}_prec_coop_c5.md',
                             f'{rnd}: k_prec_coop (C5 preconditioner, one cooperative launch), config c5',
                             algo_bytes=algo.get('k_prec_coop'))
    if os.path.exists(f'{go}/r2_k_schur_explicit.ncu-rep'):
        tr['k_schur_explicit'] = full(f'{go}/r2_k_schur_explicit.ncu-rep', f'profiles/{rnd}_schur_explicit_c5.md',
                                      f'{rnd}: k_schur_explicit (C2 explicit local Schur apply), config c5',
                                      algo_bytes=algo.get('k_schur_explicit'))
    json.dump({"config": "c5", "n_gpus": 1, "dram_bytes_per_launch": tr,
               "source": [f"profiles/{rnd}_prec_coop_c5.md", f"profiles/{rnd}_schur_explicit_c5.md"]},
              open('profiles/traffic.json', 'w'), indent=1)
    print('traffic', tr)
    for k in ('k_prec_coop', 'k_schur_blk', 'k_band_chol_panel'):
        rep = f'{go}/r2_c4_{k}.ncu-rep'
        if os.path.exists(rep):
            t = full(rep, f'profiles/{rnd}_c4_{k}.md', f'{rnd}: {k}, config c4 (3D)')
            print(k, 'c4 traffic', t)
