# per-path device time (ncu launch list) of configs[3]'s non-DMMA steps and neighbours;
# each call runs the step twice (the second is summed)
python -c "import __graft_entry__ as g; g.build()" || exit 1
for s in "10 4 4 7" "0 0 0 20" "11 7 7 2" "4 8 8 1" "8 4 4 8"; do
  for p in small skinny wide tc; do
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/l.csv python scripts/probes/path_probe.py $s c128 $p > /tmp/o.txt 2>&1
    python - "$s" $p <<'PY'
import csv, sys
rows = list(csv.reader(open('/tmp/l.csv')))
try:
    h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
except StopIteration:
    print(sys.argv[1], sys.argv[2], 'refused/no kernels'); sys.exit()
H = rows[h]; ki, vi, ui = H.index('Kernel Name'), H.index('Metric Value'), H.index('Metric Unit')
ks = [(r[ki].split('(')[0][-40:], float(r[vi].replace(',', '')) * {'ns': 1e-3, 'us': 1, 'usecond': 1, 'ms': 1e3, 'msecond': 1e3, 'nsecond': 1e-3}.get(r[ui], 1)) for r in rows[h + 1:] if len(r) > vi and ('tnd::' in r[ki] or 'tc::' in r[ki])]
half = ks[len(ks) // 2:]
print(sys.argv[1], sys.argv[2], f"{sum(t for _, t in half):.1f} us", [(n.split('::')[-1][:28], round(t, 1)) for n, t in half])
PY
  done
done
