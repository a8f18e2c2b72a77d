# whole-K vs K-sliced GEMM on one step shape: sum of device time / DRAM reads over the
# GEMM + pack launches of the last of 3 contract_pair calls, for several pack caps
# usage: bash scripts/kslab_probe.sh m n k "caps"
m=$1; n=$2; k=$3
python scripts/prof_gemm.py $m $n $k > /dev/null 2>&1 || exit 1
for cap in $4; do
  TN_PACK_CAP_LOG2=$cap ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second \
      --clock-control none -k regex:"cgemm|pack_f16" --csv python scripts/prof_gemm.py $m $n $k 2>/dev/null > /tmp/kslab_$cap.csv
  python - $cap <<'PY'
import csv, sys
rows = list(csv.reader(open('/tmp/kslab_%s.csv' % sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; data = [r for r in rows[hi + 1:] if len(r) == len(h)]
ik, im, iv, iid = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
launches = {}
for r in data:
    launches.setdefault(int(r[iid]), {'k': r[ik]})[r[im]] = float(r[iv].replace(',', ''))
ids = sorted(launches); n = len(ids) // 3; last = [launches[i] for i in ids[-n:]]
t = sum(l['gpu__time_duration.sum'] for l in last) / 1e6
rd = sum(l['dram__bytes_read.sum'] for l in last) / 1e9; wr = sum(l['dram__bytes_write.sum'] for l in last) / 1e9
clk = sum(l['sm__cycles_elapsed.avg.per_second'] * l['gpu__time_duration.sum'] for l in last) / sum(l['gpu__time_duration.sum'] for l in last) / 1e9
print('cap=%s launches=%d time=%.1f ms dram read=%.1f GB write=%.1f GB clk=%.3f GHz' % (sys.argv[1], n, t, rd, wr, clk))
PY
done
