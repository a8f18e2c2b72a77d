"""Aggregate a TN_PROFILE_DUMP log (second run) per category and step shape."""
import collections, re, sys
lines = open(sys.argv[1]).read().split("-- second run --")[-1].splitlines()
agg = collections.defaultdict(lambda: [0, 0.0])
for l in lines:
    m = re.search(r"([\d.]+) ms\s+cat (\d)\s+(\S.*?) nb=(\d+) m=(\d+) n=(\d+) k=(\d+)", l)
    if not m:
        continue
    key = (m.group(3).split(",")[0][:12],) + tuple(map(int, m.groups()[3:]))
    agg[key][0] += 1
    agg[key][1] += float(m.group(1))
for key, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(key, "n=%d ms=%.1f" % (v[0], v[1]))
print([l for l in lines if l.startswith("{")][-1][:300])
