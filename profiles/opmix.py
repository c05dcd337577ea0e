"""SASS instruction mix per event-point from an ncu source page (the profile script's
src_<workload>.csv.gz): python profiles/opmix.py src.csv.gz <event-points per launch>.
Warp-level executed instructions x 32 / event-points = thread instructions per event-point."""
import csv, gzip, sys, re, collections
f = sys.argv[1]; evpt = float(sys.argv[2])
rows = list(csv.reader(gzip.open(f, 'rt')))
hdr = rows[1]; ia = hdr.index("Source"); ie = hdr.index("Instructions Executed"); isamp = hdr.index("# Samples")
mix = collections.Counter(); tot = 0; hot = []
for r in rows[2:]:
    if len(r) <= ie: continue
    try: n = int(r[ie])
    except: continue
    op = r[ia].strip()
    m = re.match(r'(@!?U?P\w+\s+)?([A-Z0-9_.]+)', op)
    name = m.group(2) if m else op
    base = name.split('.')[0]
    mix[base] += n; tot += n
    hot.append((n, int(r[isamp] or 0), op))
warp_per = 32.0 / evpt
print("total instr per ev*pt: %.2f" % (tot * warp_per))
for k, v in mix.most_common(40):
    print("%-10s %6.2f" % (k, v * warp_per))
