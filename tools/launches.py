import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ii = h.index('ID')
for r in rows[hdr + 1:]:
    print(r[ii], r[ki][:70], r[vi])
