"""Summarise a BKT_TC_DEBUG per-chunk timeline (CTA 0 of one leafscan launch)."""
import statistics as st
import sys

rows = []
for l in open(sys.argv[1]):
    if not l.startswith('chunk'):
        continue
    f = l.split()
    rows.append({f[i]: int(f[i + 1]) for i in range(0, len(f) - 1, 2)})
tiles = {}
for r in rows:
    tiles.setdefault(r['tile'], []).append(r)
tl = sorted(tiles)
dur, gaps, work, wait = [], [], [], []
prev_end = None
for t in tl[:-1]:
    rs = tiles[t]
    s, e = rs[0]['epi_start'], rs[-1]['epi_done']
    dur.append(e - s)
    if prev_end is not None:
        gaps.append(s - prev_end)
    prev_end = e
    work += [r['epi_done'] - r['epi_ready'] for r in rs]
    wait += [r['epi_ready'] - r['epi_start'] for r in rs]
between = [rows[i + 1]['epi_start'] - rows[i]['epi_done'] for i in range(len(rows) - 1)
           if rows[i + 1]['tile'] == rows[i]['tile']]
print("chunks", len(rows), "tiles", len(tl), "chunks/tile", len(rows) / len(tl))
print("tile dur mean %.0f median %.0f" % (st.mean(dur), st.median(dur)))
print("tile gap mean %.0f median %.0f" % (st.mean(gaps), st.median(gaps)))
print("chunk work mean %.0f median %.0f p90 %d" % (st.mean(work), st.median(work), sorted(work)[int(.9 * len(work))]))
print("chunk wait mean %.0f median %.0f" % (st.mean(wait), st.median(wait)))
print("between chunks (same tile) mean %.0f median %.0f" % (st.mean(between), st.median(between)))
fw = [tiles[t][0]['epi_ready'] - tiles[t][0]['epi_start'] for t in tl[1:-1]]
print("first-chunk wait mean %.0f" % st.mean(fw))
tot = rows[-1]['epi_done'] - rows[0]['epi_start']
print("cycles/chunk %.0f" % (tot / len(rows)))

if 'ld0' in rows[0]:
    dtrip = [rows[i]['trips'] - rows[i - 1]['trips'] for i in range(1, len(rows))]
    dany = [rows[i]['anyg'] - rows[i - 1]['anyg'] for i in range(1, len(rows))]
    ld0 = [r['ld0'] - r['epi_ready'] for r in rows[1:]]
    g0 = [r['g0'] - r['ld0'] for r in rows[1:]]
    p2 = [r['g1'] - r['g0'] for r in rows[1:] if r['g1'] > 0]
    post = [r['epi_done'] - max(r['g0'], r['g1']) for r in rows[1:]]
    print("first tmem wait mean %.0f median %.0f" % (st.mean(ld0), st.median(ld0)))
    print("pass1 rest mean %.0f median %.0f" % (st.mean(g0), st.median(g0)))
    if p2:
        print("pass2 (%d chunks) mean %.0f median %.0f" % (len(p2), st.mean(p2), st.median(p2)))
    print("after last group (release) mean %.0f" % st.mean(post))
    clean = [rows[i]['epi_done'] - rows[i]['epi_ready'] for i in range(1, len(rows)) if dtrip[i - 1] == 0 and dany[i - 1] == 0]
    print("chunks with no survivor work: %d of %d, work mean %.0f median %.0f" % (len(clean), len(rows) - 1, st.mean(clean), st.median(clean)))
    per_trip = [(rows[i]['epi_done'] - rows[i]['epi_ready'], dtrip[i - 1], dany[i - 1]) for i in range(1, len(rows))]
    import numpy as np
    X = np.array([[1, t, a] for _, t, a in per_trip], float)
    y = np.array([w for w, _, _ in per_trip], float)
    coef = np.linalg.lstsq(X, y, rcond=None)[0]
    print("fit work = %.0f + %.0f*trips + %.0f*anygroups; mean trips %.2f anyg %.2f" % (coef[0], coef[1], coef[2], st.mean(dtrip), st.mean(dany)))
