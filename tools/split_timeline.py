"""Summarise a BKT_SPLIT_DEBUG timeline (CTA 0 of one split-scan launch)."""
import statistics as st
import sys

tiles, chunks = [], []
for l in open(sys.argv[1]):
    f = l.split()
    if l.startswith('stile'):
        tiles.append({f[i]: int(f[i + 1]) for i in range(2, len(f) - 1, 2)})
    elif l.startswith('schunk'):
        chunks.append({f[i]: int(f[i + 1]) for i in range(2, len(f) - 1, 2)})
if not chunks:
    sys.exit("no timeline")
span = chunks[-1]['edone'] - chunks[0]['ewait']
print(f"tiles {len(tiles)} chunks {len(chunks)} cycles/chunk {span / len(chunks):.0f}")
def m(xs):
    return f"mean {st.mean(xs):.0f} median {st.median(xs):.0f}"
print("epilogue tfull wait   ", m([c['eready'] - c['ewait'] for c in chunks]))
print("epilogue chunk work   ", m([c['edone'] - c['eready'] for c in chunks]))
print("between chunks        ", m([chunks[i + 1]['ewait'] - chunks[i]['edone'] for i in range(len(chunks) - 1)]))
print("TMA issue -> full     ", m([c['full'] - c['tma'] for c in chunks]))
print("full -> MMA committed ", m([c['mma'] - c['full'] for c in chunks]))
print("MMA committed -> epi ready", m([c['eready'] - c['mma'] for c in chunks]))
print("TMA issue lead (eready - tma)", m([c['eready'] - c['tma'] for c in chunks]))
tt = [t for t in tiles if t['eready'] >= 0]
print("epilogue afull wait   ", m([t['eready'] - t['ewait'] for t in tt]))
print("A published -> epi needs it (slack)", m([t['ewait'] - t['pub'] for t in tt]))
