import sys, statistics as st, bisect
tiles, chunks = [], []
for l in open(sys.argv[1]):
    f = l.split()
    if l.startswith('stile'):
        tiles.append({f[i]: int(f[i + 1]) for i in range(2, len(f) - 1, 2)})
    elif l.startswith('schunk'):
        chunks.append({f[i]: int(f[i + 1]) for i in range(2, len(f) - 1, 2)})
er = [t['eready'] for t in tiles]
first, rest = [], []
firstw, restw = [], []
betw_first = []
prev_tile = -1
for gi, c in enumerate(chunks):
    ti = bisect.bisect_right(er, c['ewait']) - 1
    isfirst = ti != prev_tile
    prev_tile = ti
    (first if isfirst else rest).append(c['eready'] - c['ewait'])
    (firstw if isfirst else restw).append(c['edone'] - c['eready'])
    if isfirst and gi > 0:
        betw_first.append(c['ewait'] - chunks[gi-1]['edone'])
def m(x): return f"n {len(x)} mean {st.mean(x):.0f} median {st.median(x):.0f}"
print("tfull wait, first chunk of tile:", m(first))
print("tfull wait, other chunks:       ", m(rest))
print("work, first chunk:", m(firstw))
print("work, other:      ", m(restw))
print("gap before first chunk of tile (prev edone -> ewait):", m(betw_first))
# tile-level: MMA ready (mready) vs epilogue wants (ewait)
print("afull: eready - ewait", m([t['eready']-t['ewait'] for t in tiles if t['eready']>=0]))
a_, b_ = [], []
ew = [t['ewait'] for t in tiles]
for gi, c in enumerate(chunks):
    ti = bisect.bisect_right(er, c['ewait']) - 1
    if gi == 0: continue
    prev = chunks[gi-1]
    pti = bisect.bisect_right(er, prev['ewait']) - 1
    if ti != pti:
        t = tiles[ti]
        a_.append(t['ewait'] - prev['edone'])
        b_.append(c['ewait'] - t['eready'])
print("prev chunk edone -> tile ewait:", m(a_))
print("tile eready -> first chunk ewait:", m(b_))
if 'esetup' in tiles[0]:
    s1, s2, s3 = [], [], []
    for gi, c in enumerate(chunks):
        if gi == 0: continue
        ti = bisect.bisect_right(er, c['ewait']) - 1
        pti = bisect.bisect_right(er, chunks[gi-1]['ewait']) - 1
        if ti != pti:
            t = tiles[ti]
            s1.append(t['esetup'] - t['eready']); s2.append(t['eq'] - t['esetup']); s3.append(c['ewait'] - t['eq'])
    print("eready -> esetup (smem reads, arrive):", m(s1))
    print("esetup -> eq (thr, q loads issued):", m(s2))
    print("eq -> first chunk ewait:", m(s3))
