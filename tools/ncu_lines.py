"""Diagnostic: aggregate ncu source-page stall samples of one kernel by CUDA source line (cuda,sass view)."""
import csv, collections, subprocess, sys, io
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
mix = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
cu = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda'],
                    capture_output=True, text=True).stdout
src = {int(r[0]): r[1] for r in csv.reader(io.StringIO(cu)) if r and r[0].isdigit()}
rows = list(csv.reader(io.StringIO(mix)))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'Line No'][0]
h = rows[hi]
si = h.index('Warp Stall Sampling (All Samples)')
reasons = [k for k in h if k.startswith('stall_') and 'Not Issued' not in k]
ri = [h.index(k) for k in reasons]
agg = collections.Counter()
rag = collections.defaultdict(collections.Counter)
for r in rows[hi + 1:]:
    if not r or not r[0].isdigit():
        continue
    ln = int(r[0])
    try:
        agg[ln] += int(r[si] or 0)
        for k, j in zip(reasons, ri):
            rag[ln][k] += int(r[j] or 0)
    except ValueError:
        pass
tot = sum(agg.values())
print("total samples", tot)
for ln, v in agg.most_common(top):
    rs = ", ".join(f"{k[6:]}={c}" for k, c in rag[ln].most_common(3) if c)
    print(f"{v / tot * 100:5.1f}% {ln:5d} {src.get(ln, '')[:80]:80s} | {rs}")
