"""Basic-block breakdown of an ncu source page (SASS): runs of consecutive
instructions with one execution count, by share of executed warp
instructions, with average active threads and stall-sample share.
  ncu -i prof.ncu-rep --page source --csv --print-source sass > src.csv
  python tools/sass_blocks.py src.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h = rows[1]
ix = {k: h.index(k) for k in ("Source", "Instructions Executed", "Thread Instructions Executed",
                              "Warp Stall Sampling (All Samples)")}
ins = []
for r in rows[2:]:
    try:
        ins.append((r[ix["Source"]].strip(), int(r[ix["Instructions Executed"]] or 0),
                    int(r[ix["Thread Instructions Executed"]] or 0), int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
    except (ValueError, IndexError):
        pass
tot = sum(x[1] for x in ins)
stall = sum(x[3] for x in ins) or 1
blocks = []
i = 0
while i < len(ins):
    j = i
    while j + 1 < len(ins) and ins[j + 1][1] == ins[i][1]:
        j += 1
    ex = sum(x[1] for x in ins[i:j + 1])
    th = sum(x[2] for x in ins[i:j + 1])
    st = sum(x[3] for x in ins[i:j + 1])
    blocks.append((ex, i, j, ins[i][1], th / ex if ex else 0, st / stall, ins[i][0][:60]))
    i = j + 1
print(f"total warp instructions {tot:.4e}, {len(ins)} SASS instructions, avg threads "
      f"{sum(x[2] for x in ins) / max(tot, 1):.2f}")
print("| SASS idx | instrs | executions | share | stall share | thr | first instruction |")
print("|---|---|---|---|---|---|---|")
for ex, a, b, n, thr, st, src in sorted(blocks, reverse=True)[:top]:
    print(f"| {a}-{b} | {b - a + 1} | {n} | {ex / tot:.3f} | {st:.3f} | {thr:.1f} | `{src}` |")
