"""Summarise scripts/ab_krows.sh logs: median/min of the timed repetitions per (variant, family)."""
import re, sys
for path in sys.argv[1:]:
    lines = open(path).read().splitlines()
    print(path)
    for i, l in enumerate(lines):
        if l.strip().startswith('^'):
            ms = sorted(float(x) for x in re.search(r"ms=\[(.*?)\]", lines[i - 1]).group(1).split(',')[2:])
            print(f"  {l.strip()[2:]:20s} median {ms[len(ms) // 2]:.4f}  min {ms[0]:.4f}")
