"""Prints the INTEGRATION.md symbol table from include/ffit_b200.h: every exported function,
its header line, and the reference declaration it replaces (ffit_*) or the comment above it
or its group (ffcu_*)."""
import re
import sys

DECL = re.compile(r'^[A-Za-z_][\w\s\*]*?\b((?:ffit|ffcu)_\w+)\s*\(')


def first_clause(c, limit=170):
    if len(c) <= limit:
        return c
    depth = 0
    for i, ch in enumerate(c):
        depth += ch == '(' 
        depth -= ch == ')'
        if depth == 0 and i > 40 and ch in '.;' and (i + 1 == len(c) or c[i + 1] == ' '):
            return c[:i + 1]
    return c[:limit] + '…'


def rows(path):
    lines = open(path).read().split('\n')
    comment, i, out = '', 0, []
    while i < len(lines):
        s = lines[i].strip()
        if s.startswith('/*'):
            buf = [s]
            while '*/' not in lines[i]:
                i += 1
                buf.append(lines[i].strip())
            comment = re.sub(r'\s+', ' ', ' '.join(x.strip('/* ').strip() for x in buf)).strip()
            i += 1
            continue
        m = DECL.match(lines[i])
        if m:
            sec = re.match(r'-+\s*(\w[\w ]*):\s*reference include/ffit\.h:([\d-]+)', comment)
            ref = re.match(r'reference include/ffit\.h:([\d-]+)', comment)
            if sec:
                what = f"{sec.group(1)}; replaces reference `proj/include/ffit.h:{sec.group(2)}`"
            elif ref:
                what = f"replaces reference `proj/include/ffit.h:{ref.group(1)}`"
            else:
                what = first_clause(comment)
            out.append((m.group(1), i + 1, what.replace('|', '/')))
        i += 1
    return out


if __name__ == '__main__':
    path = sys.argv[1] if len(sys.argv) > 1 else 'include/ffit_b200.h'
    print('| Symbol | Line | What |\n|---|---|---|')
    for n, ln, w in rows(path):
        print(f'| `{n}` | {ln} | {w} |')
