"""List `<file>.hpp:N[-M]` / `<file>.cpp:N` citations in the repo whose line
range does not exist in the reference (/root/reference).  Run here; prints
one line per suspicious citation."""
from __future__ import annotations

import re
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
REF = Path("/root/reference")
PAT = re.compile(r"([A-Za-z_][\w/]*\.(?:hpp|cpp|md|txt)):(\d+)(?:-(\d+))?")


def ref_lengths():
    out = {}
    for p in REF.rglob("*"):
        if p.is_file() and p.suffix in (".hpp", ".cpp", ".md", ".txt"):
            try:
                out.setdefault(p.name, []).append((p, len(p.read_text(errors="replace").splitlines())))
            except OSError:
                pass
    return out


def main() -> int:
    lens = ref_lengths()
    bad = 0
    for f in list(REPO.rglob("*")):
        if not f.is_file() or any(x in f.parts for x in (".git", "gpurun_out", "_ref", "build")):
            continue
        if f.suffix not in (".py", ".cu", ".cuh", ".h", ".hpp", ".cpp", ".c", ".md"):
            continue
        if f.name in ("SURVEY.md", "VERDICT.md", "ADVICE.md", "PAPERS.md", "SNIPPETS.md", "BASELINE.md"):
            continue
        for ln, line in enumerate(f.read_text(errors="replace").splitlines(), 1):
            for m in PAT.finditer(line):
                name = Path(m.group(1)).name
                if name not in lens:
                    continue
                hi = int(m.group(3) or m.group(2))
                if all(hi > n for _, n in lens[name]):
                    bad += 1
                    print(f"{f.relative_to(REPO)}:{ln}: {m.group(0)} (file has {max(n for _, n in lens[name])} lines)")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
