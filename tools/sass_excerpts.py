"""Per hot kernel of libtqp.so: register count (cuobjdump -res-usage), SASS instruction
count, the Blackwell-specific instructions it contains (TMA bulk copies UBLKCP, mbarrier
SYNCS, 256-bit loads LDG.*.256, match MATCH, redux REDUX) and a short excerpt around the
first of them. Writes profiles/sass_<tag>.md. Usage: python tools/sass_excerpts.py r02"""
import re
import subprocess
import sys
from collections import Counter

LIB = "paper_2203_01877_b200/libtqp.so"
HOT = ["scatter_tma_kernel", "probe_sector_kernel", "gb_dense_kernel", "expand_kernel", "bucket_r_kernel",
       "filter_mask_kernel", "gb_phase1_kernel", "andor_hist0_kernel", "part_scatter_kernel", "rank_bitmap_kernel"]
MARK = re.compile(r"\b(UBLKCP\S*|SYNCS\S*|LDG\S*256\S*|MATCH\S*|REDUX\S*|ATOMS\S*|STG\S*)")


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", sass)
    regs = dict(re.findall(r"Function (\S+):\s*\n\s*REG:(\d+)", res))
    out = [f"# SASS excerpts ({tag}): libtqp.so, sm_100a\n",
           "Counts are static (instructions in the function body).\n"]
    for hot in HOT:
        cands = [f for f in funcs if hot in f.split("\n", 1)[0]]
        if not cands:
            continue
        f = max(cands, key=len)   # the largest instantiation
        name = f.split("\n", 1)[0].strip()
        ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+([^;]+);", f)
        ops = Counter(i.split()[1] if i.startswith("@") else i.split()[0] for i in ins)
        marks = Counter(m.group(1).split(".")[0] + ("".join("." + x for x in m.group(1).split(".")[1:] if x in ("256", "NA", "ENL2", "EF")))
                        for i in ins for m in [MARK.search(i)] if m)
        out.append(f"\n## {hot}\n\n`{name[:160]}`\n")
        out.append(f"- registers: {regs.get(name, '?')}; SASS instructions: {len(ins)}")
        out.append("- Blackwell / memory-path instructions: " + ", ".join(f"{k} x{v}" for k, v in marks.most_common(10)))
        first = next((k for k, i in enumerate(ins) if re.search(r"UBLKCP|LDG\S*256|SYNCS", i)), None)
        if first is not None:
            out.append("\n```")
            out.extend(ins[max(0, first - 3):first + 5])
            out.append("```")
    open(f"profiles/sass_{tag}.md", "w").write("\n".join(out) + "\n")
    print("\n".join(out[:40]))


if __name__ == "__main__":
    main()
