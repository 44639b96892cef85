"""Per-kernel SASS instruction evidence of libupir.so (cuobjdump -sass).

    python tools/sass_summary.py [lib] > profiles/r02_sass_summary.txt

For every kernel family (template variants collapsed: the maximum count of
each mnemonic over the variants) it counts the Blackwell-native
mnemonics that show what the kernel is built from: tcgen05 MMA (UTCHMMA /
UTCHMMA.2CTA), TMEM loads (LDTM), tcgen05 commits (UTCBAR), TMA tensor loads
(UTMALDG), bulk copies (UBLKCP), 256-bit loads / stores, mbarrier ops (SYNCS)
and FP32 FMAs."""
import collections
import re
import subprocess
import sys

PATS = [("UTCHMMA", r"^UTCHMMA(?!\.2CTA)"), ("UTCHMMA.2CTA", r"^UTCHMMA\.2CTA"), ("LDTM", r"^LDTM"),
        ("UTCBAR", r"^UTCBAR"), ("UTMALDG", r"^UTMALDG"), ("UBLKCP", r"^UBLKCP"),
        ("LDG.256", r"^LDG\..*\.256$"), ("STG.256", r"^STG\..*\.256$"), ("LDG.128", r"^LDG\..*\.128"),
        ("STG.128", r"^STG\..*\.128"), ("SYNCS(mbarrier)", r"^SYNCS"), ("FFMA", r"^FFMA$"), ("FFMA2", r"^FFMA2")]


def family(mangled):
    d = subprocess.run(["c++filt", mangled], capture_output=True, text=True).stdout.strip()
    d = re.sub(r"\(anonymous namespace\)::", "", d)
    m = re.match(r"(?:void )?(?:upir::)?([A-Za-z0-9_]+)", d)
    return (m.group(1) if m else d), d


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2209_10643_b200/libupir.so"
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)[1:]
    fams = collections.defaultdict(list)
    for f in funcs:
        name, body = f.split("\n", 1)
        ops = collections.Counter()
        n = 0
        for ln in body.splitlines():
            m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", ln)
            if not m:
                continue
            n += 1
            op = m.group(2)
            for key, pat in PATS:
                if re.search(pat, op):
                    ops[key] += 1
        fam, demangled = family(name.strip())
        fams[fam].append((ops, n, demangled))
    keys = [k for k, _ in PATS]
    print(f"SASS evidence of {lib} (cuobjdump -sass), sm_100a")
    print("kernel family (variants) | " + " | ".join(keys) + " | instructions")
    for fam in sorted(fams):
        vs = fams[fam]
        mx = {k: max(v[0][k] for v in vs) for k in keys}
        print(f"{fam} ({len(vs)}) | " + " | ".join(str(mx[k]) for k in keys) + f" | {max(v[1] for v in vs)}")
        print(f"    e.g. {vs[0][2][:160]}")


if __name__ == "__main__":
    main()
