"""Per-kernel SASS instruction evidence of librmips.so: counts of the Blackwell tensor-core, TMEM and
TMA instructions (cuobjdump -sass).  Usage: python tools/sass_summary.py [lib] > profiles/r02_sass_summary.md"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2110_07131_b200/librmips.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
pats = {
    "UTCHMMA": r"\bUTCHMMA(?!\.2CTA)", "UTCHMMA.2CTA": r"\bUTCHMMA\.2CTA", "UTCBAR": r"\bUTCBAR\b(?!\.2CTA)",
    "UTCBAR.2CTA": r"\bUTCBAR\.2CTA", "UTCCP": r"\bUTCCP\.T\.S(?!\.2CTA)", "UTCCP.2CTA": r"\bUTCCP\.T\.S\.2CTA",
    "UTMALDG": r"\bUTMALDG\.2D(?!\.2CTA)", "UTMALDG.2CTA": r"\bUTMALDG\.2D\.2CTA", "LDTM": r"\bLDTM\.",
    "UTCATOMSWS (TMEM alloc)": r"\bUTCATOMSWS\.", "DFMA": r"\bDFMA\b", "instructions": r"^\s+/\*[0-9a-f]{4,}\*/",
}
cnt = collections.OrderedDict()
cur = None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        cnt[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    for k, p in pats.items():
        if re.search(p, line):
            cnt[cur][k] += 1


def short(name):
    d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    d = re.sub(r"\(.*\)$", "", d)
    return d.replace("rmips::", "").replace("(anonymous namespace)::", "")


cols = [k for k in pats if k != "instructions"]
print("# SASS evidence: `cuobjdump -sass %s`\n" % lib.rsplit("/", 1)[-1])
print("Counts of static instructions per kernel (tcgen05 MMA = UTCHMMA, commit = UTCBAR, smem->TMEM copy = UTCCP,")
print("TMA tile load = UTMALDG, TMEM load = LDTM; `.2CTA` = cta_group::2).  Kernels without any of them omitted.\n")
print("| kernel | " + " | ".join(cols) + " | SASS instr |")
print("|---|" + "---:|" * (len(cols) + 1))
for f, c in cnt.items():
    if not any(c[k] for k in cols if k != "DFMA") and not c["DFMA"]:
        continue
    print("| `%s` | " % short(f) + " | ".join(str(c[k]) for k in cols) + " | %d |" % c["instructions"])
