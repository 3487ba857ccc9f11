"""Static SASS mnemonic histogram of the hot kernels of libxpcs.so (cuobjdump, no GPU needed): proves which
instructions the kernels are built from (UTCIMMA.2CTA / UTCHMMA.2CTA tcgen05 MMAs, LDTM TMEM loads, ELECT, MUFU ...).

    python tools/sass_histogram.py [--lib paper_2204_13241_b200/lib/libxpcs.so] [--json profiles/r02_sass_histogram.json]
"""
import argparse
import collections
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KERNELS = ["k_lattice_i8", "k_lattice_tc", "k_generic32", "k_g2", "k_xsvs_warp2", "k_species_combine2", "k_fix_chunks",
           "k_stage_lattice32"]
PROOF = ["UTCIMMA", "UTCHMMA", "UTCBAR", "LDTM", "ELECT", "MUFU.SIN", "MUFU.COS", "FFMA2", "FMUL2", "I2FP.F32.S32",
         "DFMA", "LDGSTS", "SYNCS"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2204_13241_b200", "lib", "libxpcs.so"))
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", a.lib], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if cur and m:
            funcs[cur][m.group(1)] += 1
    out = {}
    for k in KERNELS:
        for name, c in funcs.items():
            if re.search(r"\d" + re.escape(k) + r"(I|E|v)", name) and c:
                key = k
                while key in out:
                    key += "_"
                full = collections.Counter()
                for op, n in c.items():
                    full[op] += n
                out[key] = {"function": name, "static_instructions": sum(c.values()),
                            "top": dict(full.most_common(40)),
                            "proof": {p: sum(n for op, n in c.items() if op.startswith(p)) for p in PROOF}}
    txt = json.dumps(out, indent=1)
    if a.json:
        with open(a.json, "w") as fh:
            fh.write(txt + "\n")
    for k, v in out.items():
        print(k, v["static_instructions"], {p: n for p, n in v["proof"].items() if n})


if __name__ == "__main__":
    main()
