# SPDX-License-Identifier: Apache-2.0
"""SASS listing of every kernel in libvsa_b200.so (north_star: "each kernel ships with
... a SASS listing").

    python tools/sass_dump.py [lib] [outdir]

Writes profiles/sass/<kernel>.sass (cuobjdump -sass, instruction text only: the /* hex */
encodings and blank lines are dropped) for every kernel, and profiles/sass/summary.json
with each kernel's instruction count and the mnemonics that prove the execution path:
tcgen05 MMA (UTC*MMA), TMEM loads/stores (LDTM/STTM), TMA (UTMALDG/UTMASTG/UTMAPF/UBLKCP),
legacy tensor cores (HMMA), FP32 FMA (FFMA/FFMA2), cp.async (LDGSTS), registers per thread.
"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "UTMACCTL", "HMMA", "FFMA",
        "FFMA2", "FADD2", "FMUL2", "MUFU.EX2", "LDGSTS", "SYNCS", "LDS", "STS", "LDG", "STG", "BAR", "SHFL", "ATOMG",
        "RED"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, out))


def short(dem: str) -> str:
    base = dem.split("(")[0].replace("vsa_dev::", "").replace("void ", "")
    base = base.replace("__nv_bfloat16", "bf16").replace("<", "_").replace(">", "").replace(", ", "_")
    return re.sub(r"[^A-Za-z0-9_]", "", base)


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2505_13389_b200", "_lib", "libvsa_b200.so")
    outdir = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "sass")
    os.makedirs(outdir, exist_ok=True)
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
    regs = {}
    for m in re.finditer(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+) SHARED:(\d+)", res):
        regs[m.group(1)] = dict(regs=int(m.group(2)), stack=int(m.group(3)), static_shared=int(m.group(4)))
    funcs = re.split(r"\n\s*Function : ", sass)[1:]
    names = [f.split("\n", 1)[0].strip() for f in funcs]
    dem = demangle(names)
    summary = {}
    for name, body in zip(names, funcs):
        lines = []
        for ln in body.split("\n")[1:]:
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*?)\s*;?\s*(/\*.*)?$", ln)
            if m and m.group(2):
                lines.append(f"/*{m.group(1)}*/ {m.group(2)}")
            elif ln.strip().startswith(".L"):
                lines.append(ln.strip())
        ops = collections.Counter()
        for ln in lines:
            parts = ln.split("*/ ", 1)
            if len(parts) < 2:
                continue
            ins = re.sub(r"^@!?U?P[T0-9]\s+", "", parts[1]).split()
            if not ins:
                continue
            op = ins[0]
            ops[op] += 1
        key = short(dem[name])
        # the SIMT fine kernels (fp32 parity / debug path, ~1 MB of unrolled FFMA each) are
        # summarised only, unless SASS_ALL=1
        if "simt" not in key or os.environ.get("SASS_ALL") == "1":
            with open(os.path.join(outdir, key + ".sass"), "w") as f:
                f.write(f"// {dem[name]}\n// {name}\n// cuobjdump -sass {os.path.basename(lib)} (encodings dropped)\n")
                f.write("\n".join(lines) + "\n")
        counts = {k: sum(v for op, v in ops.items() if op == k or op.startswith(k + ".")) for k in KEYS}
        summary[key] = dict(function=dem[name], instructions=len(lines),
                            path={k: v for k, v in counts.items() if v}, **regs.get(name, {}))
    with open(os.path.join(outdir, "summary.json"), "w") as f:
        json.dump(summary, f, indent=1, sort_keys=True)
    print(f"{len(summary)} kernels -> {outdir}")


if __name__ == "__main__":
    main()
