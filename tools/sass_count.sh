#!/bin/bash
# Opcode histogram of one block-kernel instantiation (no GPU needed):
#   tools/sass_count.sh double 5 2048 [extra nvcc -D flags...]
# compiles csrc/cbessfm_inst.cu for (real, P) and prints the per-opcode
# instruction counts of the kernels whose name contains "<real>, P, Q>".
set -e
REAL=${1:-double}; P=${2:-5}; Q=${3:-2048}; shift 3 || true
D=$(mktemp -d)
ROOT=$(cd "$(dirname "$0")/.." && pwd)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -Xptxas -v -DCB_REAL=$REAL -DCB_P=$P "$@" \
  -I"$ROOT/include" -c "$ROOT/paper_2409_14489_b200/csrc/cbessfm_inst.cu" -o $D/k.o 2> $D/ptxas.log
cuobjdump -sass $D/k.o > $D/k.sass
python3 - "$D/k.sass" "$REAL" "$P" "$Q" <<'PY'
import re, sys, collections
txt = open(sys.argv[1]).read()
real, P, Q = sys.argv[2:5]
for m in re.finditer(r"Function : (\S+)\n(.*?)(?=\n\s+Function : |\Z)", txt, re.S):
    name, body = m.group(1), m.group(2)
    if f"Li{P}ELi{Q}EE" not in name and not ("ip_kernel" in name and f"Li{P}EE" in name):
        continue
    ops = collections.Counter()
    for line in body.splitlines():
        mm = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if mm:
            ops[mm.group(1).split(".")[0]] += 1
    tot = sum(ops.values())
    fp = {k: v for k, v in ops.items() if k in ("DADD", "DFMA", "DMUL", "FADD", "FFMA", "FMUL", "FADD2", "FFMA2", "FMUL2")}
    print(name[:60], "total", tot, "fp", sum(fp.values()), dict(sorted(fp.items())))
    print("  top:", ops.most_common(14))
PY
grep -A2 -E "Li${P}ELi${Q}EE|ip_kernelI.Li${P}EE" $D/ptxas.log | grep -E "registers|spill" | head -6
rm -rf $D
