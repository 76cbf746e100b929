#!/bin/bash
# build experimental variants of libhdrlpa.so: build_exp.sh name "-DFLAG=1 ..." [name "flags"]...
# (variants build one after the other; each compiles its translation units in parallel)
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  n=$1; f=$2; shift 2
  python - "$n" "$f" <<'PY' > exp/ptxas_$n.log 2>&1 || echo "build $n failed"
import sys
from pathlib import Path
sys.path.insert(0, ".")
from paper_1308_4908_b200 import _native as N
N.compile_library(Path("exp") / f"lib_{sys.argv[1]}.so", sys.argv[2].split(), verbose_ptxas=True)
PY
  echo "$n: $(grep -A2 'lpa_fast_kernelILi2ELb1ELi6ELi0ELi2E' exp/ptxas_$n.log | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')"
done
