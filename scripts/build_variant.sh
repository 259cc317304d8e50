#!/bin/bash
# build a variant of the library into scripts/_dbg/<name>.so with extra -D flags (A/B timing);
# select it at run time with QB_LIB_PATH=scripts/_dbg/<name>.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
python - "$name" "$@" <<'PY'
import os, sys, paper_2407_14783_b200.build as b
name, flags = sys.argv[1], sys.argv[2:]
b.OBJ = f"scripts/_dbg/obj_{name}"; b.LIB = os.path.abspath(f"scripts/_dbg/{name}.so")
b.build(force=True, extra_flags=flags)
print(b.LIB)
PY
