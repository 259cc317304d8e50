#!/bin/bash
# debug build of the library with the k_render_f pixel trace (QB_RF_DEBUG) into scripts/_dbg/
set -e
cd "$(dirname "$0")/.."
python - <<'PY'
import os, shutil, paper_2407_14783_b200.build as b
b.OBJ = "scripts/_dbg/obj"; b.LIB = os.path.abspath("scripts/_dbg/libquadb200_dbg.so")
b.build(force=True, extra_flags=["-DQB_RF_DEBUG"])
print(b.LIB)
PY
