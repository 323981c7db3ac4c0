#!/bin/bash
# Build libgs from the csrc/ of git revision REV into paper_2406_18533_b200/libgs_NAME.so
# (A/B timing on the same GPU box: GS_LIB_VARIANT=NAME python bench.py ...).
#   tools/build_variant.sh REV NAME
set -e
REV=$1; NAME=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_2406_18533_b200/csrc include | tar -x -C "$TMP"
cd "$ROOT"
python - "$TMP/paper_2406_18533_b200/csrc" "$ROOT/paper_2406_18533_b200/libgs_$NAME.so" <<'PY'
import importlib, sys
b = importlib.import_module("paper_2406_18533_b200.build")
print(b.build(force=True, csrc=sys.argv[1], out=sys.argv[2]))
PY
rm -rf "$TMP"
