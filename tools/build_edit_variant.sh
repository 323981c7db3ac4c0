#!/bin/bash
# Build libgs_NAME.so from the working tree's csrc with sed edits applied to a temporary copy
# (A/B of compile-time constants without touching the tree).
#   tools/build_edit_variant.sh NAME FILE 'sed-expression' [FILE 'sed-expression' ...]
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
mkdir -p "$TMP/paper_2406_18533_b200"
cp -r "$ROOT/paper_2406_18533_b200/csrc" "$TMP/paper_2406_18533_b200/"
cp -r "$ROOT/include" "$TMP/"
while [ $# -ge 2 ]; do
  sed -i "$2" "$TMP/paper_2406_18533_b200/csrc/$1"
  grep -q . "$TMP/paper_2406_18533_b200/csrc/$1"
  shift 2
done
cd "$ROOT"
python - "$TMP/paper_2406_18533_b200/csrc" "$ROOT/paper_2406_18533_b200/libgs_$NAME.so" <<'PY'
import importlib, sys
b = importlib.import_module("paper_2406_18533_b200.build")
print(b.build(force=True, csrc=sys.argv[1], out=sys.argv[2]))
PY
rm -rf "$TMP"
