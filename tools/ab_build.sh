#!/bin/bash
# Build libsprout.so from the working tree and libsprout_A.so from a git ref
# (default HEAD) for an A/B timing on the GPU box.  Usage: bash tools/ab_build.sh [REF]
set -e
REF=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REF" paper_2403_12900_b200 include | tar -x -C "$TMP"
(cd "$TMP" && python -m paper_2403_12900_b200.build --force > /dev/null)
cp "$TMP/paper_2403_12900_b200/libsprout.so" "$ROOT/paper_2403_12900_b200/libsprout_A.so"
rm -rf "$TMP"
(cd "$ROOT" && python -m paper_2403_12900_b200.build > /dev/null)
echo "built A=$REF -> libsprout_A.so, B=worktree -> libsprout.so"
