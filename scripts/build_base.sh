#!/bin/bash
# Build libspmvb.so from a git revision (default HEAD) into build_ab/libspmvb_<rev>.so,
# for same-box A/B runs against the working tree (SPMVB_LIB_PATH selects the library).
set -eu
rev=${1:-HEAD}
root=$(cd "$(dirname "$0")/.." && pwd)
wt=$(mktemp -d /tmp/spmvb_base.XXXX)
git -C "$root" worktree add --detach "$wt" "$rev" >/dev/null
(cd "$wt" && python paper_1805_11938_b200/_build.py --force) >/dev/null
mkdir -p "$root/build_ab"
cp "$wt/paper_1805_11938_b200/libspmvb.so" "$root/build_ab/libspmvb_$rev.so"
git -C "$root" worktree remove --force "$wt"
echo "$root/build_ab/libspmvb_$rev.so"
