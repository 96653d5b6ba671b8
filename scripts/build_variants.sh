#!/usr/bin/env bash
# Same-box A/B builds: libspmvb.so compiled with extra -D flags, copied to
# ab_libs/<name>.so (git-ignored, shipped to the GPU box); select one at run
# time with SPMVB_LIB_PATH.  Restores the default build at the end.
#   bash scripts/build_variants.sh name1 "-DFOO=1" name2 "-DBAR=2" ...
set -eu
root=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$root/ab_libs"
while [ $# -ge 2 ]; do
  SPMVB_NVCC_EXTRA="$2" python "$root/paper_1805_11938_b200/_build.py" >/dev/null
  cp "$root/paper_1805_11938_b200/libspmvb.so" "$root/ab_libs/$1.so"
  echo "ab_libs/$1.so  <- $2"
  shift 2
done
python "$root/paper_1805_11938_b200/_build.py" >/dev/null
