#!/bin/bash
# Same-box A/B of two library builds: ab_lib.sh BASE_SO WORKLOADS FORMATS [ROUNDS]
# (BASE_SO from scripts/build_base.sh; the other arm is the working tree's build)
base=$1; wl=$2; fm=$3; rounds=${4:-3}
for r in $(seq "$rounds"); do
  SPMVB_LIB_PATH=$base python scripts/time_formats.py --workloads "$wl" --formats "$fm"
  python scripts/time_formats.py --workloads "$wl" --formats "$fm"
done
