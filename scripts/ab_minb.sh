set -e
for mb in 4 5; do
  SPMVB_NVCC_EXTRA="-DSPMVB_CSR5_MINB=$mb" python -c "from pathlib import Path; import importlib.util as u; s=u.spec_from_file_location('b', 'paper_1805_11938_b200/_build.py'); m=u.module_from_spec(s); s.loader.exec_module(m); m.build(force=True)"
  for t in 1 2; do python scripts/ab_flags.py 25 16 | tail -1 | sed "s/^/minb=$mb /"; done
done
python -c "from pathlib import Path; import importlib.util as u; s=u.spec_from_file_location('b', 'paper_1805_11938_b200/_build.py'); m=u.module_from_spec(s); s.loader.exec_module(m); m.build(force=True)"
