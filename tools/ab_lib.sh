# A/B of kernel-variant builds under paper_2202_13821_b200/_ab/<name>/ against the in-tree library:
#   bash tools/ab_lib.sh name1 name2 ...   (bench ms/step, interleaved, 2 rounds)
set -e
for i in 1 2; do
 for v in main "$@"; do
  if [ $v = main ]; then L=""; else L=paper_2202_13821_b200/_ab/$v/libhgks_b200.so; fi
  HGKS_LIB=$L python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e ${AB_ARGS} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['ms_per_step'],3), {k: round(v['cell_ms'],3) for k, v in d['roofline']['per_stage_ms'].items()})" || echo "$v failed"
 done
done
