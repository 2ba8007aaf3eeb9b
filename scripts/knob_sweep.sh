# Device time of one contraction per tree under executor knob settings
# (each setting in a fresh process: the knobs are read at plan time).
#   bash scripts/knob_sweep.sh "given c4 2" "reordered c4 16" -- "" "TNB_PACE_MIN_MB=64" ...
O=gpurun_out/${SWEEP_TAG:-sweep}.txt
trees=(); while [ "$1" != "--" ] && [ -n "$1" ]; do trees+=("$1"); shift; done; shift
for knobs in "$@"; do
  for t in "${trees[@]}"; do
    for rep in 1 2; do
      r=$(env $knobs timeout -s KILL 600 python scripts/diag_tree.py $t 2>&1 | tail -1)
      echo "[$knobs] [$t] rep$rep $r" | tee -a $O
    done
  done
done
