#!/bin/bash
# Round evidence pass (run under gpurun, one GPU): the GPU test suite
# (FULL=1: with the whole-kv-group oracle runs), smoke, the default bench line,
# the ncu launch list of the bench command and `ncu --set full` captures of
# K5 / K8 at the headline shape (128K) and at Llama-3-8B 32K -> gpurun_out/
# TAG names the outputs (default r2).
TAG=${TAG:-r2}
bash tools/gpu_check.sh
# launch list of the bench command (kernel durations; cold, serialised: shares only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches_bench.csv \
  python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > /dev/null 2>&1
echo "ncu launch list=$?"
for shape in "131072 40 8" "32768 32 8"; do
  set -- $shape
  # K5: 2nd tc_sel_fwd launch (the extra forward); K8: 3rd tc_sel_bwd launch
  # (the step's selected and window launches come first)
  for ks in "tc_sel_fwd 1" "tc_sel_bwd 2"; do
    set -- $shape $ks
    k=$4
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k \
      --launch-skip $5 --launch-count 1 -f -o gpurun_out/${TAG}_${k}_$1 \
      python tools/prof_k8.py $1 $2 $3 > /dev/null 2>&1
    echo "ncu $k $1=$?"
  done
done
