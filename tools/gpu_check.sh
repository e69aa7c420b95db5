#!/bin/bash
# One GPU verification pass (run under gpurun): GPU tests (without the
# whole-group oracle runs unless FULL=1), smoke, bench -> gpurun_out/
rm -f gpurun_out/parity.jsonl
if [ -n "$FULL" ]; then
  FSA_PARITY_REPORT=gpurun_out/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/gputest_all.log 2>&1
else
  FSA_PARITY_REPORT=gpurun_out/parity.jsonl timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -k "not whole" > gpurun_out/gputest_all.log 2>&1
fi
echo "pytest=$?"; tail -4 gpurun_out/gputest_all.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
if [ -z "$NOBENCH" ]; then
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench=$?"
fi
