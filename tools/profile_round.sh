# Round profile capture (run under gpurun): tools/profile_round.sh A|B TAG
# Part A: launch list of the headline bench command + --set full of cfg4/cfg5;
# part B: --set full of cfg3/cfg1 and the two kernels of a config-2 call.
# Two parts keep each call's gpurun_out/ under the 64 MiB copy-back limit.
set -x
T=${2:-r01}
if [ "$1" = A ]; then
  python -m pytest tests -q -m gpu -x 2>&1 | tail -2
  python bench.py --steps 5 --warmup 3 --no-extra --e2e-steps 0 --no-check > gpurun_out/plain_launch.json 2>&1 || exit 1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_bench_cfg4.csv \
    python bench.py --steps 5 --warmup 3 --no-extra --e2e-steps 0 --no-check > /dev/null 2>&1
  CFGS="cfg4 cfg5"
else
  CFGS="cfg3 cfg1"
fi
for c in $CFGS; do
  python tools/profile_kernel.py $c 2 > /dev/null 2>&1 || exit 1
  ncu --set full --clock-control none --import-source on -k "regex:hash_kernel|tail_kernel|small_kernel" -s 1 -c 1 \
    -o gpurun_out/${T}_$c python tools/profile_kernel.py $c 2 > gpurun_out/${T}_$c.log 2>&1
done
if [ "$1" = B ]; then
  python tools/exp_varlen.py 40 > /dev/null 2>&1 || exit 1
  ncu --set full --clock-control none --import-source on -k "regex:hash_kernel|plan_kernel" -c 2 \
    -o gpurun_out/${T}_cfg2v40 python tools/exp_varlen.py 40 > gpurun_out/${T}_cfg2.log 2>&1
fi
ls -la gpurun_out/
