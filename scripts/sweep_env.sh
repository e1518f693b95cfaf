# usage: bash scripts/sweep_env.sh <tag> VAR v1 v2 ... : bench + one-step launch-list summary per value
# (the value "-" leaves VAR unset)
O=gpurun_out/$1; V=$2; shift 2
mkdir -p $O
for x in "$@"; do
  if [ "$x" = "-" ]; then unset $V; else export $V=$x; fi
  echo "== $V=$x"
  x=$(basename "$x" | tr -c 'A-Za-z0-9_.\n-' '_')
  timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 5 --e2e-steps 1 > $O/bench_$x.json 2> $O/bench_$x.err
  python -c "import json,sys; d=json.loads(open('$O/bench_$x.json').readline()); print('ms/step', round(d['ms_per_step'],2), 'clk', d['clocks']['sm_mhz'])"
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/ll_$x.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras --e2e-steps 1 > /dev/null 2>&1
  python scripts/step_summary.py $O/ll_$x.csv | tail -n +2
done
unset $V
