# bench lines for the other BASELINE configs (refresh)
for c in c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c --no-ref-engine > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"; tail -c 300 gpurun_out/bench_$c.json
done
