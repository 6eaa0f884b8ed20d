cd $GRAFT_REPO_ROOT
for n in 17 1023 1024 1025 2000 5000 70001 300007; do
  timeout 60 python tools/debug_sort.py rec100 $n >> gpurun_out/dbg_rec.log 2>&1 || echo "rec100 $n rc=$?" >> gpurun_out/dbg_rec.log
done
timeout 300 python bench.py --config H --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_H2.json 2>gpurun_out/bench_H2.err
