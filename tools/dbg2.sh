cd $GRAFT_REPO_ROOT
for n in 1025 1100 2000 5000 70001 300007; do
  timeout 60 python tools/debug_sort.py rec100 $n 2>&1 | cut -c1-60 >> gpurun_out/dbg_rec.log
  IPS4O_K3=regs timeout 60 python tools/debug_sort.py rec100 $n 2>&1 | cut -c1-60 | sed 's/^/regs /' >> gpurun_out/dbg_rec.log
done
