cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ALGOS="winograd" bash scripts/algo_launches.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm|winograd" -s 6 -c 3 -o gpurun_out/prof_wino -f \
  python scripts/layer_bench.py conv3_2 winograd --reps 2 > gpurun_out/ncu_wino.log 2>&1; echo "ncu rc=$?"
python scripts/layer_bench.py conv3_2 winograd implicit_gemm --reps 20
