cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in g1 g2 g4; do cp libsim_$v.so.alt paper_2503_15078_b200/libsim.so; echo "== $v"; timeout 300 python tools/prof_kpass_exp.py 2>&1 | tail -1;
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_kpass_pl" -s 4 -c 2 --csv python tools/prof_batched.py 1024 1 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | awk -F'","' '{print $5, $(NF-2), $NF}' | head -4; done > gpurun_out/ab5.txt 2>&1
