O=gpurun_out; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ks_cluster -s 3 -c 1 -f -o $O/kc_c3 python tools/time_ops.py 16 30 2 1 > $O/kc_prof_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ks_cluster -s 3 -c 1 -f -o $O/kc_c4 python tools/time_ops.py 13 5 2 51 > $O/kc_prof_c4.log 2>&1
ls -la $O
