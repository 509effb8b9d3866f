set -u
O=gpurun_out/walkprof
mkdir -p $O
for c in 2 5s; do
  PS_LIB=paper_2505_00448_b200/libpairstat_b200_timing.so timeout 300 python tools/profile_one.py --config $c > $O/walk_cycles_$c.txt 2>&1
done
for c in 2 5s; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:spearman_walk -c 1 -o $O/ncu_$c python tools/profile_one.py --config $c > $O/ncu_$c.log 2>&1
  ncu -i $O/ncu_$c.ncu-rep --page source --csv --print-source cuda,sass > $O/src_$c.csv 2>/dev/null
  python tools/srcprof.py $O/src_$c.csv 60 > $O/srcprof_$c.txt 2>&1
done
echo done
