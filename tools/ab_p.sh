mkdir -p gpurun_out/ab_p
for lib in default lentz; do
  if [ $lib = default ]; then L=""; else L="PS_LIB=$PWD/paper_2505_00448_b200/libpairstat_b200_lentz.so"; fi
  env $L timeout 600 ncu --metrics gpu__time_duration.sum -k regex:pearson_p_kernel --clock-control none --csv python tools/profile_one.py --config 5 --scale 0.5 > gpurun_out/ab_p/$lib.csv 2> gpurun_out/ab_p/$lib.err
done
