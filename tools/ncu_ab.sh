M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_read.sum
mkdir -p gpurun_out/ncuab
for v in default nopack; do
  if [ $v = nopack ]; then export OCTF_NO_PACK=1; else unset OCTF_NO_PACK; fi
  timeout 600 ncu --metrics $M --clock-control none -k regex:"k_leaf_pass|k_pd_pass" -s 2 -c 4 --csv python tools/profile_cfg5.py --passes 3 > gpurun_out/ncuab/$v.csv 2> gpurun_out/ncuab/$v.err
done
