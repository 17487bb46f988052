for g in "" 32 64 128; do
  CH_L2_FETCH=$g timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --profile-from-start off -k regex:k_points --csv python scripts/hull_prof.py 2>&1 | grep -o 'L2 fetch.*\|"gpu__time_duration.sum".*\|"dram__bytes_read.sum".*\|"lts__t_sectors_srcunit_tex_op_read.sum".*' | sed "s/^/g$g /" | cut -c1-120
done
