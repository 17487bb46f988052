for v in 0 1; do
  CH_NVCC_EXTRA="-DHG_PTS_CG=$v" python -m paper_2303_10581_b200.build --force > /dev/null 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --profile-from-start off -k regex:k_points --csv python scripts/hull_prof.py 2>/dev/null | grep -o '"gpu__time_duration.sum".*\|"dram__bytes_read.sum".*\|"lts__t_sectors_srcunit_tex_op_read.sum".*' | sed "s/^/cg$v /" | cut -c1-100
done
python -m paper_2303_10581_b200.build --force > /dev/null 2>&1
