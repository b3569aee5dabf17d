# round 2, job 33: objective terms with L2-only loads (variant) -- DRAM bytes and J cost
set -x
python tools/probe.py e2e_alt > gpurun_out/j33_main.log 2>&1
LBGPU_LIB=$PWD/variants/cg.so python tools/probe.py e2e_alt > gpurun_out/j33_cg.log 2>&1
for v in main cg; do
  if [ $v = cg ]; then export LBGPU_LIB=$PWD/variants/cg.so; fi
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:k_objective_terms -c 3 --csv --log-file gpurun_out/j33_${v}_obj.csv python tools/probe.py ncu e2e > /dev/null 2>&1
done
