# round 2, job 10: in-place register bounds (variants) + the gated e2e kernel under ncu
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_facade.py tests/test_gpu_fdcheck.py -m gpu -q -p no:cacheprovider > gpurun_out/j10_gpu.log 2>&1; echo gpu_rc=$?
python tools/probe.py e2e > gpurun_out/j10_e2e.log 2>&1
python tools/probe.py rates streaming=aa > gpurun_out/j10_aa_main.log 2>&1
python tools/probe.py variants variants streaming=aa > gpurun_out/j10_aa_variants.log 2>&1
prof() {  # name regex skip target...
  local name=$1 re=$2 skip=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:$re -s $skip -c 1 -o /tmp/$name "$@" > gpurun_out/${name}_ncu.log 2>&1; echo ncu_$name=$?
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/${name}_details.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${name}_sass.csv.gz
  rm -f /tmp/$name.ncu-rep
}
prof j10_gated k_pair 1 python tools/probe.py ncu e2e
prof j10_pair k_pair 2 python tools/probe.py ncu pair
prof j10_obj k_objective_terms 1 python tools/probe.py ncu e2e
du -sh gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j10_e2e_launches.csv python tools/probe.py ncu e2e > gpurun_out/j10_e2e_ncu.log 2>&1; echo ncu_rc=$?
