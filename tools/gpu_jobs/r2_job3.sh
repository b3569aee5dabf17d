# round 2, job 3: parity suite + full-size + bench + AA / e2e probes + ncu captures
# (ncu reports are exported to CSV on the box and deleted: gpurun_out must stay < 64 MiB)
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/j3_gpu.log 2>&1; echo gpu_rc=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/j3_bench.log 2>&1; echo bench_rc=$?
python tools/probe.py aa > gpurun_out/j3_aa.log 2>&1
python tools/probe.py e2e > gpurun_out/j3_e2e.log 2>&1
LBGPU_TRACE_PAIR=1 python tools/probe.py ncu e2e > gpurun_out/j3_e2e_trace.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/j3_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/j3_ncu_launch.log 2>&1; echo ncu1=$?
prof() {  # name regex skip target...
  local name=$1 re=$2 skip=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:$re -s $skip -c 1 -o /tmp/$name "$@" > gpurun_out/${name}_ncu.log 2>&1; echo ncu_$name=$?
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/${name}_details.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${name}_sass.csv.gz
  rm -f /tmp/$name.ncu-rep
}
prof j3_pair k_pair 2 python tools/probe.py ncu pair
prof j3_grad k_gradient 1 python tools/probe.py ncu gradient
prof j3_pair_aa k_pair_aa 2 python tools/probe.py ncu aa
du -sh gpurun_out
