# decode-ahead / late-decode re-tuning after the quad decode; stream-K alignment; ncu evidence; cfg sweep
set -x
python tools/ab_bench.py main=paper_2209_04161_b200/libamsim.so da2=build/variants/libamsim_da2.so da0=build/variants/libamsim_da0.so align3=build/variants/libamsim_align3.so --rounds 2 > gpurun_out/ab_da_mbm.jsonl 2>&1
python tools/ab_bench.py main=paper_2209_04161_b200/libamsim.so da2=build/variants/libamsim_da2.so late8off=build/variants/libamsim_late8off.so --rounds 2 --args "--steps 5 --warmup 3 --model mitchell" > gpurun_out/ab_da_mitchell.jsonl 2>&1
for v in main=paper_2209_04161_b200/libamsim.so align3=build/variants/libamsim_align3.so; do
  n=${v%%=*}; lib=${v#*=}
  AMSIM_LIB=$PWD/$lib timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_$n.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-full-step --no-exact-step > gpurun_out/bench_ncu_$n.log 2>&1
done
mkdir -p /tmp/reps
timeout 600 ncu --set full --clock-control none --import-source on -k regex:amsim_mm_kernel -s 2 -c 1 -o /tmp/reps/gemm8_4096 python tools/sweep.py --sizes 4096 --ms 7 --models mitchell > gpurun_out/ncu_gemm8.log 2>&1
ncu -i /tmp/reps/gemm8_4096.ncu-rep --page source --csv --print-source sass > gpurun_out/src_gemm8_4096.csv 2>/dev/null
bash tools/ncu_source.sh "l3.1.conv2 dgrad 256" "l1.1.conv2 dgrad 256" "l1.1.conv2 wgrad 256"
python tools/ncu_summary.py /tmp/reps/gemm8_4096.ncu-rep >> gpurun_out/ncu_summary_src.md
timeout 1500 python tools/cfg_sweep.py --reps 3 > gpurun_out/cfg_sweep_b256.jsonl 2> gpurun_out/cfg_sweep.err
