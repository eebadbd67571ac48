mkdir -p /tmp/reps
for LP in "l4.1.conv2 dgrad 32" "l4.1.conv2 dgrad 256" "l1.1.conv1 dgrad 32" "l2.1.conv2 fwd 32"; do
  set -- $LP
  AMSIM_DEBUG_PLAN=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:amsim_mm_kernel -s 1 -c 1 \
      -o /tmp/reps/prof_$1_$2_b$3 python tools/prof_layer.py --layer $1 --pass $2 --batch $3 --reps 2 > gpurun_out/ncu_$1_$2_b$3.log 2>&1
  AMSIM_DEBUG_PLAN=1 python tools/prof_layer.py --layer $1 --pass $2 --batch $3 --reps 5 >> gpurun_out/time_b32.log 2>&1
done
python tools/ncu_summary.py /tmp/reps/*.ncu-rep > gpurun_out/ncu_summary_b32.md
for f in /tmp/reps/*.ncu-rep; do ncu -i $f --page raw --csv > gpurun_out/raw_$(basename $f .ncu-rep).csv 2>/dev/null; done
