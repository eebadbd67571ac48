# ncu --set full captures with source-level (SASS) stall attribution for a few
# layer passes; writes summaries and the source pages (CSV) to gpurun_out/.
#   bash tools/ncu_source.sh "l2.1.conv1 dgrad 256" "l3.1.conv2 dgrad 256" ...
mkdir -p /tmp/reps gpurun_out
for LP in "$@"; do
  set -- $LP
  tag=$1_$2_b$3
  AMSIM_DEBUG_PLAN=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:amsim_mm_kernel -s 1 -c 1 \
      -o /tmp/reps/prof_$tag python tools/prof_layer.py --layer $1 --pass $2 --batch $3 --reps 2 > gpurun_out/ncu_$tag.log 2>&1
  ncu -i /tmp/reps/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$tag.csv 2>/dev/null
done
python tools/ncu_summary.py /tmp/reps/*.ncu-rep > gpurun_out/ncu_summary_src.md
