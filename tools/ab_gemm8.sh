# A/B of 8-bit GEMM variants in one GPU session (tools/sweep.py per library build)
set -x
for r in 1 2; do
for v in main=paper_2209_04161_b200/libamsim.so pk8a=build/variants/libamsim_pk8a.so huge8=build/variants/libamsim_huge8.so huge8pk8a=build/variants/libamsim_huge8pk8a.so; do
  n=${v%%=*}; lib=${v#*=}
  for f in "" 5; do
    AMSIM_LIB=$PWD/$lib AMSIM_FORCE_CFG=$f timeout 300 python tools/sweep.py --sizes 4096 16384 --ms 7 --models mitchell 2>/dev/null | sed "s/^/{\"lib\": \"$n\", \"force\": \"$f\", \"round\": $r, \"r\": /; s/\$/}/"
  done
done
done
