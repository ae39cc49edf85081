mkdir -p gpurun_out
R=$GRAFT_REPO_ROOT
for spec in "fix:." "r1:variants/w_7922f40"; do
  IFS=: read label d <<< "$spec"
  (cd $d && timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_kernel -s 1 -c 1 -o /tmp/ab_$label python $R/tools/c5_once.py > $R/gpurun_out/ab_${label}_ncu.log 2>&1)
  python tools/ncu_summary.py /tmp/ab_$label.ncu-rep > gpurun_out/ab_${label}_summary.json 2>&1
  python tools/ncu_lines.py /tmp/ab_$label.ncu-rep > gpurun_out/ab_${label}_lines.txt 2>&1
  cp /tmp/ab_$label.ncu-rep gpurun_out/
done
