set -u
LIB=paper_2405_11671_b200/libgbg.so
cp $LIB /tmp/orig.so
for v in pr_base pg3; do
  cp profiles/ab/$v.so $LIB
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:pr_tile_k -s 1 -c 1 -o gpurun_out/ncu_$v python profiles/prof_pr.py 24 > gpurun_out/ncu_$v.log 2>&1
  echo "$v=$?"
done
cp /tmp/orig.so $LIB
