out=gpurun_out
mkdir -p $out
for k in "fa_fwd_tc3:attn_fwd" "fa_bwd_tc4:attn_bwd"; do
  IFS=: read -r name tag <<< "$k"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$name -s 2 -c 1 \
    -o $out/final_prof_$tag -f python tools/ncu_targets.py $tag > $out/final_ncu_$tag.log 2>&1
  ncu -i $out/final_prof_$tag.ncu-rep --page raw --csv > $out/final_raw_$tag.csv 2>/dev/null
  rm -f $out/final_prof_$tag.ncu-rep
done
