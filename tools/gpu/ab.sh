# A/B per-phase timings: bash tools/gpu/ab.sh "ENV1=a ENV2=b" "ENV1=c" ...  (each arg one variant)
out=gpurun_out/ab_$(date +%s).log
for v in "$@"; do
  echo "== $v" >> $out
  env $v timeout 300 python tools/ab_phases.py c1_500k 30 >> $out 2>&1
done
cat $out
