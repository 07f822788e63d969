# Encode the bench workload with the REFERENCE pipeline (dev container only; ~5 min on 8 cores).
# Outputs cache/<kind>_<M>x<K>_s<sparsity>_seed<seed>.ecsr, read by bench.py.
set -e
cd "$(dirname "$0")/.."
mkdir -p cache
jobs=(
 "magnitude 4096 4096 0.5 101" "magnitude 4096 4096 0.5 102" "magnitude 4096 4096 0.5 103"
 "magnitude 4096 4096 0.5 104" "magnitude 11008 4096 0.5 105" "magnitude 11008 4096 0.5 106"
 "magnitude 4096 11008 0.5 107"
)
for j in "${jobs[@]}"; do
  set -- $j
  out=cache/$1_$2x$3_s$4_seed$5.ecsr
  [ -f "$out" ] || python scripts/ref_convert.py $1 $2 $3 $4 $5 $out &
done
wait
