# A/B: the same explicit configurations with the kernel source of 6e70025 (oldtree/) and the current one
declare -a CFGS=(
 'tsmttsm d 41 41 {"AP": 41, "BP": 41, "EI": 1, "MT": 5, "NT": 160, "NTL": 3, "R": 32, "ctas": 3, "impl": 1, "stages": 3}'
 'tsmttsm d 49 49 {"AP": 49, "BP": 49, "EDGE": 4, "MT": 3, "NT": 288, "NTL": 3, "PLAIN": 1, "R": 32, "ctas": 2, "impl": 1, "stages": 4}'
 'tsmttsm d 50 50 {"AP": 50, "BP": 50, "MT": 2, "NT": 544, "NTL": 7, "R": 32, "ctas": 1, "impl": 1, "stages": 6}'
 'tsmttsm d 57 57 {"AP": 57, "BP": 57, "MT": 4, "NT": 544, "NTL": 4, "PLAIN": 1, "R": 64, "ctas": 1, "impl": 1, "stages": 3}'
 'tsmttsm d 26 26 {"AP": 26, "BP": 26, "EI": 1, "MT": 3, "NT": 160, "NTL": 3, "R": 64, "ctas": 2, "impl": 1, "stages": 3}'
 'tsmttsm d 64 64 {"AP": 64, "BP": 64, "MT": 4, "NT": 544, "NTL": 4, "PAIR": 1, "R": 64, "ctas": 1, "impl": 2, "stages": 3}'
)
for round in 1 2; do
for c in "${CFGS[@]}"; do
  set -- $c; op=$1; dt=$2; M=$3; N=$4; shift 4; cfg="$*"
  o=$(cd oldtree && timeout 120 python tools/one_config.py $op $dt $M $N "$cfg" --reps 9 2>/dev/null | tail -1 | python -c "import json,sys; print(round(json.load(sys.stdin)['ms'],4))")
  n=$(timeout 120 python tools/one_config.py $op $dt $M $N "$cfg" --reps 9 2>/dev/null | tail -1 | python -c "import json,sys; print(round(json.load(sys.stdin)['ms'],4))")
  echo "AB $op $dt $M old $o new $n"
done
done
