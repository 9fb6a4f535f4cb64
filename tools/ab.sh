# A/B timing of library variants: bash tools/ab.sh CONFIG LANES variant.so...
c=$1; n=$2; shift 2
for v in "$@"; do
  echo "== $v"; B2S_LIBRARY=$PWD/$v python tools/prof_kernel.py --config $c --lanes $n --reps 5
done
