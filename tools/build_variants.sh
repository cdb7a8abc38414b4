# Builds A/B variants of libelimtw.so into tools/ab/ (compile-time macros).
# usage: bash tools/build_variants.sh name "NVEXTRA flags" [name "flags" ...]
set -e
cd "$(dirname "$0")/../paper_1709_09990_b200"
mkdir -p ../tools/ab
while [ $# -ge 2 ]; do
  make -s -j8 BUILD=../build/v_$1 LIBOUT=../tools/ab/libelimtw_$1.so NVEXTRA="$2" > /dev/null
  echo "built tools/ab/libelimtw_$1.so ($2): $(grep -A2 'k_exact_scatterILi1ELb0ELb0' ../build/v_$1/ptxas.log | grep -o 'Used [0-9]* registers')"
  shift 2
done
