for v in "" r32 r40 r48; do
  if [ -n "$v" ]; then export PCCP_LIB=$PWD/paper_2207_12116_b200/variants/libpccp_b200_$v.so; else unset PCCP_LIB; fi
  for g in 4 8 16; do
    echo "lib=$v gpc=$g $(python scripts/explore.py q14 --gpc $g 2>&1 | grep -v '{\"n_words' | grep -o 'kernel_ms[^,]*')"
  done
done
