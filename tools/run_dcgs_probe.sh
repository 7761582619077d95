for lib in base dc4 du3 dc4du3; do
  for tg in 8 4 2; do
    HELM_LIB=paper_2308_06152_b200/libhelm_$lib.so HELM_GS_TARGET=$tg timeout 120 python tools/dcgs_probe.py
  done
done
