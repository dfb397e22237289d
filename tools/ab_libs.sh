# A/B of library builds on the graph-mode step: LIBS="libibgm.so libibgm_B.so" CFGS="4" bash tools/ab_libs.sh
for rep in 1 2; do
  for cfg in ${CFGS:-4}; do
    for l in ${LIBS}; do
      K=$([ "$cfg" = 4 ] && echo ${K4:-60} || echo 400)
      IBGM_LIB_PATH=$PWD/paper_1305_3976_b200/$l timeout 300 python tools/ab_step.py $cfg $K
    done
  done
done
