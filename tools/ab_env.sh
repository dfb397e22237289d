# A/B of an environment knob on the graph-mode step: VAR=name VALS="a b c" CFGS="4 3" K4=60 bash tools/ab_env.sh
# (each value runs in its own process: the library reads its knobs once)
for rep in 1 2; do
  for cfg in ${CFGS:-4 3}; do
    for v in ${VALS}; do
      K=$([ "$cfg" = 4 ] && echo ${K4:-60} || echo 400)
      echo -n "$VAR=$v "; env $VAR=$v timeout 300 python tools/ab_step.py $cfg $K
    done
  done
done
