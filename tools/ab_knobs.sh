# graph-mode ms/step of one config under each knob setting (one process each):
#   CFG=3 KNOBS="NONE=0 IBGM_R_K0=8 IBGM_RI=8" bash tools/ab_knobs.sh
for rep in 1 2; do
  for kv in ${KNOBS}; do
    K=$([ "${CFG:-3}" = 4 ] && echo 60 || echo 400)
    echo -n "$kv "; env $kv timeout 300 python tools/ab_step.py ${CFG:-3} $K
  done
done
