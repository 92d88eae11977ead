# A/B two builds of libgsde.so over bench workloads (per-launch device times, back to back).
# usage: A=path/libgsde.so B=path/libgsde.so WORKLOADS="star3 hub64" R=2 bash tools/ab.sh
for r in $(seq ${R:-2}); do for w in ${WORKLOADS:-star3 hub64 vascular}; do for v in A B; do
  lib=${!v}
  echo -n "$v "; GSDE_LIB_PATH=$lib timeout 300 python tools/jitter.py $w ${N:-6} 2>/dev/null | tail -1
done; done; done
