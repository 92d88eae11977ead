# A/B/n: per-launch device times of several libgsde.so builds over bench workloads.
# usage: LIBS="build_exp/a/libgsde.so build_exp/b/libgsde.so" WORKLOADS="star3 hub64" R=2 N=6 bash tools/abn.sh
for r in $(seq ${R:-2}); do for w in ${WORKLOADS:-star3 hub64 vascular}; do for lib in $LIBS; do
  echo -n "$(basename $(dirname $lib)) "; GSDE_LIB_PATH=$lib timeout 300 python tools/jitter.py $w ${N:-6} 2>/dev/null | tail -1
done; done; done
