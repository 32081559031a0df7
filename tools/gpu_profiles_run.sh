#!/bin/bash
# Round profile session: launch lists + full captures (tools/gpu_profiles.sh),
# summarised on the box (make_profiles.py, ncu_digest.py) so only the small
# JSON / text digests come back; the .ncu-rep files are deleted.
TAG=${1:-r2c}
bash tools/gpu_profiles.sh $TAG
mkdir -p gpurun_out/prof_$TAG gpurun_out/digests_$TAG
python tools/make_profiles.py $TAG gpurun_out/prof_$TAG > gpurun_out/prof_$TAG/make.log 2>&1
for r in gpurun_out/prof_*_$TAG.ncu-rep; do
  wl=$(basename $r .ncu-rep | sed "s/^prof_//; s/_$TAG$//")
  python tools/ncu_digest.py $r > gpurun_out/digests_$TAG/digest_${wl}_$TAG.txt 2>&1
done
rm -f gpurun_out/*.ncu-rep
ls gpurun_out/prof_$TAG gpurun_out/digests_$TAG
