set -x
bash tools/gpu_sanitize.sh racecheck smoke
bash tools/gpu_sanitize.sh racecheck syev
bash tools/gpu_sanitize.sh synccheck all
bash tools/gpu_sanitize.sh memcheck smoke
