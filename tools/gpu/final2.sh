# final records + the checked-build suite in one call: $1 = commit label
bash tools/gpu/final.sh "$1"
bash tools/gpu/checked.sh
