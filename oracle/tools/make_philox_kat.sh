#!/bin/sh
# Regenerates tests/golden/philox_kat.json from torch's Philox header.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
TI=$(python -c "import torch,os;print(os.path.join(os.path.dirname(torch.__file__),'include'))")
mkdir -p "$HERE/../build"
g++ -std=c++17 -O1 -I"$TI" -o "$HERE/../build/philox_kat" "$HERE/philox_kat.cpp"
"$HERE/../build/philox_kat" > "$HERE/../../tests/golden/philox_kat.json"
echo "wrote tests/golden/philox_kat.json"
