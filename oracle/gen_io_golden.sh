#!/bin/bash
# TEST INFRASTRUCTURE ONLY: regenerate tests/golden/io/ with the reference's
# own raw / checkpoint writers (compiled from /root/reference in place; the
# nlohmann json header the reference includes comes from the image's
# cudnn_frontend include tree).  Not needed on the GPU box.
set -euo pipefail
HERE=$(cd "$(dirname "$0")" && pwd)
REF=${REF:-/root/reference/proj}
JSON=${JSON:-$(python -c 'import os, site; print(next(p for p in (os.path.join(s, "include/cudnn_frontend/thirdparty/nlohmann") for s in site.getsitepackages()) if os.path.exists(os.path.join(p, "json.hpp"))))')}
mkdir -p "$HERE/_build" "$HERE/../tests/golden/io"
g++ -O2 -std=c++20 -ffp-contract=off -w -I"$REF/include" -I"$JSON" -o "$HERE/_build/gen_io_golden" \
    "$HERE/gen_io_golden.cpp" "$REF/src/io_raw.cpp" "$REF/src/checkpoint.cpp" "$REF/src/nifti.cpp"
"$HERE/_build/gen_io_golden" "$HERE/../tests/golden/io"
