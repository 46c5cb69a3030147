#!/bin/bash
# Run the reference's own test modules against the product (see INTEGRATION.md,
# "Conformance against the reference's own tests").  Needs the git-ignored
# conformance/ harness (reference tests + rqcsim shim) in the tree; on a GPU box.
cd "$(dirname "$0")/../conformance" || exit 2
export NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1
timeout 1800 python -m pytest tests -q -p no:cacheprovider -rfE --tb=line "$@"
