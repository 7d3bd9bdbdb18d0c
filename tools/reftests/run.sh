#!/bin/bash
# Run the reference's own test-suite (pkg/tests, 13 files) against the B200 drop-in.
#   build container:  tools/reftests/run.sh prepare     (copies the tests to baseline/_ref_tests)
#   GPU box:          tools/reftests/run.sh [pytest args]
# test_cli.py, test_bridge.py and test_config.py (its overrides go through cli.RunCfg) exercise the CLI and
# the websocket viewer, which are out of scope
# (SURVEY 2), and are not collected.
set -e
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
DST="$ROOT/baseline/_ref_tests"
if [ "$1" = "prepare" ]; then
    rm -rf "$DST" && mkdir -p "$DST"
    cp /root/reference/pkg/tests/*.py "$DST/"
    echo "copied $(ls "$DST" | wc -l) files to $DST"
    exit 0
fi
cd "$DST"
PYTHONPATH="$ROOT/tools/reftests:$ROOT:$PYTHONPATH" python -m pytest -q -p no:cacheprovider \
    --ignore=test_cli.py --ignore=test_bridge.py --ignore=test_config.py -rf "$@"
