#!/bin/bash
cd "$GRAFT_REPO_ROOT"
for i in 1 2; do
  TAG=old python abt/oldpkg/hemm_timing_old.py 30000 3000 20
  TAG=new python tools/hemm_timing.py 30000 3000 20
done
