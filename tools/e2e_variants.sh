#!/bin/bash
# device-resident vs end-to-end (ABI host path, HostPipeline) for bench variants: bash tools/e2e_variants.sh "" "--fused --wave 64" ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in "$@"; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-volume $v 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']
print('%-28s dev %7.0f  e2e %7.0f  pipeline %7.0f  wave %s' % ('$v', d['value'], e['value'], e.get('host_pipeline',{}).get('value',0), d['config'].get('wave')))"
done
