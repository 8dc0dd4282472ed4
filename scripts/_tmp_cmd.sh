cd $GRAFT_REPO_ROOT
for lib in paper_1712_09789_b200/_lib/libccl_b200*.so; do echo "== $lib"; CCL_LIB_PATH=$lib PROBE_CHECK=0 timeout 200 python -c "
import sys; sys.argv=['probe']; sys.path.insert(0,'scripts'); sys.path.insert(0,'.')
import probe, paper_1712_09789_b200 as ccl
img=ccl.random_image(8192,8192,0.5,0)
for v in ['c2fl','rc2fl']: probe.run('random 8192 d0.5', img, v)
probe.run('random 8192 d0.9', ccl.random_image(8192,8192,0.9,0))
" 2>&1 | grep -v "^NVIDIA"; done > gpurun_out/sweep2.log 2>&1
