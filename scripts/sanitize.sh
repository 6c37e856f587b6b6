# compute-sanitizer passes over the GPU tests (the full-size cases excluded:
# they take minutes under the tools) and the smoke entry point.
mkdir -p gpurun_out
for tool in memcheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 30 \
      python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not baseline_size and not loss_curve and not ipc and not concurrent" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitize_$tool.log
done
timeout 300 compute-sanitizer --tool initcheck python __graft_entry__.py smoke > gpurun_out/sanitize_smoke.log 2>&1
echo "smoke rc=$?"; tail -2 gpurun_out/sanitize_smoke.log
