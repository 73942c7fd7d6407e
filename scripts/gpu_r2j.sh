#!/bin/bash
set -u
TAG=${TAG} bash scripts/gpu_quick2.sh
TAG=${TAG} bash scripts/gpu_sanitize.sh
