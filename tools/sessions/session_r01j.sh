#!/bin/bash
tools/gpu_session.sh r01j tests
tools/ab_session.sh r01j u1
tools/gpu_session.sh r01j ncu
